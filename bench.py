#!/usr/bin/env python3
"""Benchmark of the Occult expert-parallel MoE layer on B200.

Metric (BASELINE.json): MoE layer tokens/s at 1/2/4/8 B200; all-to-all
bytes/token vs naive top-k.  Workload: the Mixtral-8x7B MoE layer
(BASELINE configs[1]: 8 experts top-2, d=4096, ffn=14336, SwiGLU) prefilling
16,384 tokens; EP degree = number of GPUs; synthetic tokens and random-init
experts of that shape.  One step = route (gate GEMV, softmax, top-2) +
dispatch plan + pack/exchange + grouped SwiGLU FFN + intra-device partial
combine + return + combine, over one 16k-token batch.

Arms:
  default            this package's sm_100a path (C-ABI via the Python mirror)
  --impl reference   the reference's own CPU implementation (oracle/_ref,
                     compiled from /root/reference sources) on the host cores
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE layer tokens/s at 1/2/4/8 B200; all-to-all bytes/token vs naive top-k"
# BASELINE.json configs.  The driver's bench line is "mixtral" (configs[1]);
# the others are selectable with --workload for the record (profiles/).
WORKLOADS = {
    "mixtral": dict(E=8, k=2, D=4096, F=14336, act="swiglu", tokens=16384, nd_sim=1, plan_ep=8, train=False,
                    prune=None, name="Mixtral-8x7B MoE layer (8 experts top-2, d=4096, ffn=14336, SwiGLU) "
                                     "prefill 16384 tokens, EP=#GPUs"),
    "c1": dict(E=8, k=2, D=512, F=1024, act="silu", tokens=2048, nd_sim=2, plan_ep=2, train=False, prune=None,
               name="single MoE layer, 8 experts top-2, d=512, d_ff=1024, 2048 tokens, 2 simulated EP ranks "
                    "(reference CPU oracle shape; 2-matrix SiLU experts)"),
    "deepseek": dict(E=64, k=6, D=2048, F=1408, act="swiglu", tokens=16384, nd_sim=1, plan_ep=8, train=False,
                     prune=None, shared=(2, 1408, False), coactivation_placement=True,
                     name="DeepSeek-MoE-16B layer (64 routed experts top-6 + 2 shared experts, d=2048, ffn=1408, "
                          "SwiGLU) 16384 tokens"),
    "olmoe": dict(E=64, k=8, D=2048, F=1024, act="swiglu", tokens=65536, nd_sim=1, plan_ep=8, train=True,
                  prune=None, name="OLMoE-1B-7B layer (64 experts top-8, d=2048, ffn=1024, SwiGLU) "
                                   "forward+backward at 65536 tokens/step"),
    "qwen": dict(E=60, k=4, D=2048, F=1408, act="swiglu", tokens=16384, nd_sim=4, plan_ep=4, train=False,
                 prune=("router", 2), shared=(1, 5632, True), extra_eps=(2, 8),
                 name="Qwen1.5-MoE-A2.7B layer (60 routed experts top-4, d=2048, ffn=1408, SwiGLU; + gated shared "
                      "expert ffn=5632) with collaboration pruning to <=2 devices/token, EP=4 simulated on one GPU"),
}
W = WORKLOADS["mixtral"]
E, K_TOP, D, F = W["E"], W["k"], W["D"], W["F"]
TOKENS = W["tokens"]
WORKLOAD = W["name"]


def select_workload(name):
    global W, E, K_TOP, D, F, TOKENS, WORKLOAD
    W = WORKLOADS[name]
    E, K_TOP, D, F = W["E"], W["k"], W["D"], W["F"]
    TOKENS = W["tokens"]
    WORKLOAD = W["name"]


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                c = [x.strip() for x in line.split(",")]
                if len(c) < 9:
                    continue
                try:
                    sm.append(float(c[1]))
                    mx = max(mx, float(c[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, c[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "samples": len(sm), "reasons": sorted(reasons)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------- reference arm --
def reference_sample(threads, tokens_per_thread, seed=1):
    """Mixtral-shaped layer on the reference CPU path.  The reference has no
    gated experts, so its closest layer is the 2-matrix SiLU
    expert at the same shape (2/3 of the SwiGLU FLOPs)."""
    import numpy as np
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    n = threads * tokens_per_thread
    x = rng.uniform(-1, 1, (n, D))
    g = rng.uniform(-1, 1, (E, D)) * (3.0 / np.sqrt(D))
    w1 = rng.uniform(-1, 1, (E, D, F)) / np.sqrt(D)
    w2 = rng.uniform(-1, 1, (E, F, D)) / np.sqrt(F)
    return O, x, g, w1, w2


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import ctypes as C

    import numpy as np
    threads = os.cpu_count() or 1
    tpt = args.ref_tokens_per_thread
    O, x, g, w1, w2 = reference_sample(threads, tpt)
    L = O.ref_lib()
    n = x.shape[0]
    out = np.empty_like(x)
    P = lambda a: a.ctypes.data_as(C.c_void_p)
    # the layer's experts / gate / placement held in the reference's own types
    # (built once, outside the timed steps, as a moesim caller would)
    sess = L.ref_session_create(P(g), E, K_TOP, P(w1), P(w2), D, F, 8, 1, 1)
    if not sess:
        raise RuntimeError("reference session could not be created")

    def step():
        t0 = time.perf_counter()
        rc = L.ref_session_forward(sess, P(x), n, threads, P(out))
        if rc < 0:
            raise RuntimeError(f"reference failed: status {-rc}")
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    tot = sum(times)
    value = n * args.steps / tot
    L.ref_session_destroy(sess)
    sample = (f"{n} tokens/step ({tpt} per thread x {threads} threads) through the reference's "
              f"forward_expert_parallel (gate_scores + topk_route + forward_given_routing; reference sources, "
              f"g++ -O2; experts converted to moesim types once, outside the timed steps), 2-matrix SiLU experts "
              f"at d=4096, ffn=14336, EP=8 simulated (reference has no gated experts)")
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "experts": E, "top_k": K_TOP, "d_model": D, "d_ff": F,
                       "tokens_per_step": n},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_port_baseline(seconds_target=15.0):
    """The oracle restatement (SwiGLU-capable, the reference's loops) on all
    host cores: same workload shape, bounded token sample."""
    import ctypes as C

    import numpy as np
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(7)
    w1 = rng.uniform(-1, 1, (E, D, F)) / np.sqrt(D)
    w3 = rng.uniform(-1, 1, (E, D, F)) / np.sqrt(D)
    w2 = rng.uniform(-1, 1, (E, F, D)) / np.sqrt(F)
    lib = O.port_lib()
    plist = np.arange(E, dtype=np.int32).reshape(1, E)
    P = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)

    def chunk(tokens, out_times, idx):
        x = rng.uniform(-1, 1, (tokens, D))
        ids = np.stack([np.random.default_rng(idx * 1000 + t).permutation(E)[:K_TOP] for t in range(tokens)])
        ids = ids.astype(np.int32)
        w = np.full((tokens, K_TOP), 0.5)
        src = np.zeros(tokens, np.int32)
        y = np.empty_like(x)
        rep = O.Report()
        t0 = time.perf_counter()
        lib.orc_forward_given_routing(P(x), tokens, D, P(ids), P(w), K_TOP, P(w1), P(w2), P(w3), E, F, P(plist), 1,
                                      P(src), 1, 1, 2, -1.0, P(y), C.byref(rep), None, None, None, None, None)
        out_times[idx] = time.perf_counter() - t0

    # calibrate on one token, then size the sample to ~seconds_target
    t = [0.0]
    chunk(1, t, 0)
    per_tok = max(t[0], 1e-3)
    tpt = max(1, int(seconds_target / per_tok))
    times = [0.0] * threads
    ths = [threading.Thread(target=chunk, args=(tpt, times, i)) for i in range(threads)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    wall = time.perf_counter() - t0
    n = tpt * threads
    return {"value": n / wall, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"{n} tokens ({tpt} per thread x {threads} threads) of the SwiGLU layer at d=4096, ffn=14336, "
                      f"top-2 of 8, EP=1, oracle/occ_oracle.c (fp64, the reference's loop order), wall {wall:.1f} s"}


# ----------------------------------------------------------------- our arm --
def run_ours(args):
    import numpy as np
    import torch

    import paper_2505_13345_b200 as occ

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    peaks, peaks_src = load_peaks()
    n_local = args.tokens // world
    torch.manual_seed(1234 + rank)

    nd = W["nd_sim"] if world == 1 else world
    gated = W["act"] == "swiglu"
    prune = occ.PruneSpec(W["prune"][0], W["prune"][1]) if W["prune"] else None
    e_local = E if world == 1 else E // world

    def build_layer(use_peer, dedup=True):
        """The layer of this rank: NCCL communicator, optionally the fused
        peer-memory exchange, resident experts (+ shared experts); dedup=False
        is the replicate-k dispatch (one row per (token, expert))."""
        cfg = occ.MoEConfig(E, K_TOP, nd, D, F, activation=W["act"], dedup=dedup)
        layer = occ.ExpertParallelLayer(cfg, world_size=world, rank=rank)
        exchange = "local"
        if world > 1:
            layer.comm_init()
            exchange = "nccl all-to-all"
            if use_peer:  # fused pack/return stores over NVLink peer memory
                try:
                    layer.comm_enable_peer(n_local)
                    exchange = "peer memory (fused)"
                except Exception as exc:  # keep the collective path, say so in the line
                    exchange = f"nccl all-to-all (peer mapping failed: {exc})"
        if W["train"]:
            layer.set_training(True)
        w1 = torch.empty((e_local, D, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5)
        w3 = torch.empty((e_local, D, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5) \
            if gated else None
        w2 = torch.empty((e_local, F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(F ** -0.5)
        layer.load_experts(w1, w2, w3)
        del w1, w2, w3
        sh = W.get("shared")
        if sh:  # shared experts: dense FFN on every token at its source (+ Qwen's sigmoid gate)
            ns, fs, with_gate = sh
            s1 = torch.empty((ns, D, fs), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5)
            s3 = torch.empty_like(s1).uniform_(-1, 1).mul_(D ** -0.5) if gated else None
            s2 = torch.empty((ns, fs, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_((ns * fs) ** -0.5)
            sg = torch.empty(D, dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5) if with_gate else None
            layer.load_shared_experts(s1, s2, s3, sg)
            del s1, s2, s3, sg
        if args.micro_batches > 1 and not W["train"]:  # two micro-batches: exchange of one overlaps GEMMs of the other
            layer.set_micro_batches(args.micro_batches)
        return layer, exchange

    layer, exchange = build_layer(world > 1 and args.exchange == "peer")
    torch.cuda.empty_cache()
    gate = torch.empty((E, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(3.0 / D ** 0.5)
    x = torch.empty((n_local, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    out = torch.empty_like(x)
    layer.set_validate(False)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    upstream = torch.empty_like(x).uniform_(-1, 1) if W["train"] else None

    def step():
        layer.forward_expert_parallel(x, gate, prune=prune, out=out)
        if W["train"]:
            layer.backward(upstream)

    ok, fail_note = True, "on another rank"
    try:  # world > 1: a peer mapping that does not deliver (arrival timeout) falls back to NCCL on every rank
        step()
        torch.cuda.synchronize()
    except Exception as exc:  # noqa: BLE001
        ok, fail_note = False, str(exc)
    if world > 1:
        import torch.distributed as dist
        flag = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok = bool(flag.item())
    if not ok:
        if world == 1 or args.exchange != "peer":
            raise RuntimeError(f"first step failed: {fail_note}")
        del layer
        torch.cuda.empty_cache()
        layer, exchange = build_layer(False)
        exchange += " (peer-memory exchange failed its first step; fell back)"
        layer.set_validate(False)
    for _ in range(args.warmup):
        flush.zero_()
        step()
    barrier()
    # one step captured as a CUDA graph, replayed per step: world_size 1, and
    # world_size > 1 with the fused peer-memory exchange (counts, arrivals and
    # the received-row count all stay on the device: no host synchronisation)
    graph, per_step = None, None
    capturable = world == 1 or (exchange.startswith("peer memory") and not W["train"])
    if capturable and not args.no_graph:
        s_cap = torch.cuda.Stream()
        s_cap.wait_stream(stream)
        with torch.cuda.stream(s_cap):
            step()
        stream.wait_stream(s_cap)
        graph = torch.cuda.CUDAGraph()
        c0 = occ.launch_count()
        with torch.cuda.graph(graph):
            step()
        per_step = occ.launch_count() - c0
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
    run_step = graph.replay if graph is not None else step
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    l0 = occ.launch_count()
    barrier()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        run_step()
        ev[i][1].record(stream)
    barrier()
    launches = occ.launch_count() - l0 if graph is None else per_step * args.steps
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = args.tokens * args.steps / (tot_ms / 1e3)

    # --- end to end through the public API with host buffers -------------
    xh = torch.empty_like(x, device="cpu").pin_memory()
    xh.copy_(x)
    oh = torch.empty_like(xh).pin_memory()
    uh = upstream.cpu().pin_memory() if W["train"] else None
    # mixed-precision training: the token gradient leaves the device in bf16
    gxh = torch.empty((x.shape[0], D), dtype=torch.bfloat16).pin_memory() if W["train"] else None

    def e2e_step():
        if W["train"]:  # H2D tokens + upstream, forward + backward, D2H token gradient (double-buffered)
            layer.train_step_host(xh, gate, uh, gxh, prune=prune, wait=False)
            return
        # public API, host buffers: this step's H2D copy and the previous
        # step's D2H copy overlap the layer (double-buffered staging)
        layer.forward_host(xh, gate, oh, prune=prune, chunks=args.e2e_chunks, wait=False)

    for _ in range(3):
        e2e_step()
    layer.host_wait()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    # L2 between e2e steps: flushed unless one step's working set (resident
    # experts + tokens in + tokens out) is already > 2x the 126 MB L2
    ws_bytes = (e_local * D * F * (3 if gated else 2) + 2 * x.numel()) * 2
    e2e_flush = args.e2e_flush or ws_bytes < 2 * 126 * 2 ** 20
    for i in range(args.steps):
        if e2e_flush:
            flush.zero_()
        e2e_step()
    layer.host_wait()  # the last step's result has landed in host memory
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": args.tokens * args.steps / (e2e_ms / 1e3), "unit": "tokens/s",
           "h2d_bytes_per_step": x.numel() * x.element_size() * (2 if W["train"] else 1),
           "d2h_bytes_per_step": out.numel() * out.element_size(),
           "ms_per_step": e2e_ms / args.steps,
           "l2": ("flushed between steps" if e2e_flush else
                  f"not flushed: per-step working set {ws_bytes / 2 ** 30:.2f} GiB > 2x L2"),
           "api": (f"ExpertParallelLayer.train_step_host (pinned host tokens + upstream in, bf16 token gradient "
                   f"out; double-buffered so the copies of steps i+1 / i-1 overlap step i)" if W["train"] else
                   f"ExpertParallelLayer.forward_host (occ_forward_host: pinned host buffers, double-buffered so "
                   f"H2D of step i+1 and D2H of step i-1 overlap the layer of step i; {args.e2e_chunks} chunk(s))")
           + "; timed from before the first H2D to after the last D2H"}

    # --- stage profile (CUDA events on the launching stream) --------------
    layer.set_profiling(True)
    acc = {}
    for i in range(args.steps):
        flush.zero_()
        step()
        for kk, v in layer.stage_ms().items():
            acc.setdefault(kk, []).append(v)
    layer.set_profiling(False)
    stages = {kk: statistics.mean(v) for kk, v in acc.items()}
    rep = layer.comm_report(bytes_per_scalar=2)
    n_epd = rep.n_epd
    flops1 = 2.0 * n_epd * D * ((2 if gated else 1) * F)
    flops2 = 2.0 * n_epd * F * D
    train_flops = 2.0 * (flops1 + flops2) if W["train"] else 0.0
    shared_flops = 0.0
    if W.get("shared"):
        ns, fs, _ = W["shared"]
        shared_flops = 2.0 * args.tokens * D * ns * fs * (3 if gated else 2)
    tflops1 = flops1 / (stages["gemm1"] / 1e3) / 1e12
    tflops2 = flops2 / (stages["gemm2"] / 1e3) / 1e12
    # burst peak (cuBLAS timed alone): our timed loop is ~0.1 s, far shorter than
    # the 4 s sustained measurement, so burst is the conservative denominator
    peak = peaks.get("bf16_tflops")
    peak_sus = peaks.get("bf16_tflops_sustained", peak)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm1_traffic.json")
    if os.path.exists(tpath) and args.workload == "mixtral":
        with open(tpath) as f:
            traffic = json.load(f).get("bytes_per_launch")
    roofline = {"kernel": "wide_gemm_kernel<SWIGLU> (GEMM-1: x @ [w1|w3], 256x512 super-tiles, silu*up*gate-weight epilogue)",
                "bound": "tensor", "achieved": tflops1, "peak": peak, "unit": "TFLOP/s", "frac": tflops1 / peak,
                "peak_source": f"{peaks_src} bf16_tflops (burst)", "frac_of_sustained": tflops1 / peak_sus,
                "traffic": traffic,
                "flops_per_launch": flops1, "launch_ms": stages["gemm1"],
                "gemm2": {"achieved": tflops2, "frac": tflops2 / peak, "launch_ms": stages["gemm2"]},
                "layer_frac": (flops1 + flops2 + shared_flops) / (sum(stages.values()) / 1e3) / 1e12 / peak}
    if shared_flops:
        roofline["shared_tflops"] = shared_flops / (stages["shared"] / 1e3) / 1e12
    if W["train"]:
        roofline["step_tflops_fwd_bwd"] = (flops1 + flops2 + train_flops) / (tot_ms / args.steps / 1e3) / 1e12

    # --- the non-dedup GPU baseline of the north star: the same layer with the
    # replicate-k dispatch (one Sfd row per (token, expert)), same steps, same
    # exchange, timed the same way; speedup = its step time / ours ------------
    non_dedup = None
    if not W["train"] and not args.no_baseline_layer:
        nlayer, _ = build_layer(world > 1 and exchange.startswith("peer"), dedup=False)
        nlayer.set_validate(False)
        nout = torch.empty_like(out)

        def nstep():
            nlayer.forward_expert_parallel(x, gate, prune=prune, out=nout)

        for _ in range(args.warmup):
            flush.zero_()
            nstep()
        barrier()
        nrun = nstep
        if world == 1 and not args.no_graph:
            s2 = torch.cuda.Stream()
            s2.wait_stream(stream)
            with torch.cuda.stream(s2):
                nstep()
            stream.wait_stream(s2)
            ngraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(ngraph):
                nstep()
            nrun = ngraph.replay
        nev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        for i in range(args.steps):
            flush.zero_()
            nev[i][0].record(stream)
            nrun()
            nev[i][1].record(stream)
        barrier()
        n_ms = sum(a.elapsed_time(b) for a, b in nev)
        if world > 1:
            t = torch.tensor([n_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            n_ms = float(t.item())
        nrep = nlayer.comm_report(bytes_per_scalar=2)
        non_dedup = {"what": "same layer, replicate-k dispatch (one row per (token, expert): the non-dedup GPU "
                             "baseline of the north star), same exchange and timing",
                     "ms_per_step": n_ms / args.steps, "speedup": n_ms / tot_ms,
                     "crossing_rows_per_step": nrep.crossing_rows, "dedup_crossing_rows_per_step": rep.crossing_rows}
        del nlayer, nout
        torch.cuda.empty_cache()

    # --- all-to-all bytes/token: dedup vs naive top-k at the config's EP ------
    def a2a_at(ep, placement=None):
        e_pad = -(-E // ep) * ep  # Qwen's 60 experts at EP=8: 4 never-routed padding experts
        plan = occ.ExpertParallelLayer(occ.MoEConfig(e_pad, K_TOP, ep, D, F, activation=W["act"]), placement)
        if e_pad == E:
            ids_, _ = plan.route(x, gate, prune=prune)
        else:
            base = occ.ExpertParallelLayer(occ.MoEConfig(E, K_TOP, 1, D, F, activation=W["act"]))
            ids_, w_, sc = base.route(x, gate, want_scores=True)
            if prune is not None:
                sc = torch.cat([sc.double(), torch.zeros((sc.shape[0], e_pad - E), dtype=torch.float64,
                                                         device=sc.device)], 1)
                ids_, _ = plan.prune_routing(sc, ids_, w_.double(), prune)
        plan.build_dispatch_index(ids_)
        r = plan.comm_report(bytes_per_scalar=2)
        meta = 8 * K_TOP  # every dispatched row also carries its k ids (int32) + k weights (f32)
        return ids_, {"ep": ep, "payload": "bf16", "dedup_bytes_per_token": r.crossing_rows * D * 2 / n_local,
                      "naive_bytes_per_token": r.naive_crossing_rows * D * 2 / n_local,
                      "dedup_bytes_per_token_with_metadata": r.crossing_rows * (D * 2 + meta) / n_local,
                      "naive_bytes_per_token_with_metadata": r.naive_crossing_rows * (D * 2 + meta) / n_local,
                      "ratio": (r.crossing_rows / r.naive_crossing_rows) if r.naive_crossing_rows else None,
                      "mean_replicas": r.mean_replicas, "intra_share": r.intra_share}
    ep = W["plan_ep"]
    ids8, a2a = a2a_at(ep)
    a2a.update({"pruning": W["prune"],
                "note": ("Mixtral at EP=8 hosts one expert per GPU: dedup == naive" if E == 8 and ep == 8 else
                         "round-robin sources over the EP ranks; naive = one row per (token, expert)")})
    if W.get("coactivation_placement"):  # config 3: Occult co-activation placement
        pl = occ.collaboration_aware_placement([ids8], E, ep)
        _, a2a["coactivation_placement"] = a2a_at(ep, pl)
    for ep_x in W.get("extra_eps", ()):  # config 5: EP = 2 / 4 / 8
        a2a.setdefault("by_ep", {})[ep_x] = a2a_at(ep_x)[1]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "mixtral":
        try:
            cpu = cpu_port_baseline(args.cpu_seconds)
        except Exception as exc:  # report, never fake
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (uniform tokens, random-init experts and gate of the named layer shape)",
                "config": {"workload": WORKLOAD, "experts": E, "top_k": K_TOP, "d_model": D, "d_ff": F,
                           "ffn": "SwiGLU" if gated else W["act"], "tokens_per_step": args.tokens, "ep": world,
                           "ep_simulated_on_one_gpu": nd if world == 1 else None, "exchange": exchange,
                           "micro_batches": args.micro_batches if not W["train"] else 1,
                           "l2": "flushed between steps (512 MiB write)",
                           "step": ("route + plan + pack + grouped GEMM-1/2 + partial combine + combine"
                                    + (" + backward (dgrad x2, wgrad x2, routing-weight grads)" if W["train"]
                                       else ""))},
                "e2e": e2e, "gpu_launches": launches, "cuda_graph": graph is not None, "clocks": clk,
                "roofline": roofline,
                "stages_ms": stages, "a2a": a2a, "non_dedup_baseline": non_dedup, "cpu_baseline": cpu,
                "comm_report": {"mean_replicas": rep.mean_replicas, "n_sfd": rep.n_sfd, "n_epd": rep.n_epd}}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="mixtral", choices=sorted(WORKLOADS))
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of the captured CUDA graph")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"], help="world > 1 token exchange")
    ap.add_argument("--micro-batches", type=int, default=1, choices=[1, 2],
                    help="run each forward as two micro-batches on two streams (overlap of exchange and GEMMs)")
    ap.add_argument("--no-baseline-layer", action="store_true",
                    help="skip timing the replicate-k (non-dedup) layer next to ours")
    ap.add_argument("--e2e-chunks", type=int, default=1)
    ap.add_argument("--e2e-flush", action="store_true", help="flush L2 between e2e steps even for large layers")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-tokens-per-thread", type=int, default=2)
    args = ap.parse_args()
    select_workload(args.workload)
    if args.tokens is None:
        args.tokens = TOKENS
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
