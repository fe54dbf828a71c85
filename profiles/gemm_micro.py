"""Grouped-GEMM microbenchmark through the layer API: forward_given_routing
with BALANCED routing (token t -> experts (k*t + j) mod E, every expert gets
exactly n*k/E rows) vs the bench's random routing, so grouping/padding
effects on GEMM-1/GEMM-2 throughput can be separated.  Prints one JSON line
per case: stage ms and TFLOP/s (CUDA events)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13345_b200 as occ  # noqa: E402

CASES = {
    "deepseek": (64, 6, 2048, 1408, 16384),
    "deepseek_p": (64, 6, 2048, 1408, 16395),   # balanced -> 1537-1538 rows/expert: 7 m-tiles, last nearly empty
    "deepseek_m": (64, 6, 2048, 1408, 16373),   # balanced -> 1534-1535 rows/expert: 6 m-tiles, nearly full
    "olmoe": (64, 8, 2048, 1024, 65536),
    "mixtral": (8, 2, 4096, 14336, 16384),
    "dense_2816": (1, 1, 2048, 2816, 16384),
    "dense_1408_98k": (1, 1, 2048, 1408, 98304),
}


def run(name, E, k, D, F, n, routings, steps=10, reps=4):
    dev = torch.device("cuda", 0)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(E, k, 1, D, F, activation="swiglu"))
    w1 = torch.empty((E, D, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5)
    w3 = torch.empty_like(w1).uniform_(-1, 1).mul_(D ** -0.5)
    w2 = torch.empty((E, F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(F ** -0.5)
    layer.load_experts(w1, w2, w3)
    del w1, w2, w3
    x = torch.empty((n, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    t = torch.arange(n, device=dev)[:, None]
    rt = {"balanced": ((k * t + torch.arange(k, device=dev)[None, :]) % E).to(torch.int32),
          "random": torch.argsort(torch.rand(n, E, device=dev), dim=1)[:, :k].to(torch.int32)}
    perm = torch.randperm(n, device=dev)[:, None]
    rt["balanced_perm"] = ((k * perm + torch.arange(k, device=dev)[None, :]) % E).to(torch.int32)
    rt["balanced_rot"] = ((k * t + torch.arange(k, device=dev)[None, :] + 1) % E).to(torch.int32)
    w = torch.full((n, k), 1.0 / k, device=dev)
    layer.set_validate(False)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for r in routings:
        for _ in range(3):
            layer.forward_given_routing(x, rt[r], w)
    layer.set_profiling(True)
    acc = {r: {} for r in routings}
    for _ in range(reps):  # alternate so power/clock drift hits every routing alike
        for r in routings:
            for _ in range(steps):
                flush.zero_()
                layer.forward_given_routing(x, rt[r], w)
                for kk, v in layer.stage_ms().items():
                    acc[r].setdefault(kk, []).append(v)
    f1 = 2.0 * n * k * D * 2 * F
    f2 = 2.0 * n * k * F * D
    # same-box cuBLAS reference: one dense GEMM with the same FLOPs/shape (one weight matrix)
    cub = {}
    if os.environ.get("OCC_MICRO_CUBLAS", "1") == "1":
        a1 = torch.empty((n * k, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
        b1 = torch.empty((D, 2 * F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
        a2 = torch.empty((n * k, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
        b2 = torch.empty((F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
        for nm, (a, b, fl) in {"cublas1": (a1, b1, f1), "cublas2": (a2, b2, f2)}.items():
            ts = []
            for _ in range(reps * steps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                torch.matmul(a, b)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            cub[nm + "_tflops"] = round(fl / sorted(ts)[len(ts) // 2] / 1e9)
        del a1, b1, a2, b2
    for r in routings:
        med = {kk: sorted(v)[len(v) // 2] for kk, v in acc[r].items()}
        print(json.dumps({"case": name, "routing": r, "band": os.environ.get("OCC_GEMM_BAND"),
                          "gemm1_ms": med["gemm1"], "gemm2_ms": med["gemm2"],
                          "gemm1_tflops": f1 / med["gemm1"] / 1e9, "gemm2_tflops": f2 / med["gemm2"] / 1e9, **cub,
                          "other_ms": {kk: round(v, 4) for kk, v in med.items() if not kk.startswith("gemm")}}),
              flush=True)
    del layer
    torch.cuda.empty_cache()


if __name__ == "__main__":
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(CASES)
    routings = sys.argv[2].split(",") if len(sys.argv) > 2 else ["balanced", "random"]
    for nm in names:
        run(nm, *CASES[nm], routings)
