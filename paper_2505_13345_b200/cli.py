"""`moesim`-compatible command line over the B200 layer (SURVEY.md 8(f) rows
3-4): the reference CLI's trace / profiling / placement / simulation commands
(cli.cpp:446-567) with the same options, output files, stdout lines and exit
codes, the data path running on the GPU.

    python -m paper_2505_13345_b200.cli gen-trace --experts 64 --topk 8 --tokens 65536 --dist blocks --blocks 8 --seed 1 --out t.trace
    python -m paper_2505_13345_b200.cli profile --trace t.trace --out-prefix t
    python -m paper_2505_13345_b200.cli reschedule --graph t.collab.mat --devices 8 --out t.place
    python -m paper_2505_13345_b200.cli simulate --seed 1 --trace t.trace --devices 8 --placement t.place --out r.txt

What runs where: trace generation and placement are host code in libocc
(std::mt19937_64, Alg. 1); the co-activation histogram, component-growth
edges, fp64 router, top-k, pruning and the expert-parallel forward are CUDA
kernels.  Files written are byte-identical to the reference CLI's on the same
inputs (tests/test_cli.py, tests/test_gpu_parity.py).  The simulate data path
is bf16 storage with fp32 accumulation whatever `--precision` says: the
precision only rounds the synthetic inputs (and therefore routing), as in the
reference; `--check-oracle` reports the GPU output's max relative error
against a dense fp64 evaluation of the same routing.  `fit-latency` (the
least-squares fit of measured latency on replicas, host arithmetic) completes
the command set.
"""
from __future__ import annotations

import argparse
import sys
from typing import List, Optional

import numpy as np

from . import api
from . import formats as F
from .report import format_double, render_simulate_report

EXIT = ((api.UsageError, 2, "usage error"), (api.ConfigError, 2, "usage error"), (api.DataError, 3, "data error"),
        (api.CapacityError, 4, "capacity error"), (api.PlacementError, 4, "placement error"))


def _slurp(path: str) -> str:
    """slurp_file (io.cpp:215-221)."""
    try:
        with open(path, "rb") as f:
            return f.read().decode("latin-1")
    except OSError:
        raise api.DataError(f"cannot open '{path}'") from None


def _write(path: str, text: str):
    """write_file (io.cpp:223-227)."""
    try:
        with open(path, "wb") as f:
            f.write(text.encode("latin-1"))
    except OSError:
        raise api.DataError(f"cannot write '{path}'") from None


# ------------------------------------------------------------- gen-trace --
def cmd_gen_trace(o) -> int:
    """cli.cpp:92-110."""
    if o.dist not in F.DISTS:
        raise api.UsageError(f"unknown distribution '{o.dist}'")
    spec = F.TraceSpec(o.dist, o.experts, o.topk, o.tokens, o.alpha, o.blocks, o.p_in, o.tag)
    _write(o.out, F.write_trace(F.gen_trace(spec, o.seed)))
    return 0


# --------------------------------------------------------------- profile --
def cmd_profile(o, out) -> int:
    """cli.cpp:112-171: co-activation counts + normalised graph + component
    growth over 256-token batches, histogram and growth edges on the GPU."""
    import torch
    trace = F.read_trace(_slurp(o.trace))
    ne = trace.num_experts
    dev = torch.device("cuda", torch.cuda.current_device())
    ids = torch.from_numpy(np.ascontiguousarray(trace.ids)).to(dev)
    counts = api.build_collab_graph(ids, ne).cpu().numpy()
    norm = api.normalize_graph(counts)
    growth = api.component_growth(ids, ne, 256)
    _write(o.out_prefix + ".collab.mat", F.write_matrix(counts.astype(np.float64)))
    _write(o.out_prefix + ".norm.mat", F.write_matrix(norm))
    upper = counts[np.triu_indices(ne, 1)]
    edges, coact = int(np.count_nonzero(upper > 0)), int(upper.sum())
    from .report import ReportWriter
    w = ReportWriter()
    w.kv("command", "profile")
    w.kv("trace.experts", ne)
    w.kv("trace.topk", trace.top_k)
    w.kv("trace.tokens", trace.num_tokens)
    if trace.tag:
        w.kv("trace.tag", trace.tag)
    w.kv("graph.edges", edges)
    w.kv("graph.coactivations", coact)
    w.kv("graph.max_component", growth[-1][1])
    for tokens, size in growth:
        w.kv(f"growth.{tokens}", size)
    _write(o.out_prefix + ".profile.txt", w.text())
    out.write(f"profile: {trace.num_tokens} tokens, {edges} edges, max component {growth[-1][1]}\n")
    return 0


# ------------------------------------------------------------ reschedule --
def norm_graph_from_matrix(m: np.ndarray) -> np.ndarray:
    """cli.cpp:62-80: validate a symmetric non-negative zero-diagonal graph and
    scale it by its maximum (raw counts or an already-normalised graph)."""
    rows, cols = m.shape
    if rows != cols:
        raise api.DataError("graph: matrix must be square")
    for i in range(rows):  # the reference's scan order decides which error is reported
        for j in range(cols):
            if m[i, j] < 0.0:
                raise api.DataError("graph: negative edge value")
            if m[i, j] != m[j, i]:
                raise api.DataError("graph: matrix must be symmetric")
            if i == j and m[i, j] != 0.0:
                raise api.DataError("graph: diagonal must be zero")
    mx = float(m.max()) if m.size else 0.0
    return np.zeros_like(m) if mx == 0.0 else m / mx


def cmd_reschedule(o) -> int:
    """cli.cpp:173-188."""
    m = F.read_matrix(_slurp(o.graph))
    if o.devices < 1 or m.shape[0] % max(o.devices, 1):
        raise api.UsageError(f"reschedule: expert count {m.shape[0]} is not divisible by --devices {o.devices}")
    placement = api.reschedule_placement(norm_graph_from_matrix(m), o.devices)
    _write(o.out, F.write_placement(placement))
    return 0


# -------------------------------------------------------------- simulate --
def _validate_config(ne, nd, k, dim, hidden):
    """MoEConfig::validate (core.cpp:10-23), raised as UsageError (cli.cpp:235-238)."""
    if ne < 1:
        raise api.UsageError("config: num_experts must be >= 1")
    if nd < 1:
        raise api.UsageError("config: num_devices must be >= 1")
    if k < 1 or k > ne:
        raise api.UsageError(f"config: top_k must satisfy 1 <= k <= num_experts (k={k}, experts={ne})")
    if ne % nd:
        raise api.UsageError(f"config: num_experts ({ne}) must be divisible by num_devices ({nd})")
    if dim < 1 or hidden < 1:
        raise api.UsageError("config: dims must be >= 1")


def _similarity_from_matrix(tm: np.ndarray, ne: int):
    if tm.shape != (ne, ne):
        raise api.DataError("similarity table shape mismatch")
    return np.ascontiguousarray(tm, dtype=np.float64)


def run_simulate(o):
    """cli.cpp:201-320 on the GPU. Returns (config, placement, ids, CommReport,
    baseline_k, oracle error or None)."""
    import torch
    if o.precision not in ("single", "double"):
        raise api.UsageError(f"unknown precision '{o.precision}'")
    if o.activation not in ("identity", "silu", "relu"):
        raise api.UsageError(f"unknown activation '{o.activation}'")
    if o.prune not in api.PRUNE:
        raise api.UsageError(f"unknown prune mode '{o.prune}'")
    if o.weight_policy not in ("inherit", "own"):
        raise api.UsageError(f"unknown weight policy '{o.weight_policy}'")
    trace = None
    if o.trace:
        if o.prune != "none":
            raise api.UsageError("pruning needs gate scores; drop --trace to simulate from a seed")
        trace = F.read_trace(_slurp(o.trace))
        ne, k = trace.num_experts, trace.top_k
    else:
        ne, k = o.experts, o.topk
    _validate_config(ne, o.devices, k, o.dim, o.hidden)
    if min(o.tile_m, o.tile_k, o.tile_n) < 1:
        raise api.UsageError("config: tile sizes must be >= 1")
    if o.placement:
        placement = F.read_placement(_slurp(o.placement))
        F.validate_placement(placement.devices, ne)
    else:
        placement = api.trivial_placement(ne, o.devices)
    single = o.precision == "single"
    master = F.Rng(o.seed)  # cli.cpp:248-251: token, gate, expert streams in that order
    token_rng, gate_rng, expert_rng = F.Rng(master.next()), F.Rng(master.next()), F.Rng(master.next())
    n = trace.num_tokens if trace is not None else o.tokens
    x = token_rng.random_matrix(n, o.dim, single)
    w1 = np.empty((ne, o.dim, o.hidden))
    w2 = np.empty((ne, o.hidden, o.dim))
    for e in range(ne):  # ExpertWeights::random (core.cpp:40-52): w1 then w2 per expert
        w1[e] = expert_rng.random_matrix(o.dim, o.hidden, single)
        w2[e] = expert_rng.random_matrix(o.hidden, o.dim, single)
    if o.source_mode == "single":
        sources_np = np.zeros(n, np.int32)
    elif o.source_mode == "roundrobin":
        sources_np = (np.arange(n) % o.devices).astype(np.int32)
    else:
        raise api.UsageError(f"unknown source mode '{o.source_mode}'")

    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = api.MoEConfig(ne, k, o.devices, o.dim, o.hidden, renormalize=o.renormalize, activation=o.activation)
    layer = api.ExpertParallelLayer(cfg, placement)
    layer.load_experts(torch.from_numpy(w1).to(dev, torch.bfloat16), torch.from_numpy(w2).to(dev, torch.bfloat16))
    xd = torch.from_numpy(x).to(dev)
    sources = torch.from_numpy(sources_np).to(dev)
    cap = None
    if trace is not None:
        ids = torch.from_numpy(np.ascontiguousarray(trace.ids)).to(dev)
        w = torch.from_numpy(np.ascontiguousarray(trace.weights)).to(dev)
    else:
        gate = torch.from_numpy(gate_rng.random_matrix(ne, o.dim, single)).to(dev)
        scores = api.gate_scores_f64(xd, gate)
        ids, w = api.topk_route(scores, k, o.renormalize)
        prune = api.PruneSpec(o.prune, o.budget, None, o.weight_policy)
        if o.prune == "similarity":
            if o.table:
                prune.table = _similarity_from_matrix(F.read_matrix(_slurp(o.table)), ne)
            else:  # profile the batch's own router logits (cli.cpp:296-299)
                prune.table = api.build_similarity_table([api.gate_logits_f64(xd, gate)], ne)
        if prune.table is not None and o.dump_table:
            _write(o.dump_table, F.write_matrix(np.asarray(prune.table).reshape(ne, ne)))
        if o.prune != "none":
            if o.budget < 1 or o.budget > o.devices:  # prune_routing's check (pruning.cpp:13-15)
                raise api.ConfigError("prune: device budget must be in [1, num_devices]")
            ids, w = layer.prune_routing(scores, ids, w, prune)
            cap = float(min(k, o.devices, o.budget))
    layer.forward_given_routing(xd.to(torch.bfloat16), ids, w.float(), sources=sources)
    rep = layer.comm_report(bytes_per_scalar=o.bytes_per_scalar, cap_replicas=cap)
    baseline_k = float(k) if n else 0.0  # baseline_replication_ct ReplicateK (simnet.cpp:26-34)
    err = None
    if o.check_oracle:
        err = _dense_check(layer, xd, ids, w, w1, w2, o.activation)
    return cfg, placement, ids, rep, baseline_k, err, n


def _dense_check(layer, xd, ids, w, w1, w2, act):
    """max_rel_error (matrix.cpp:52-62) of the GPU output against a dense fp64
    evaluation of the same routing (dense_given_routing, pipeline.cpp)."""
    import torch
    out = layer.forward_given_routing(xd.to(torch.bfloat16), ids, w.float()).double()
    dev = xd.device
    w1d, w2d = torch.from_numpy(w1).to(dev), torch.from_numpy(w2).to(dev)
    ref = torch.zeros_like(xd)
    ids_l = ids.long()
    for j in range(ids.shape[1]):
        h = torch.einsum("nd,ndh->nh", xd, w1d[ids_l[:, j]])
        h = torch.nn.functional.silu(h) if act == "silu" else torch.relu(h) if act == "relu" else h
        ref += w[:, j:j + 1].double() * torch.einsum("nh,nhd->nd", h, w2d[ids_l[:, j]])
    diff = float((out - ref).abs().max()) if ref.numel() else 0.0
    scale = float(ref.abs().max()) if ref.numel() else 0.0
    return diff / scale if scale > 0.0 else diff


def write_simulate_report(o, result):
    cfg, placement, ids, rep, _baseline_k, err, n = result
    counts = api.build_collab_graph(ids, cfg.num_experts).cpu().numpy()
    text = render_simulate_report(
        # config.seed is printed as static_cast<long long> of the uint64 seed (cli.cpp:337)
        cfg, rep, counts, placement.devices, n, seed=o.seed - (1 << 64) if o.seed >= 1 << 63 else o.seed,
        precision=o.precision, activation=o.activation,
        prune_mode=o.prune, prune_budget=o.budget, trace=o.trace or "-", placement_name=o.placement or "trivial",
        bytes_per_scalar=o.bytes_per_scalar, oracle_max_rel_error=err)
    _write(o.out, text)


def cmd_simulate(o, out) -> int:
    """cli.cpp:380-391."""
    result = run_simulate(o)
    write_simulate_report(o, result)
    rep = result[3]
    out.write(f"simulate: mean replicas {format_double(rep.mean_replicas)} (cap {format_double(rep.cap_replicas)}), "
              f"cross-device bytes {int(rep.cross_device_bytes)}\n")
    if result[5] is not None:
        out.write(f"oracle max relative error: {format_double(result[5])}\n")
    return 0


def cmd_sweep_prune(o, out) -> int:
    """cli.cpp:422-441: one simulate report per feasible device budget."""
    if o.mode == "none":
        raise api.UsageError("sweep-prune: --mode must be router or similarity")
    o.prune = o.mode
    o.trace = ""
    per = o.experts // max(o.devices, 1)
    d_min = max(1, (o.topk + per - 1) // per) if per else 1
    for d in range(1, d_min):
        out.write(f"budget {d}: skipped ({d} device(s) host fewer than k={o.topk} experts)\n")
    for d in range(d_min, o.devices + 1):
        o.budget = d
        o.out = f"{o.out_prefix}.d{d}.txt"
        result = run_simulate(o)
        write_simulate_report(o, result)
        out.write(f"budget {d}: mean replicas {format_double(result[3].mean_replicas)} -> {o.out}\n")
    return 0


# ---------------------------------------------------------- fit-latency --
def fit_latency(points):
    """fit_latency (simnet.cpp:36-66): least squares of latency on replicas,
    the reference's summation order."""
    distinct = sum(1 for i, p in enumerate(points) if all(q[0] != p[0] for q in points[:i]))
    if len(points) < 2 or distinct < 2:
        raise api.UsageError("fit: need at least 2 points with distinct x values")
    n = float(len(points))
    mx = my = 0.0
    for px, py in points:
        mx += px
        my += py
    mx /= n
    my /= n
    sxx = sxy = syy = 0.0
    for px, py in points:
        sxx += (px - mx) * (px - mx)
        sxy += (px - mx) * (py - my)
        syy += (py - my) * (py - my)
    slope = sxy / sxx
    return slope, my - slope * mx, 1.0 if syy == 0.0 else (sxy * sxy) / (sxx * syy)


def cmd_fit_latency(o, out) -> int:
    """cli.cpp:393-422: `replicas seconds` per line ('#' comments), one report."""
    points = []
    for line_no, line in enumerate(F._lines(_slurp(o.points)), 1):
        if not line or line[0] == "#":
            continue
        parts = F._split_ws(line)
        if len(parts) != 2:
            raise api.DataError(f"line {line_no}: expected 'replicas seconds'")
        points.append((F.parse_double(parts[0], line_no), F.parse_double(parts[1], line_no)))
    slope, intercept, r2 = fit_latency(points)
    from .report import ReportWriter
    w = ReportWriter()
    w.kv("command", "fit-latency")
    w.kv("points.count", len(points))
    w.kv("fit.slope", slope)
    w.kv("fit.intercept", intercept)
    w.kv("fit.r_squared", r2)
    _write(o.out, w.text())
    out.write(f"fit: slope {format_double(slope)}, intercept {format_double(intercept)}, R^2 {format_double(r2)}\n")
    return 0


# ---------------------------------------------------------------- parser --
def _parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="moesim", description="Expert-parallel MoE communication simulator (B200)")
    sub = p.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen-trace", help="Generate a synthetic routing trace")
    g.add_argument("--dist", default="uniform")
    g.add_argument("--experts", type=int, required=True)
    g.add_argument("--topk", type=int, required=True)
    g.add_argument("--tokens", type=int, required=True)
    g.add_argument("--alpha", type=float, default=1.0)
    g.add_argument("--blocks", type=int, default=1)
    g.add_argument("--p-in", dest="p_in", type=float, default=0.9)
    g.add_argument("--tag", default="")
    g.add_argument("--seed", type=int, required=True)
    g.add_argument("--out", required=True)
    pr = sub.add_parser("profile", help="Build collaboration graphs from a trace")
    pr.add_argument("--trace", required=True)
    pr.add_argument("--out-prefix", dest="out_prefix", required=True)
    r = sub.add_parser("reschedule", help="Build an expert placement from a graph")
    r.add_argument("--graph", required=True)
    r.add_argument("--devices", type=int, required=True)
    r.add_argument("--out", required=True)

    def sim_common(s):
        s.add_argument("--seed", type=int, required=True)
        s.add_argument("--devices", type=int, default=1)
        s.add_argument("--experts", type=int, default=8)
        s.add_argument("--topk", type=int, default=2)
        s.add_argument("--tokens", type=int, default=64)
        s.add_argument("--dim", type=int, default=32)
        s.add_argument("--hidden", type=int, default=64)
        s.add_argument("--weight-policy", dest="weight_policy", default="inherit")
        s.add_argument("--precision", default="single")
        s.add_argument("--renormalize", dest="renormalize", action="store_true", default=True)
        s.add_argument("--no-renormalize", dest="renormalize", action="store_false")
        s.add_argument("--activation", default="identity")
        s.add_argument("--bytes-per-scalar", dest="bytes_per_scalar", type=int, default=4)
        for name, dv in (("--trace", ""), ("--placement", ""), ("--table", ""), ("--dump-table", ""),
                         ("--source-mode", "roundrobin")):
            s.add_argument(name, dest=name[2:].replace("-", "_"), default=dv)
        for name in ("--tile-m", "--tile-k", "--tile-n"):
            s.add_argument(name, dest=name[2:].replace("-", "_"), type=int, default=32)
        s.add_argument("--budget", type=int, default=1)
        s.add_argument("--check-oracle", dest="check_oracle", action="store_true")

    s = sub.add_parser("simulate", help="Run the expert-parallel pipeline")
    sim_common(s)
    s.add_argument("--prune", default="none")
    s.add_argument("--out", required=True)
    fl = sub.add_parser("fit-latency", help="Least-squares fit of latency vs replicas")
    fl.add_argument("--points", required=True)
    fl.add_argument("--out", required=True)
    w = sub.add_parser("sweep-prune", help="Prune-budget sweep, one report per budget")
    sim_common(w)
    w.add_argument("--mode", required=True)
    w.add_argument("--out-prefix", dest="out_prefix", required=True)
    return p


def run(argv: List[str], out=None, err=None) -> int:
    """cli::run (cli.cpp:446-567): parse, dispatch, map errors to exit codes."""
    out = out or sys.stdout
    err = err or sys.stderr
    try:
        o = _parser().parse_args(argv)
    except SystemExit as e:  # argparse: usage errors exit 2, --help exits 0
        return int(e.code or 0)
    try:
        if o.cmd == "gen-trace":
            return cmd_gen_trace(o)
        if o.cmd == "profile":
            return cmd_profile(o, out)
        if o.cmd == "reschedule":
            return cmd_reschedule(o)
        if o.cmd == "simulate":
            return cmd_simulate(o, out)
        if o.cmd == "sweep-prune":
            return cmd_sweep_prune(o, out)
        if o.cmd == "fit-latency":
            return cmd_fit_latency(o, out)
    except Exception as e:  # noqa: BLE001 — the reference's catch-all maps to exit 1
        for cls, code, label in EXIT:
            if isinstance(e, cls):
                err.write(f"{label}: {e}\n")
                return code
        err.write(f"error: {e}\n")
        return 1
    return 2


def main(argv: Optional[List[str]] = None) -> int:
    return run(sys.argv[1:] if argv is None else argv)


if __name__ == "__main__":
    sys.exit(main())
