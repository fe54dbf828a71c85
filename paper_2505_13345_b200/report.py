"""`#moesim-report v1` key=value reports from a GPU run.

Mirrors the reference's report writer (io.cpp:206-213, ReportWriter) and the
`simulate` command's report body (cli.cpp:326-378) so a report produced from
the B200 layer diffs line-for-line against the reference CPU simulator's on
the integer fields, and on the double fields wherever the value itself is
bit-exact (E(C_T), shares, bounds, collaboration means from the bit-exact
co-activation histogram).  Doubles use std::to_chars' shortest round-trip
form (io.cpp:55-60).
"""
from __future__ import annotations

from decimal import Decimal
import math
from typing import Optional

import numpy as np

REPORT_HEADER = "#moesim-report v1"  # io.cpp:18


def format_double(v: float) -> str:
    """std::to_chars(double) (io.cpp:55-60): shortest round-trip digits, in the
    shorter of fixed and scientific notation (fixed on ties; an integral value
    in fixed notation prints its exact integer digits), exponent with a sign
    and at least two digits."""
    v = float(v)
    if not math.isfinite(v):
        from .api import DataError
        raise DataError("refusing to serialize non-finite value")
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    sign, digits, exp = Decimal(repr(v)).as_tuple()
    ds = "".join(map(str, digits)).rstrip("0") or "0"
    exp += len("".join(map(str, digits))) - len(ds)  # value = ds * 10^exp
    neg = "-" if sign else ""
    n = len(ds)
    point = n + exp  # position of the decimal point relative to ds
    if exp >= 0:  # integral: %f-style prints the exact integer value
        fixed = str(int(abs(v)))
    elif point > 0:
        fixed = ds[:point] + "." + ds[point:]
    else:
        fixed = "0." + "0" * (-point) + ds
    e10 = point - 1
    sci = ds[0] + ("." + ds[1:] if n > 1 else "") + "e" + ("-" if e10 < 0 else "+") + f"{abs(e10):02d}"
    return neg + (fixed if len(fixed) <= len(sci) else sci)


class ReportWriter:
    """io.cpp:206-213."""

    def __init__(self):
        self.lines = [REPORT_HEADER]

    def kv(self, key: str, value):
        if isinstance(value, (bool, np.bool_)):
            value = int(value)
        if isinstance(value, (float, np.floating)):
            s = format_double(value)
        else:
            s = str(value)
        self.lines.append(f"{key}={s}")

    def text(self) -> str:
        return "\n".join(self.lines) + "\n"


def replica_bounds(k: int, num_experts: int, num_devices: int):
    """collab.cpp:63-74."""
    lower = float((k * num_devices + num_experts - 1) // num_experts)
    upper = float(min(k, num_devices))
    return lower, upper


def intra_inter_metrics(p: np.ndarray, devices):
    """collab.cpp:76-103, same summation order."""
    nd = len(devices)
    intra = [0.0] * nd
    for d, ex in enumerate(devices):
        n = len(ex)
        if n < 2:
            continue
        s = 0.0
        for a in range(n):
            for b in range(n):
                if a != b:
                    s += float(p[ex[a], ex[b]])
        intra[d] = s / float(n * (n - 1))
    inter = {}
    for d1 in range(nd):
        for d2 in range(nd):
            if d1 == d2:
                continue
            s = 0.0
            for i in devices[d1]:
                for j in devices[d2]:
                    s += float(p[i, j])
            inter[(d1, d2)] = s / float(len(devices[d1]) * len(devices[d2]))
    return intra, inter


def simulate_report(layer, ids, **kw) -> str:
    """The `simulate` report (cli.cpp:326-378) for the layer's last forward
    over routing `ids` (device int32 [n, k]): CommReport from the device plan,
    collaboration means from the device co-activation histogram."""
    from . import api
    cfg = layer.config
    rep = layer.comm_report(bytes_per_scalar=kw.get("bytes_per_scalar", 4))
    counts = api.build_collab_graph(ids, cfg.num_experts).cpu().numpy()
    return render_simulate_report(cfg, rep, counts, layer.placement.devices, int(ids.shape[0]), **kw)


def render_simulate_report(cfg, rep, counts, devices, n, *, seed: int = 1, precision: str = "single",
                           activation: Optional[str] = None, prune_mode: str = "none",
                           prune_budget: Optional[int] = None, trace: str = "-", placement_name: str = "trivial",
                           bytes_per_scalar: int = 4, oracle_max_rel_error: Optional[float] = None) -> str:
    """Report body of write_simulate_report (cli.cpp:326-378) from a
    CommReport-like `rep` (mean_replicas, cap_replicas, intra_share,
    inter_share, cross_device_bytes, per_device_token_counts) and the int64
    co-activation counts."""
    from . import api
    w = ReportWriter()
    w.kv("command", "simulate")
    w.kv("config.devices", cfg.num_devices)
    w.kv("config.experts", cfg.num_experts)
    w.kv("config.topk", cfg.top_k)
    w.kv("config.tokens", n)
    w.kv("config.dim", cfg.embed_dim)
    w.kv("config.hidden", cfg.hidden_dim)
    w.kv("config.seed", seed)
    w.kv("config.precision", precision)
    w.kv("config.activation", activation or cfg.activation)
    w.kv("config.renormalize", 1 if cfg.renormalize else 0)
    w.kv("config.prune.mode", prune_mode)
    if prune_mode != "none":
        w.kv("config.prune.budget", prune_budget)
    w.kv("config.trace", trace)
    w.kv("config.placement", placement_name)
    lo, hi = replica_bounds(cfg.top_k, cfg.num_experts, cfg.num_devices)
    w.kv("replicas.mean", float(rep.mean_replicas))
    w.kv("replicas.cap", float(rep.cap_replicas))
    w.kv("replicas.lower_bound", lo)
    w.kv("replicas.upper_bound", hi)
    w.kv("replicas.baseline_k", float(cfg.top_k) if n else 0.0)  # simnet.cpp:26-34, ReplicateK
    w.kv("shares.intra", float(rep.intra_share))
    w.kv("shares.inter", float(rep.inter_share))
    w.kv("bytes.cross_device", int(rep.cross_device_bytes))
    w.kv("bytes.per_scalar", bytes_per_scalar)
    total = 0
    for d, c in enumerate(rep.per_device_token_counts):
        w.kv(f"device.{d}.received", int(c))
        total += int(c)
    w.kv("tokens.sfd_total", total)
    p = api.normalize_graph(counts)
    intra, inter = intra_inter_metrics(p, devices)
    for d in range(cfg.num_devices):
        w.kv(f"collab.intra.{d}", intra[d])
    for d1 in range(cfg.num_devices):
        for d2 in range(d1 + 1, cfg.num_devices):
            w.kv(f"collab.inter.{d1}.{d2}", inter[(d1, d2)])
    if oracle_max_rel_error is not None and oracle_max_rel_error >= 0.0:
        w.kv("oracle.max_rel_error", oracle_max_rel_error)
    return w.text()
