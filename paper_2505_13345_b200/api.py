"""Host-side mirror of the reference's C++ API (namespace ``moesim``) over the
C-ABI in ``include/occult.h`` (``libocc.so``, sm_100a).

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/moesim/*.hpp) so callers and parity tests read
like the reference's own; tensors are torch CUDA tensors (PyTorch provides
device memory and streams only — every op below runs in this package's CUDA
kernels).  There is no CPU fallback: importing on a machine without the
built library, or calling without a GPU, raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OCC_LIB_EXPERIMENT") or os.path.join(_HERE, "libocc.so")  # env: A/B builds (profiles/)

# ---------------------------------------------------------------- errors ---
# common.hpp:11-34 taxonomy; occ_status 1..6.


class MoesimError(RuntimeError):
    pass


class ShapeError(MoesimError):
    pass


class ConfigError(MoesimError):
    pass


class PlacementError(MoesimError):
    pass


class RoutingError(MoesimError):
    pass


class CapacityError(MoesimError):
    pass


class StateError(MoesimError):
    pass


class DataError(MoesimError):
    """common.hpp DataError: malformed input files (CLI exit code 3)."""


class UsageError(MoesimError):
    """common.hpp UsageError: bad command-line arguments (CLI exit code 2)."""


class DeviceError(MoesimError):
    """CUDA / NCCL failure or unsupported configuration on the B200 path."""


_STATUS = {1: ShapeError, 2: ConfigError, 3: PlacementError, 4: RoutingError, 5: CapacityError, 6: StateError}

ACT = {"identity": 0, "silu": 1, "relu": 2, "swiglu": 3}
PRUNE = {"none": 0, "router": 1, "similarity": 2}


class _Config(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("num_experts", "top_k", "num_devices", "embed_dim", "hidden_dim",
                                       "renormalize", "activation", "dedup")]


class _Prune(C.Structure):
    _fields_ = [("mode", C.c_int), ("device_budget", C.c_int), ("own_score", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("mean_replicas", C.c_double), ("cap_replicas", C.c_double), ("intra_share", C.c_double),
                ("inter_share", C.c_double), ("cross_device_bytes", C.c_longlong), ("crossing_rows", C.c_longlong),
                ("naive_crossing_rows", C.c_longlong), ("n_sfd", C.c_longlong), ("n_epd", C.c_longlong),
                ("per_device_rows", C.c_longlong * 64)]


EXPORTS = (
    "occ_create", "occ_destroy", "occ_set_placement", "occ_load_experts", "occ_set_similarity", "occ_set_validate",
    "occ_comm_unique_id", "occ_comm_init", "occ_gate_scores_f64", "occ_topk_route_f64", "occ_prune_routing_f64",
    "occ_route", "occ_build_dispatch", "occ_forward", "occ_forward_expert_parallel", "occ_comm_report_get",
    "occ_saved_index", "occ_coactivation_histogram", "occ_normalize_graph", "occ_reschedule_placement",
    "occ_allreduce_histogram", "occ_last_error", "occ_launch_count", "occ_set_profiling", "occ_stage_ms", "occ_forward_host", "occ_host_wait", "occ_comm_init_loopback", "occ_exchange_layout", "occ_set_training", "occ_backward",
    "occ_load_shared_experts", "occ_comm_enable_peer", "occ_similarity_accumulate", "occ_similarity_finalize",
    "occ_router_logits", "occ_set_grad_x_bf16", "occ_gate_logits_f64", "occ_set_micro_batches", "occ_set_router_mode", "occ_route_exact",
    "occ_dispatch", "occ_build_compute", "occ_expert_compute", "occ_combine", "occ_comm_init_host",
    "occ_set_plan_kernels",
)

STAGES = ("route", "plan", "pack", "compute_index", "gather", "gemm1", "gemm2", "shared", "partial_combine", "combine")

_LIB = None
_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


def lib():
    """Load libocc.so (built in-tree by ``__graft_entry__.build()``). Fails loudly."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.occ_last_error.restype = C.c_char_p
        L.occ_launch_count.restype = C.c_longlong
        _LIB = L
    return _LIB


def _check(rc, what=""):
    if rc != 0:
        msg = lib().occ_last_error().decode(errors="replace")
        raise _STATUS.get(rc, DeviceError)(f"{what}: {msg} (status {rc})")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise DeviceError("B200 path: tensors must live on the GPU (no CPU fallback)")


def _arg(t: Optional[torch.Tensor], name: str, dtype: torch.dtype, shape: tuple):
    """Validate a tensor handed to the C-ABI (which takes raw pointers): the
    dtype and shape must match exactly (a wrong dtype would be reinterpreted,
    not converted), and the result is contiguous.  The caller keeps the
    returned tensor alive until the call returns.  None passes through."""
    if t is None:
        return None
    if t.dtype != dtype:
        raise ShapeError(f"{name}: expected {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ShapeError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t.contiguous()


def launch_count() -> int:
    return int(lib().occ_launch_count())

# ------------------------------------------------------------ config types --


@dataclass
class MoEConfig:
    """config.hpp:12-28 (``tiles``/``seed``/``precision`` have no GPU meaning:
    the device path is bf16 storage with fp32 accumulation)."""

    num_experts: int
    top_k: int
    num_devices: int = 1
    embed_dim: int = 0
    hidden_dim: int = 0
    renormalize: bool = True
    activation: str = "identity"
    dedup: bool = True

    def experts_per_device(self) -> int:
        return self.num_experts // self.num_devices

    def _c(self):
        return _Config(self.num_experts, self.top_k, self.num_devices, self.embed_dim, self.hidden_dim,
                       int(self.renormalize), ACT[self.activation], int(self.dedup))


@dataclass
class Placement:
    """placement.hpp:14-25: per-device expert lists, list order significant."""

    devices: list

    def num_devices(self) -> int:
        return len(self.devices)

    def num_experts(self) -> int:
        return sum(len(d) for d in self.devices)

    def expert_to_device(self):
        n = self.num_experts()
        dev = [-1] * n
        for d, lst in enumerate(self.devices):
            for e in lst:
                if e < 0 or e >= n or dev[e] >= 0:
                    raise PlacementError(f"placement: device lists are not a partition of [0, {n})")
                dev[e] = d
        return dev

    def flat(self):
        return [e for d in self.devices for e in d]


def trivial_placement(num_experts: int, num_devices: int) -> Placement:
    """placement.cpp:47-58."""
    if num_devices < 1 or num_experts < 1 or num_experts % num_devices:
        raise ConfigError("trivial_placement: num_experts must be a positive multiple of num_devices")
    per = num_experts // num_devices
    return Placement([list(range(d * per, (d + 1) * per)) for d in range(num_devices)])


@dataclass
class PruneSpec:
    """pruning.hpp:32-39 (the similarity table is given as its E x E values)."""

    mode: str = "none"
    device_budget: int = 1
    table: Optional[Sequence[float]] = None
    weight_policy: str = "inherit"

    def _c(self):
        return _Prune(PRUNE[self.mode], self.device_budget, int(self.weight_policy == "own"))


@dataclass
class CommReport:
    """collab.hpp:36-43 + naive top-k comparison."""

    mean_replicas: float = 0.0
    cap_replicas: float = 0.0
    intra_share: float = 0.0
    inter_share: float = 0.0
    cross_device_bytes: int = 0
    crossing_rows: int = 0
    naive_crossing_rows: int = 0
    n_sfd: int = 0
    n_epd: int = 0
    per_device_token_counts: list = field(default_factory=list)


# -------------------------------------------------------------- the layer ---


class ExpertParallelLayer:
    """One handle of the C-ABI: router config + placement table + resident
    experts (+ optional similarity table), the drop-in for
    forward_given_routing / forward_expert_parallel (pipeline.hpp:178-189)."""

    def __init__(self, config: MoEConfig, placement: Optional[Placement] = None, world_size: int = 1, rank: int = 0):
        self.config = config
        self.placement = placement or trivial_placement(config.num_experts, config.num_devices)
        if self.placement.num_devices() != config.num_devices:
            raise ConfigError("placement device count disagrees with the config")
        if self.placement.num_experts() != config.num_experts:
            raise PlacementError(f"placement: covers {self.placement.num_experts()} experts, expected {config.num_experts}")
        per = {len(d) for d in self.placement.devices}
        if len(per) != 1:
            raise PlacementError("placement: uneven device lists")
        self.placement.expert_to_device()
        cfg = config._c()
        pl = (C.c_int32 * config.num_experts)(*self.placement.flat())
        h = C.c_void_p()
        _check(lib().occ_create(C.byref(cfg), pl, world_size, rank, C.byref(h)), "occ_create")
        self._h = h
        self._world = world_size
        self._prune_cache = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _LIB is not None:
            _LIB.occ_destroy(h)
            self._h = None

    # weights (reference layout: w1 [E, D, F], w3 [E, D, F], w2 [E, F, D]) --------
    def load_experts(self, w1: torch.Tensor, w2: torch.Tensor, w3: Optional[torch.Tensor] = None):
        _need_cuda(w1, w2, w3)
        ts = [t.to(torch.bfloat16).contiguous() if t is not None else None for t in (w1, w3, w2)]
        _check(lib().occ_load_experts(self._h, _ptr(ts[0]), _ptr(ts[1]), _ptr(ts[2]), _stream()), "load_experts")
        torch.cuda.current_stream().synchronize()
        self._weights = ts

    def load_shared_experts(self, w1: torch.Tensor, w2: torch.Tensor, w3: Optional[torch.Tensor] = None,
                            gate: Optional[torch.Tensor] = None):
        """Shared (always-active) experts, DeepSeek-MoE / Qwen-MoE style (not in
        the reference): w1/w3 [S, D, F_s], w2 [S, F_s, D]; optional
        gate [D] gives each token the weight sigmoid(x . gate) (Qwen's
        shared_expert_gate).  Computed at every token's source device and
        added last in the combine (include/occult.h)."""
        _need_cuda(w1, w2, w3, gate)
        ts = [t.to(torch.bfloat16).contiguous() if t is not None else None for t in (w1, w3, w2, gate)]
        _check(lib().occ_load_shared_experts(self._h, int(ts[0].shape[0]), int(ts[0].shape[2]), _ptr(ts[0]),
                                             _ptr(ts[1]), _ptr(ts[2]), _ptr(ts[3]), _stream()), "load_shared_experts")
        torch.cuda.current_stream().synchronize()
        self._shared = ts

    def set_placement(self, placement: Placement):
        pl = (C.c_int32 * self.config.num_experts)(*placement.flat())
        _check(lib().occ_set_placement(self._h, pl), "set_placement")
        self.placement = placement

    def set_similarity(self, values):
        import numpy as np
        v = np.ascontiguousarray(values, dtype=np.float64)
        _check(lib().occ_set_similarity(self._h, v.ctypes.data_as(C.c_void_p)), "set_similarity")

    def comm_init(self, group=None):
        """NCCL communicator for world_size > 1 (one process per GPU): rank 0
        creates the unique id, torch.distributed broadcasts it."""
        import torch.distributed as dist
        buf = (C.c_uint8 * 128)()
        if dist.get_rank(group) == 0:
            _check(lib().occ_comm_unique_id(buf), "comm_unique_id")
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        idb = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        _check(lib().occ_comm_init(self._h, idb), "comm_init")

    def comm_init_host(self, group=None):
        """occ_comm_init_host: the rank's exchanges bootstrapped over a host
        all-gather -- here torch.distributed on `group` (any backend that takes
        CPU tensors, e.g. gloo) -- instead of NCCL.  Pair with
        comm_enable_peer (CUDA IPC mapping; the forward then runs without any
        host involvement).  Works for several processes on one GPU."""
        self._host_fn = host_allgather_fn(group)  # kept alive with the handle
        _check(lib().occ_comm_init_host(self._h, self._host_fn, None), "comm_init_host")

    def router_logits(self, x: torch.Tensor, gate: torch.Tensor) -> torch.Tensor:
        """The production router's f32 logits x g^T [n, E] (tcgen05), e.g. to
        profile the similarity table of the similarity pruning mode."""
        _need_cuda(x, gate)
        c = self.config
        x = _arg(x, "router_logits: x", torch.bfloat16, (x.shape[0], c.embed_dim))
        gate = _arg(gate, "router_logits: gate", torch.bfloat16, (c.num_experts, c.embed_dim))
        out = torch.empty((x.shape[0], c.num_experts), dtype=torch.float32, device=x.device)
        _check(lib().occ_router_logits(self._h, _ptr(x), _ptr(gate), x.shape[0], _ptr(out), _stream()),
               "router_logits")
        return out

    def comm_enable_peer(self, max_tokens_per_rank: int):
        """Fused dispatch / return over peer memory instead of all-to-all calls
        (collective; after comm_init / comm_init_loopback)."""
        _check(lib().occ_comm_enable_peer(self._h, int(max_tokens_per_rank)), "comm_enable_peer")

    def set_micro_batches(self, micro_batches: int = 2, comm_sms: int = -1):
        """occ_set_micro_batches: run every forward as two micro-batches on two
        streams so one half's exchange overlaps the other half's GEMMs
        (collective when world_size > 1; after comm_init / comm_enable_peer)."""
        _check(lib().occ_set_micro_batches(self._h, micro_batches, comm_sms), "set_micro_batches")

    def comm_init_loopback(self, key: int):
        """Validation transport: world_size ranks as threads on one GPU."""
        _check(lib().occ_comm_init_loopback(self._h, C.c_long(key)), "comm_init_loopback")

    def allreduce_histogram(self, counts: torch.Tensor):
        _check(lib().occ_allreduce_histogram(self._h, _ptr(counts), _stream()), "allreduce_histogram")
        return counts

    def set_training(self, on: bool = True):
        """Keep what backward needs (call before load_experts)."""
        _check(lib().occ_set_training(self._h, int(on)), "set_training")

    def backward(self, upstream: torch.Tensor, grad_x_dtype: torch.dtype = torch.float32):
        """backward_vjps (backward.cpp:24-161) of the last forward: returns
        dict(x, w1, w3, w2, routing_weights) of gradients (ids fixed): fp32,
        except the token gradient in ``grad_x_dtype`` (fp32 or bf16)."""
        _need_cuda(upstream)
        c = self.config
        dev = upstream.device
        e_l = c.num_experts if self._world == 1 else c.experts_per_device()  # this rank's experts
        n = upstream.shape[0]
        if grad_x_dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError("backward: grad_x_dtype must be float32 or bfloat16")
        _check(lib().occ_set_grad_x_bf16(self._h, int(grad_x_dtype == torch.bfloat16)), "set_grad_x_bf16")
        g = {"x": torch.empty((n, c.embed_dim), dtype=grad_x_dtype, device=dev),
             "w1": torch.empty((e_l, c.embed_dim, c.hidden_dim), dtype=torch.float32, device=dev),
             "w2": torch.empty((e_l, c.hidden_dim, c.embed_dim), dtype=torch.float32, device=dev),
             "routing_weights": torch.empty((n, c.top_k), dtype=torch.float32, device=dev)}
        g["w3"] = torch.empty_like(g["w1"]) if c.activation == "swiglu" else None
        _check(lib().occ_backward(self._h, _ptr(upstream.to(torch.bfloat16).contiguous()), _ptr(g["x"]),
                                  _ptr(g["w1"]), _ptr(g["w3"]), _ptr(g["w2"]), _ptr(g["routing_weights"]),
                                  _stream()), "backward")
        return g

    def set_plan_kernels(self, fused: bool):
        """One cooperative kernel for the one-GPU index chain (default) or the
        multi-kernel chain (occ_set_plan_kernels); identical results."""
        _check(lib().occ_set_plan_kernels(self._h, int(fused)), "set_plan_kernels")

    def set_validate(self, on: bool):
        _check(lib().occ_set_validate(self._h, int(on)), "set_validate")

    def set_profiling(self, on: bool):
        _check(lib().occ_set_profiling(self._h, int(on)), "set_profiling")

    def stage_ms(self) -> dict:
        """CUDA-event time of each stage of the last forward (profiling on)."""
        buf = (C.c_float * len(STAGES))()
        n = lib().occ_stage_ms(self._h, buf, len(STAGES))
        return {STAGES[i]: float(buf[i]) for i in range(max(n, 0)) if buf[i] >= 0}

    # routing ------------------------------------------------------------------
    def route(self, x: torch.Tensor, gate: torch.Tensor, prune: Optional[PruneSpec] = None, want_scores=False):
        """Production router: ids int32 [n,k], weights f32 [n,k] (+ scores)."""
        _need_cuda(x, gate)
        n = x.shape[0]
        k = self.config.top_k
        x = _arg(x, "route: x", torch.bfloat16, (n, self.config.embed_dim))
        gate = _arg(gate, "route: gate", torch.bfloat16, (self.config.num_experts, self.config.embed_dim))
        ids = torch.empty((n, k), dtype=torch.int32, device=x.device)
        w = torch.empty((n, k), dtype=torch.float32, device=x.device)
        sc = torch.empty((n, self.config.num_experts), dtype=torch.float32, device=x.device) if want_scores else None
        pr = self._prune(prune)
        _check(lib().occ_route(self._h, _ptr(x), _ptr(gate), n,
                               C.byref(pr) if pr else None, _ptr(ids), _ptr(w), _ptr(sc), _stream()), "route")
        return (ids, w, sc) if want_scores else (ids, w)

    def set_router_mode(self, mode: str):
        """"tc" (default): tcgen05 router, equal to the reference except at
        f32-level near-ties; "exact": the reference's fp64 arithmetic with
        glibc's exp, bit-exact ids and weights (occ_set_router_mode)."""
        _check(lib().occ_set_router_mode(self._h, {"tc": 0, "exact": 1}[mode]), "set_router_mode")

    def route_exact(self, x: torch.Tensor, gate: torch.Tensor, prune: Optional[PruneSpec] = None,
                    want_scores=False):
        """gate_scores -> topk_route -> prune_routing of forward_expert_parallel
        (pipeline.cpp:509-512) bit for bit on the bf16 operands: ids int32
        [n,k], weights f64 [n,k] (+ f64 softmax scores [n,E])."""
        _need_cuda(x, gate)
        c = self.config
        n = x.shape[0]
        x = _arg(x, "route_exact: x", torch.bfloat16, (n, c.embed_dim))
        gate = _arg(gate, "route_exact: gate", torch.bfloat16, (c.num_experts, c.embed_dim))
        ids = torch.empty((n, c.top_k), dtype=torch.int32, device=x.device)
        w = torch.empty((n, c.top_k), dtype=torch.float64, device=x.device)
        sc = torch.empty((n, c.num_experts), dtype=torch.float64, device=x.device) if want_scores else None
        pr = self._prune(prune)
        _check(lib().occ_route_exact(self._h, _ptr(x), _ptr(gate), n, C.byref(pr) if pr else None, _ptr(ids),
                                     _ptr(w), _ptr(sc), _stream()), "route_exact")
        return (ids, w, sc) if want_scores else (ids, w)

    def _prune(self, prune):
        if prune is None or prune.mode == "none":
            return None
        if prune.mode == "similarity" and prune.table is not None and self._prune_cache is not prune.table:
            self.set_similarity(prune.table)
            self._prune_cache = prune.table
        return prune._c()

    def prune_routing(self, scores: torch.Tensor, ids: torch.Tensor, w: torch.Tensor, prune: PruneSpec):
        """prune_routing (pruning.cpp:141-163) on fp64 scores, bit-exact."""
        _need_cuda(scores, ids, w)
        oi = torch.empty_like(ids)
        ow = torch.empty_like(w)
        pr = self._prune(prune) or _Prune(0, 1, 0)
        _check(lib().occ_prune_routing_f64(self._h, _ptr(scores), _ptr(ids), _ptr(w), ids.shape[0], C.byref(pr),
                                           _ptr(oi), _ptr(ow), _stream()), "prune_routing")
        return oi, ow

    # EP path -------------------------------------------------------------------
    def build_dispatch_index(self, ids: torch.Tensor, sources: Optional[torch.Tensor] = None):
        """BRIM0 (pipeline.cpp:24-50) + the Sfd row counts.  world_size 1: every
        source (BRIM0s concatenated, counts [N_d, N_d]); world_size > 1: this
        rank's tokens as one source (BRIM0 [N_d * n], counts [N_d])."""
        _need_cuda(ids, sources)
        n = ids.shape[0]
        nd = self.config.num_devices
        ids = _arg(ids, "build_dispatch_index: ids", torch.int32, (n, self.config.top_k))
        sources = _arg(sources, "build_dispatch_index: sources", torch.int32, (n,))
        brim0 = torch.empty(n * nd, dtype=torch.int32, device=ids.device)
        counts = torch.empty((nd, nd) if self._world == 1 else (nd,), dtype=torch.int32, device=ids.device)
        _check(lib().occ_build_dispatch(self._h, _ptr(ids), _ptr(sources), n, _ptr(brim0),
                                        _ptr(counts), _stream()), "build_dispatch")
        return brim0, counts

    # stage-level entry points (pipeline.hpp:89-123) ------------------------------
    def dispatch(self, x: torch.Tensor, ids: torch.Tensor, w: torch.Tensor, brim0: torch.Tensor,
                 n_sfd: Optional[int] = None):
        """dispatch (pipeline.cpp:91-123) of one source's tokens by its BRIM0
        [N_d * n]: the SfdBatch (x rows, ids, weights, token index), device-major."""
        _need_cuda(x, ids, w, brim0)
        c = self.config
        n = x.shape[0]
        x = _arg(x, "dispatch: x", torch.bfloat16, (n, c.embed_dim))
        ids = _arg(ids, "dispatch: ids", torch.int32, (n, c.top_k))
        w = _arg(w, "dispatch: weights", torch.float32, (n, c.top_k))
        brim0 = _arg(brim0.reshape(-1), "dispatch: brim0", torch.int32, (c.num_devices * n,))
        if n_sfd is None:
            n_sfd = int((brim0 >= 0).sum())
        dev = x.device
        sx = torch.empty((n_sfd, c.embed_dim), dtype=torch.bfloat16, device=dev)
        si = torch.empty((n_sfd, c.top_k), dtype=torch.int32, device=dev)
        sw = torch.empty((n_sfd, c.top_k), dtype=torch.float32, device=dev)
        st = torch.empty(n_sfd, dtype=torch.int32, device=dev)
        _check(lib().occ_dispatch(self._h, _ptr(x), _ptr(ids), _ptr(w), n, _ptr(brim0), _ptr(sx), _ptr(si), _ptr(sw),
                                  _ptr(st), _stream()), "dispatch")
        return sx, si, sw, st

    def build_compute_index(self, device: int, in_ids: torch.Tensor, in_w: torch.Tensor):
        """build_compute_index (pipeline.cpp:52-89) of EP device `device` over
        its inbox rows: (cindex [P, R] int32, n_epd)."""
        _need_cuda(in_ids, in_w)
        c = self.config
        r = in_ids.shape[0]
        in_ids = _arg(in_ids, "build_compute: ids", torch.int32, (r, c.top_k))
        in_w = _arg(in_w, "build_compute: weights", torch.float32, (r, c.top_k))
        cix = torch.empty((c.experts_per_device(), r), dtype=torch.int32, device=in_ids.device)
        ne = torch.zeros(1, dtype=torch.int32, device=in_ids.device)
        _check(lib().occ_build_compute(self._h, device, _ptr(in_ids), _ptr(in_w), r, _ptr(cix), _ptr(ne), _stream()),
               "build_compute")
        return cix, int(ne.item())

    def expert_compute(self, device: int, in_x: torch.Tensor, in_ids: torch.Tensor, in_w: torch.Tensor,
                       out: Optional[torch.Tensor] = None):
        """scatter_matmul -> apply_activation -> weight_modulate -> merge_matmul
        (pipeline.cpp:178-283) of EP device `device`: the partial-combined
        return rows [R, D] bf16."""
        _need_cuda(in_x, in_ids, in_w)
        c = self.config
        r = in_x.shape[0]
        in_x = _arg(in_x, "expert_compute: x", torch.bfloat16, (r, c.embed_dim))
        in_ids = _arg(in_ids, "expert_compute: ids", torch.int32, (r, c.top_k))
        in_w = _arg(in_w, "expert_compute: weights", torch.float32, (r, c.top_k))
        if out is None:
            out = torch.empty_like(in_x)
        _check(lib().occ_expert_compute(self._h, device, _ptr(in_x), _ptr(in_ids), _ptr(in_w), r, _ptr(out),
                                        _stream()), "expert_compute")
        return out

    def combine(self, y_returned: torch.Tensor, brim0: torch.Tensor, n: int, out: Optional[torch.Tensor] = None):
        """combine (pipeline.cpp:285-300) of one source: Ori rows [n, D] bf16."""
        _need_cuda(y_returned, brim0)
        c = self.config
        y = _arg(y_returned, "combine: rows", torch.bfloat16, (y_returned.shape[0], c.embed_dim))
        brim0 = _arg(brim0.reshape(-1), "combine: brim0", torch.int32, (c.num_devices * n,))
        if out is None:
            out = torch.empty((n, c.embed_dim), dtype=torch.bfloat16, device=y.device)
        _check(lib().occ_combine(self._h, _ptr(y), _ptr(brim0), n, _ptr(out), _stream()), "combine")
        return out

    def forward_given_routing(self, x: torch.Tensor, ids: torch.Tensor, w: torch.Tensor,
                              sources: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None):
        """pipeline.cpp:360-501 (values) — returns the Ori-order output."""
        _need_cuda(x, ids, w, sources)
        if x.dtype != torch.bfloat16:
            raise ShapeError("forward: tokens must be bf16")
        n = x.shape[0]
        if ids.shape[0] != n:
            raise ShapeError("forward: routing token count mismatch")
        if x.shape[1] != self.config.embed_dim:
            raise ShapeError("forward: token width != expert input width")
        if sources is not None and sources.shape[0] != n:
            raise ShapeError("forward: one source device per token required")
        c = self.config
        x = x.contiguous()
        ids = _arg(ids, "forward: ids", torch.int32, (n, c.top_k))
        w = w.float().contiguous() if w.dtype != torch.float32 else w.contiguous()
        if tuple(w.shape) != (n, c.top_k):
            raise ShapeError(f"forward: routing weights must be [{n}, {c.top_k}]")
        sources = _arg(sources, "forward: sources", torch.int32, (n,))
        if out is None:
            out = torch.empty_like(x)
        out = _arg(out, "forward: out", torch.bfloat16, tuple(x.shape))
        _check(lib().occ_forward(self._h, _ptr(x), _ptr(ids), _ptr(w), _ptr(sources), n, _ptr(out), _stream()),
               "forward")
        return out

    def forward_expert_parallel(self, x, gate, prune: Optional[PruneSpec] = None, sources=None, out=None):
        """pipeline.cpp:503-517: route (+prune) then the indexed data path."""
        _need_cuda(x, gate, sources)
        c = self.config
        n = x.shape[0]
        x = _arg(x, "forward_expert_parallel: x", torch.bfloat16, (n, c.embed_dim))
        gate = _arg(gate, "forward_expert_parallel: gate", torch.bfloat16, (c.num_experts, c.embed_dim))
        sources = _arg(sources, "forward_expert_parallel: sources", torch.int32, (n,))
        if out is None:
            out = torch.empty_like(x)
        out = _arg(out, "forward_expert_parallel: out", torch.bfloat16, (n, c.embed_dim))
        pr = self._prune(prune)
        _check(lib().occ_forward_expert_parallel(self._h, _ptr(x), _ptr(gate), C.byref(pr) if pr else None,
                                                 _ptr(sources), x.shape[0], _ptr(out), _stream()), "forward_ep")
        return out

    def forward_host(self, x_host: torch.Tensor, gate: torch.Tensor, out_host: torch.Tensor,
                     prune: Optional[PruneSpec] = None, chunks: int = 1, wait: bool = True):
        """End to end from pinned host memory (occ_forward_host): the H2D copy
        of this call and the D2H copy of the previous call overlap the layer.
        ``wait=False`` leaves the result pending until ``host_wait()``."""
        if x_host.is_cuda or out_host.is_cuda:
            raise ShapeError("forward_host: x and out are host tensors")
        _need_cuda(gate)
        c = self.config
        n = x_host.shape[0]
        for t, nm in ((x_host, "x_host"), (out_host, "out_host")):
            # asynchronous: the library keeps reading / writing these pointers
            # after the call returns, so no temporary copies
            if t.dtype != torch.bfloat16 or tuple(t.shape) != (n, c.embed_dim) or not t.is_contiguous():
                raise ShapeError(f"forward_host: {nm} must be a contiguous bf16 [{n}, {c.embed_dim}] host tensor")
        gate = _arg(gate, "forward_host: gate", torch.bfloat16, (c.num_experts, c.embed_dim))
        self._host_gate = gate  # the captured graph reads it on later replays
        pr = self._prune(prune)
        _check(lib().occ_forward_host(self._h, _ptr(x_host), _ptr(gate), C.byref(pr) if pr else None,
                                      x_host.shape[0], _ptr(out_host), chunks, _stream()), "forward_host")
        if wait:
            self.host_wait()
        return out_host

    def host_wait(self):
        _check(lib().occ_host_wait(self._h, _stream()), "host_wait")
        tp = getattr(self, "_tpipe", None)
        if tp is not None and tp["last"] is not None:
            torch.cuda.current_stream().wait_event(tp["last"])

    def train_step_host(self, x_host: torch.Tensor, gate: torch.Tensor, upstream_host: torch.Tensor,
                        grad_x_host: torch.Tensor, prune: Optional[PruneSpec] = None, wait: bool = True):
        """Training step end to end from pinned host memory: H2D of tokens and
        upstream gradient, forward_expert_parallel + backward_vjps on the
        device, D2H of the token gradient (fp32, or bf16 when grad_x_host is
        bf16 — mixed precision halves the D2H); expert / routing-weight
        gradients stay on the device (returned).  Double-buffered like
        forward_host: the copies of step i+1 / i-1 run on two copy streams
        while step i computes.  ``wait=False`` leaves the D2H pending until
        ``host_wait()``; host buffers must stay untouched until then."""
        if x_host.is_cuda or upstream_host.is_cuda or grad_x_host.is_cuda:
            raise ShapeError("train_step_host: x, upstream and grad_x are host tensors")
        _need_cuda(gate)
        dev = gate.device
        tp = getattr(self, "_tpipe", None)
        if tp is None or tp["shape"] != tuple(x_host.shape):
            torch.cuda.synchronize(dev)
            tp = {"shape": tuple(x_host.shape), "calls": 0, "last": None,
                  "s_in": torch.cuda.Stream(dev), "s_out": torch.cuda.Stream(dev),
                  "x": [torch.empty(x_host.shape, dtype=torch.bfloat16, device=dev) for _ in range(2)],
                  "up": [torch.empty(x_host.shape, dtype=torch.bfloat16, device=dev) for _ in range(2)],
                  "out": [torch.empty(x_host.shape, dtype=torch.bfloat16, device=dev) for _ in range(2)],
                  "free": [None, None], "gx": [None, None], "gdone": [None, None]}
            self._tpipe = tp
        slot = tp["calls"] & 1
        tp["calls"] += 1
        main = torch.cuda.current_stream(dev)
        with torch.cuda.stream(tp["s_in"]):
            if tp["free"][slot] is not None:  # the step that last used this slot has read x / upstream
                tp["s_in"].wait_event(tp["free"][slot])
            tp["x"][slot].copy_(x_host, non_blocking=True)
            tp["up"][slot].copy_(upstream_host, non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(tp["s_in"])
        main.wait_event(ev_in)
        if tp["gdone"][slot] is not None:  # the D2H that last read this slot's gradient finished
            main.wait_event(tp["gdone"][slot])
        self.forward_expert_parallel(tp["x"][slot], gate, prune=prune, out=tp["out"][slot])
        g = self.backward(tp["up"][slot], grad_x_dtype=grad_x_host.dtype)
        ev_c = torch.cuda.Event()
        ev_c.record(main)
        tp["free"][slot] = ev_c
        tp["gx"][slot] = g["x"]
        with torch.cuda.stream(tp["s_out"]):
            tp["s_out"].wait_event(ev_c)
            grad_x_host.copy_(g["x"], non_blocking=True)
            ev_o = torch.cuda.Event()
            ev_o.record(tp["s_out"])
        tp["gdone"][slot] = ev_o
        tp["last"] = ev_o
        if wait:
            self.host_wait()
        return g

    def comm_report(self, bytes_per_scalar: int = 4, cap_replicas: Optional[float] = None) -> CommReport:
        r = _Report()
        _check(lib().occ_comm_report_get(self._h, bytes_per_scalar, C.byref(r), _stream()), "comm_report")
        nd = self.config.num_devices
        return CommReport(r.mean_replicas, r.cap_replicas if cap_replicas is None else cap_replicas, r.intra_share,
                          r.inter_share, r.cross_device_bytes, r.crossing_rows, r.naive_crossing_rows, r.n_sfd,
                          r.n_epd, [int(r.per_device_rows[d]) for d in range(nd)])

    def saved_index(self):
        """Inbox records (token, source, slot) and BRIM1 of the last forward."""
        rep = self.comm_report()
        R = sum(rep.per_device_token_counts)
        P = self.config.experts_per_device()
        dev = torch.device("cuda")
        tok = torch.empty(R, dtype=torch.int32, device=dev)
        src = torch.empty(R, dtype=torch.int32, device=dev)
        slot = torch.empty(R, dtype=torch.int32, device=dev)
        cix = torch.empty(R * P, dtype=torch.int32, device=dev)
        _check(lib().occ_saved_index(self._h, _ptr(tok), _ptr(src), _ptr(slot), _ptr(cix), _stream()), "saved_index")
        return tok, src, slot, cix, rep.per_device_token_counts


# ------------------------------------------------------ stateless functions --

def gate_scores_f64(x: torch.Tensor, gate: torch.Tensor) -> torch.Tensor:
    """gate_scores (routing.cpp:33-52), exact fp64 mode."""
    _need_cuda(x, gate)
    x, gate = x.double().contiguous(), gate.double().contiguous()
    out = torch.empty((x.shape[0], gate.shape[0]), dtype=torch.float64, device=x.device)
    if x.shape[1] != gate.shape[1]:
        raise ShapeError(f"gate_scores: token width {x.shape[1]} != gate width {gate.shape[1]}")
    _check(lib().occ_gate_scores_f64(_ptr(x), x.shape[0], x.shape[1], _ptr(gate), gate.shape[0], _ptr(out),
                                     _stream()), "gate_scores")
    return out


def gate_logits_f64(x: torch.Tensor, gate: torch.Tensor) -> torch.Tensor:
    """Router logits x @ gate^T in fp64, k ascending (tiled_matmul Double,
    matrix.cpp:9-38); bit-exact with the reference."""
    _need_cuda(x, gate)
    x, gate = x.double().contiguous(), gate.double().contiguous()
    if x.shape[1] != gate.shape[1]:
        raise ShapeError(f"gate_logits: token width {x.shape[1]} != gate width {gate.shape[1]}")
    out = torch.empty((x.shape[0], gate.shape[0]), dtype=torch.float64, device=x.device)
    _check(lib().occ_gate_logits_f64(_ptr(x), x.shape[0], x.shape[1], _ptr(gate), gate.shape[0], _ptr(out),
                                     _stream()), "gate_logits")
    return out


def topk_route(scores: torch.Tensor, k: int, renormalize: bool = True):
    """topk_route (routing.cpp:60-84) on fp64 scores; bit-exact."""
    _need_cuda(scores)
    s = scores.double().contiguous()
    n, e = s.shape
    ids = torch.empty((n, k), dtype=torch.int32, device=s.device)
    w = torch.empty((n, k), dtype=torch.float64, device=s.device)
    _check(lib().occ_topk_route_f64(_ptr(s), n, e, k, int(renormalize), _ptr(ids), _ptr(w), _stream()), "topk_route")
    return ids, w


def accumulate_collab(counts: torch.Tensor, ids: torch.Tensor) -> torch.Tensor:
    """accumulate_collab (collab.cpp:10-23): int64 [E,E] device histogram, in place."""
    _need_cuda(counts, ids)
    e = counts.shape[0]
    n, k = ids.shape
    ids = _arg(ids, "accumulate_collab: ids", torch.int32, (n, k))
    if counts.dtype != torch.int64 or tuple(counts.shape) != (e, e) or not counts.is_contiguous():
        raise ShapeError("accumulate_collab: counts must be a contiguous int64 [E, E] tensor (accumulated in place)")
    _check(lib().occ_coactivation_histogram(_ptr(ids), n, k, e, _ptr(counts), _stream()), "collab")
    return counts


def build_collab_graph(ids: torch.Tensor, num_experts: int) -> torch.Tensor:
    counts = torch.zeros((num_experts, num_experts), dtype=torch.int64, device=ids.device)
    return accumulate_collab(counts, ids)


def normalize_graph(counts) -> "numpy.ndarray":
    """normalize_graph (collab.cpp:31-39), host."""
    import numpy as np
    c = np.ascontiguousarray(counts.cpu().numpy() if isinstance(counts, torch.Tensor) else counts, dtype=np.int64)
    e = c.shape[0]
    p = np.empty((e, e), np.float64)
    _check(lib().occ_normalize_graph(c.ctypes.data_as(C.c_void_p), e, p.ctypes.data_as(C.c_void_p)), "normalize")
    return p


def reschedule_placement(p, num_devices: int) -> Placement:
    """reschedule_placement (placement.cpp:88-148), host, bit-exact."""
    import numpy as np
    p = np.ascontiguousarray(p, dtype=np.float64)
    e = p.shape[0]
    out = np.empty(e, np.int32)
    _check(lib().occ_reschedule_placement(p.ctypes.data_as(C.c_void_p), e, num_devices,
                                          out.ctypes.data_as(C.c_void_p)), "reschedule_placement")
    per = e // num_devices
    return Placement([out[d * per:(d + 1) * per].tolist() for d in range(num_devices)])


def build_similarity_table(logit_batches, num_experts: int):
    """build_similarity_table (pruning.cpp:213-218): the squared-cosine table
    of router-logit columns, accumulated batch by batch on the device
    (SimilarityAccumulator::add in fp64; bit-exact for fp64 logits), finalised
    on the host.  Batches: CUDA tensors [n, E], float64 or float32.
    Returns the [E, E] float64 numpy table for ExpertParallelLayer.set_similarity."""
    import numpy as np
    inner = None
    tokens = 0
    for b in logit_batches:
        _need_cuda(b)
        if inner is None:
            inner = torch.zeros((num_experts, num_experts), dtype=torch.float64, device=b.device)
        fp64 = b.dtype == torch.float64
        bb = b.contiguous() if fp64 else b.float().contiguous()
        _check(lib().occ_similarity_accumulate(_ptr(bb), int(fp64), bb.shape[0], num_experts, _ptr(inner),
                                               _stream()), "similarity_accumulate")
        tokens += bb.shape[0]
    if inner is None:
        raise ShapeError("build_similarity_table: no batches")
    h = np.ascontiguousarray(inner.cpu().numpy())
    v = np.empty_like(h)
    _check(lib().occ_similarity_finalize(h.ctypes.data_as(C.c_void_p), C.c_longlong(tokens), num_experts,
                                         v.ctypes.data_as(C.c_void_p)), "similarity_finalize")
    return v


def collaboration_aware_placement(routing_batches, num_experts: int, num_devices: int,
                                  layer: Optional["ExpertParallelLayer"] = None) -> Placement:
    """The profiling -> placement loop (Occult Alg. 1):
    co-activation histogram of the profiled routing batches on the device
    (accumulate_collab, collab.cpp:10-23; summed across ranks with
    occ_allreduce_histogram when `layer` is a world_size > 1 handle), then the
    host normalize_graph + reschedule_placement (placement.cpp:88-148)."""
    counts = None
    for ids in routing_batches:
        if counts is None:
            counts = torch.zeros((num_experts, num_experts), dtype=torch.int64, device=ids.device)
        accumulate_collab(counts, ids)
    if counts is None:
        raise ShapeError("collaboration_aware_placement: no routing batches")
    if layer is not None and getattr(layer, "_world", 1) > 1:
        layer.allreduce_histogram(counts)
    return reschedule_placement(normalize_graph(counts), num_devices)


def host_allgather_fn(group=None):
    """The occ_host_allgather_fn of occ_comm_init_host over torch.distributed:
    fn(ctx, send, bytes, recv) gathers `bytes` from every rank of `group` into
    recv [world * bytes] in rank order (CPU tensors: gloo), 0 on success."""
    import torch.distributed as dist

    def fn(_ctx, send, nbytes, recv):
        try:
            if nbytes == 0:
                return 0
            world = dist.get_world_size(group)
            src = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8)
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, src, group=group)
            cat = torch.cat(outs)  # (kept referenced until the copy is done)
            C.memmove(recv, cat.data_ptr(), world * nbytes)
            return 0
        except Exception:  # noqa: BLE001 -- reported as OCC_ERR_NCCL by the library
            return 1

    return _ALLGATHER_FN(fn)


def exchange_layout(counts, rank: int):
    """occ_exchange_layout: (send_off, send_cnt, recv_off, recv_cnt) per peer."""
    import numpy as np
    c = np.ascontiguousarray(counts, dtype=np.int32)
    nd = c.shape[0]
    outs = [np.zeros(nd, np.int64) for _ in range(4)]
    _check(lib().occ_exchange_layout(c.ctypes.data_as(C.c_void_p), nd, rank,
                                     *[o.ctypes.data_as(C.c_void_p) for o in outs]), "exchange_layout")
    return tuple(outs)


def round_robin_sources(num_tokens: int, num_devices: int, device="cuda") -> torch.Tensor:
    """pipeline.cpp:12-16."""
    return (torch.arange(num_tokens, dtype=torch.int32, device=device) % num_devices).to(torch.int32)
