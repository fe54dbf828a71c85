"""numpy/ctypes front-end to the CPU parity checkers.

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs; never by the product package.

Two backends with identical semantics:
  * ``Port`` wraps oracle/liboccoracle.so, the C restatement (occ_oracle.c).
  * ``Ref``  wraps oracle/_ref/libmoesim_ref.so, the reference sources
    compiled where they lie plus the extern "C" shim ref_capi.cpp.  It exists
    only where /root/reference was present at build time (this container;
    the built .so travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboccoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoesim_ref.so")

ACT = {"identity": 0, "silu": 1, "relu": 2}
PRUNE = {"none": 0, "router": 1, "similarity": 2}

_i = C.c_int
_d = C.c_double
_p = C.c_void_p


class Report(C.Structure):
    """orc_report / ref_report: CommReport (collab.hpp:36-43) + index sizes."""

    _fields_ = [
        ("mean_replicas", _d), ("cap_replicas", _d), ("intra_share", _d), ("inter_share", _d),
        ("cross_device_bytes", C.c_longlong), ("crossing_rows", C.c_longlong),
        ("per_device_rows", C.c_longlong * 64), ("n_sfd_src", _i * 64), ("n_epd_dev", _i * 64),
    ]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: status {code}")
        self.code = code


def _check(rc, what):
    if rc != 0:
        raise OracleError(rc, what)


def _build_if_missing():
    if not os.path.exists(PORT_SO) or (os.path.isdir("/root/reference") and not os.path.exists(REF_SO)):
        import subprocess
        subprocess.run(["make", "-s", "-C", HERE], check=True)


class Rng:
    """std::mt19937_64 + rng.hpp draws (oracle restatement)."""

    def __init__(self, seed: int):
        lib = port_lib()
        self._buf = C.create_string_buffer(lib.orc_rng_size())
        lib.orc_rng_seed(self._buf, C.c_uint64(seed))
        self._lib = lib

    def next(self) -> int:
        return self._lib.orc_rng_next(self._buf)

    def uniform(self) -> float:
        return self._lib.orc_rng_uniform(self._buf)

    def uniform_int(self, n: int) -> int:
        return self._lib.orc_rng_uniform_int(self._buf, n)

    def random_matrix(self, rows, cols, single=True):
        out = np.empty((rows, cols), np.float64)
        self._lib.orc_random_matrix(self._buf, rows, cols, int(single), _ptr(out))
        return out


_PORT = None
_REF = None


def port_lib():
    global _PORT
    if _PORT is None:
        _build_if_missing()
        lib = C.CDLL(PORT_SO)
        lib.orc_rng_size.restype = C.c_size_t
        lib.orc_rng_next.restype = C.c_uint64
        lib.orc_rng_uniform.restype = _d
        lib.orc_rng_uniform_range.restype = _d
        lib.orc_mean_token_replicas.restype = _d
        lib.orc_max_rel_error.restype = _d
        for fn in ("orc_gate_scores", "orc_gate_logits", "orc_softmax_rows", "orc_normalize_graph",
                   "orc_similarity_table", "orc_random_matrix", "orc_dense_given_routing", "orc_rng_seed",
                   "orc_trivial_placement", "orc_collaboration_shares", "orc_shared_experts",
                   "orc_dense_rows_bf16"):
            getattr(lib, fn).restype = None
        lib.orc_rng_seed.argtypes = [_p, C.c_uint64]
        lib.orc_max_rel_error.argtypes = [_p, _p, C.c_long]
        lib.orc_forward_given_routing.argtypes = (
            [_p, _i, _i, _p, _p, _i, _p, _p, _p, _i, _i, _p, _i, _p, _i, _i, _i, _d] + [_p] * 7)
        lib.orc_dense_given_routing.argtypes = [_p, _i, _i, _p, _p, _i, _p, _p, _p, _i, _i, _i, _p, _i, _p]
        lib.orc_shared_experts.argtypes = [_p, _i, _i, _p, _p, _p, _i, _i, _i, _p, _p]
        lib.orc_dense_rows_bf16.argtypes = ([_p, _i, _i, _p, _p, _i, _i, _p, _p, _p, _i, _i, _i, _p, _p, _p, _i, _p,
                                             _p, _i, _p])
        _PORT = lib
    return _PORT


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir("/root/reference")


def ref_lib():
    global _REF
    if _REF is None:
        _build_if_missing()
        lib = C.CDLL(REF_SO)
        lib.ref_forward_given_routing.argtypes = (
            [_p, _i, _i, _p, _p, _i, _p, _p, _i, _i, _p, _i, _p, _i, _i, _i, _d] + [_p] * 7)
        lib.ref_dense_given_routing.argtypes = [_p, _i, _i, _p, _p, _i, _p, _p, _i, _i, _i, _i, _p]
        lib.ref_rng_uniform_stream.argtypes = [C.c_uint64, _i, _p]
        lib.ref_random_matrix.argtypes = [C.c_uint64, _i, _i, _i, _p]
        lib.ref_forward_expert_parallel_mt.argtypes = [_p, _i, _i, _p, _i, _i, _p, _p, _i, _i, _i, _i, _i, _p]
        lib.ref_session_create.restype = _p
        lib.ref_session_create.argtypes = [_p, _i, _i, _p, _p, _i, _i, _i, _i, _i]
        lib.ref_session_destroy.argtypes = [_p]
        lib.ref_session_forward.argtypes = [_p, _p, _i, _i, _p]
        lib.ref_backward.argtypes = [_p, _i, _i, _p, _p, _i, _p, _p, _i, _i, _p, _i, _p, _i, _i] + [_p] * 5
        lib.ref_gen_trace_text.restype = C.c_longlong
        lib.ref_gen_trace_text.argtypes = [_i] * 4 + [_d, _i, _d, C.c_char_p, C.c_uint64, C.c_char_p, C.c_longlong]
        lib.ref_roundtrip_text.restype = C.c_longlong
        lib.ref_roundtrip_text.argtypes = [_i, C.c_char_p, C.c_char_p, C.c_longlong]
        lib.ref_write_matrix_text.restype = C.c_longlong
        lib.ref_write_matrix_text.argtypes = [_p, _i, _i, C.c_char_p, C.c_longlong]
        lib.ref_write_placement_text.restype = C.c_longlong
        lib.ref_write_placement_text.argtypes = [_p, _i, _i, C.c_char_p, C.c_longlong]
        lib.ref_component_points.argtypes = [_p, _i, _i, _i, _i, _p, _p]
        _REF = lib
    return _REF


def _ref_text(call):
    """Run a ref_*_text shim (returns the full length, -1 on error) with a
    buffer that grows until the text fits: (ok, text)."""
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        n = call(buf, cap)
        if n < cap:
            return n >= 0, buf.value.decode("latin-1")
        cap = n + 1


def ref_gen_trace(dist, ne, k, n, alpha, blocks, p_in, tag, seed):
    """write_trace(gen_trace(spec, seed)) of the reference (trace_gen.cpp,
    io.cpp:71-86); dist 0 uniform, 1 zipf, 2 blocks."""
    L = ref_lib()
    return _ref_text(lambda b, c: L.ref_gen_trace_text(dist, ne, k, n, alpha, blocks, p_in, tag.encode(),
                                                       seed & (2 ** 64 - 1), b, c))


def ref_roundtrip(kind, text):
    """read_* then write_* in the reference (0 trace, 1 matrix, 2 placement)."""
    L = ref_lib()
    return _ref_text(lambda b, c: L.ref_roundtrip_text(kind, text.encode("latin-1"), b, c))


def ref_write_matrix(m):
    m = _f64(m)
    L = ref_lib()
    return _ref_text(lambda b, c: L.ref_write_matrix_text(_ptr(m), m.shape[0], m.shape[1], b, c))[1]


def ref_write_placement(plist):
    a = _i32(plist)
    L = ref_lib()
    return _ref_text(lambda b, c: L.ref_write_placement_text(_ptr(a), a.shape[0], a.shape[1], b, c))[1]


def ref_component_points(ids, ne, batch=256):
    """ComponentTracker over batch-token slices (collab.cpp:120-169)."""
    ids = _i32(ids)
    n, k = ids.shape
    npts = (n + batch - 1) // batch + 1
    tok = np.zeros(npts, np.int64)
    size = np.zeros(npts, np.int32)
    got = ref_lib().ref_component_points(_ptr(ids), n, k, ne, batch, _ptr(tok), _ptr(size))
    return [(int(tok[i]), int(size[i])) for i in range(got)]


class _Backend:
    prefix = ""

    def __init__(self):
        self.lib = None

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    # ---------------------------------------------------------------- routing
    def gate_scores(self, x, g):
        x, g = _f64(x), _f64(g)
        n, d = x.shape
        e = g.shape[0]
        out = np.empty((n, e), np.float64)
        rc = self._fn("gate_scores")(_ptr(x), n, d, _ptr(g), e, _ptr(out))
        _check(rc or 0, "gate_scores")
        return out

    def topk_route(self, scores, k, renormalize=True):
        s = _f64(scores)
        n, e = s.shape
        ids = np.empty((n, k), np.int32)
        w = np.empty((n, k), np.float64)
        _check(self._fn("topk_route")(_ptr(s), n, e, k, int(renormalize), _ptr(ids), _ptr(w)), "topk_route")
        return ids, w

    # ---------------------------------------------------------------- collab
    def accumulate_collab(self, ids, ne, counts=None):
        ids = _i32(ids)
        n, k = ids.shape
        c = np.zeros((ne, ne), np.int64) if counts is None else np.ascontiguousarray(counts, np.int64).copy()
        if self.prefix == "ref_":
            w = np.ones((n, k), np.float64)
            rc = self.lib.ref_accumulate_collab(_ptr(ids), _ptr(w), n, k, ne, _ptr(c))
        else:
            rc = self.lib.orc_accumulate_collab(_ptr(ids), n, k, ne, _ptr(c))
        _check(rc, "accumulate_collab")
        return c

    def normalize_graph(self, counts):
        c = np.ascontiguousarray(counts, np.int64)
        ne = c.shape[0]
        p = np.empty((ne, ne), np.float64)
        rc = self._fn("normalize_graph")(_ptr(c), ne, _ptr(p))
        _check(rc or 0, "normalize_graph")
        return p

    def reschedule_placement(self, p, nd):
        p = _f64(p)
        ne = p.shape[0]
        out = np.empty((nd, ne // nd), np.int32)
        _check(self._fn("reschedule_placement")(_ptr(p), ne, nd, _ptr(out)), "reschedule_placement")
        return out

    # --------------------------------------------------------------- pipeline
    def forward_given_routing(self, x, ids, w, w1, w2, plist, sources=None, act="silu", single=True,
                              bytes_per_scalar=4, cap_replicas=-1.0, w3=None, want_index=False):
        x, w, w1, w2 = _f64(x), _f64(w), _f64(w1), _f64(w2)
        ids, plist = _i32(ids), _i32(plist)
        n, dm = x.shape
        k = ids.shape[1]
        ne, _, dh = w1.shape
        nd = plist.shape[0]
        if sources is None:
            sources = np.arange(n, dtype=np.int32) % nd  # round_robin_sources, pipeline.cpp:12-16
        sources = _i32(sources)
        out = np.empty((n, dm), np.float64)
        rep = Report()
        idx = {}
        if want_index:
            idx["dindex"] = np.empty(nd * n, np.int32)
            idx["inbox_token"] = np.empty(n * nd, np.int32)
            idx["inbox_source"] = np.empty(n * nd, np.int32)
            idx["inbox_slot"] = np.empty(n * nd, np.int32)
            idx["cindex"] = np.empty((ne // nd) * n * nd, np.int32)
        args = [_ptr(idx.get(key)) for key in ("dindex", "inbox_token", "inbox_source", "inbox_slot", "cindex")]
        if self.prefix == "ref_":
            if w3 is not None:
                raise ValueError("the reference has no gated experts (SPEC.md:73)")
            rc = self.lib.ref_forward_given_routing(
                _ptr(x), n, dm, _ptr(ids), _ptr(w), k, _ptr(w1), _ptr(w2), ne, dh, _ptr(plist), nd,
                _ptr(sources), ACT[act], int(single), bytes_per_scalar, cap_replicas, _ptr(out),
                C.byref(rep), *args)
        else:
            w3p = None if w3 is None else _f64(w3)
            rc = self.lib.orc_forward_given_routing(
                _ptr(x), n, dm, _ptr(ids), _ptr(w), k, _ptr(w1), _ptr(w2), _ptr(w3p), ne, dh,
                _ptr(plist), nd, _ptr(sources), ACT[act], int(single), bytes_per_scalar, cap_replicas,
                _ptr(out), C.byref(rep), *args)
        _check(rc, "forward_given_routing")
        if want_index:
            return out, rep, _split_index(idx, rep, nd, ne // nd, sources)
        return out, rep

    def dense_given_routing(self, x, ids, w, w1, w2, act="silu", single=True, rows=None, w3=None):
        x, w, w1, w2, ids = _f64(x), _f64(w), _f64(w1), _f64(w2), _i32(ids)
        n, dm = x.shape
        k = ids.shape[1]
        ne, _, dh = w1.shape
        if self.prefix == "ref_":
            assert rows is None and w3 is None
            out = np.empty((n, dm), np.float64)
            _check(self.lib.ref_dense_given_routing(_ptr(x), n, dm, _ptr(ids), _ptr(w), k, _ptr(w1), _ptr(w2),
                                                    ne, dh, ACT[act], int(single), _ptr(out)), "dense")
            return out
        r = None if rows is None else _i32(rows)
        cnt = n if r is None else len(r)
        out = np.empty((cnt, dm), np.float64)
        self.lib.orc_dense_given_routing(_ptr(x), n, dm, _ptr(ids), _ptr(w), k, _ptr(w1), _ptr(w2),
                                         None if w3 is None else _ptr(_f64(w3)), dh, ACT[act], int(single),
                                         _ptr(r), cnt, _ptr(out))
        return out

    def shared_experts(self, x, w1, w2, w3=None, gate=None, act="silu", out=None):
        """Shared-expert extension (not in the reference): out += g * sum_s FFN_s(x)
        (occ_oracle.c orc_shared_experts).  Port only."""
        if self.prefix == "ref_":
            raise ValueError("the reference has no shared experts (SPEC.md:9)")
        x, w1, w2 = _f64(x), _f64(w1), _f64(w2)
        n, dm = x.shape
        ns, _, dh = w1.shape
        out = np.zeros((n, dm), np.float64) if out is None else np.array(out, dtype=np.float64, copy=True)
        self.lib.orc_shared_experts(_ptr(x), n, dm, _ptr(w1), _ptr(w2), None if w3 is None else _ptr(_f64(w3)),
                                    ns, dh, ACT[act], None if gate is None else _ptr(_f64(gate)), _ptr(out))
        return out

    def prune_routing(self, scores, ids, w, plist, mode, budget, sim_values=None, own_score=False,
                      renormalize=True):
        s, w, ids, plist = _f64(scores), _f64(w), _i32(ids), _i32(plist)
        n, ne = s.shape
        k = ids.shape[1]
        nd = plist.shape[0]
        oi = np.empty_like(ids)
        ow = np.empty_like(w)
        if self.prefix == "ref_":
            sv = None if sim_values is None else _f64(sim_values)
            rc = self.lib.ref_prune_routing(_ptr(s), n, ne, _ptr(ids), _ptr(w), k, _ptr(plist), nd, PRUNE[mode],
                                            budget, _ptr(sv), int(own_score), int(renormalize), _ptr(oi), _ptr(ow))
        else:
            dev_of = np.empty(ne, np.int32)
            _check(self.lib.orc_expert_to_device(_ptr(plist), nd, ne // nd, _ptr(dev_of)), "placement")
            rank = None
            if sim_values is not None:
                rank = ranking_from_values(sim_values)
            rc = self.lib.orc_prune_routing(_ptr(s), n, ne, _ptr(ids), _ptr(w), k, _ptr(dev_of), nd, PRUNE[mode],
                                            budget, _ptr(rank), int(own_score), int(renormalize), _ptr(oi), _ptr(ow))
        _check(rc, "prune_routing")
        return oi, ow

    def similarity_table(self, logits):
        h = _f64(logits)
        n, ne = h.shape
        v = np.empty((ne, ne), np.float64)
        rk = np.empty((ne, ne - 1), np.int32)
        _check(self._fn("similarity_table")(_ptr(h), n, ne, _ptr(v), _ptr(rk)) or 0, "similarity")
        return v, rk


def ref_backward(x, ids, w, w1, w2, plist, sources, upstream, act="silu", single=False):
    """backward_vjps (backward.cpp:24-161) of the REFERENCE after a saving
    forward: returns (gx, gw1, gw2, g_routing_weights)."""
    L = ref_lib()
    x, w, w1, w2, up = _f64(x), _f64(w), _f64(w1), _f64(w2), _f64(upstream)
    ids, plist, sources = _i32(ids), _i32(plist), _i32(sources)
    n, dm = x.shape
    k = ids.shape[1]
    ne, _, dh = w1.shape
    gx = np.empty_like(x)
    gw1 = np.empty_like(w1)
    gw2 = np.empty_like(w2)
    gr = np.empty_like(w)
    rc = L.ref_backward(_ptr(x), n, dm, _ptr(ids), _ptr(w), k, _ptr(w1), _ptr(w2), ne, dh, _ptr(plist),
                        plist.shape[0], _ptr(sources), ACT[act], int(single), _ptr(up), _ptr(gx), _ptr(gw1),
                        _ptr(gw2), _ptr(gr))
    _check(rc, "backward_vjps")
    return gx, gw1, gw2, gr


def ranking_from_values(values):
    """Per-expert ranking (desc similarity, ties -> lower index), pruning.cpp:203-211."""
    v = np.asarray(values, np.float64)
    ne = v.shape[0]
    rk = np.empty((ne, ne - 1), np.int32)
    for i in range(ne):
        others = [j for j in range(ne) if j != i]
        others.sort(key=lambda j: (-v[i, j], j))
        rk[i] = others
    return rk


def _split_index(idx, rep, nd, per, sources):
    """Split the concatenated index outputs into per-source / per-device lists."""
    ntok = [int(np.sum(sources == s)) for s in range(nd)]
    out = {"dindex": [], "inbox": [], "cindex": []}
    pos = 0
    for s in range(nd):
        out["dindex"].append(idx["dindex"][pos:pos + nd * ntok[s]].reshape(nd, ntok[s]))
        pos += nd * ntok[s]
    ipos = cpos = 0
    for d in range(nd):
        rows = int(rep.per_device_rows[d])
        out["inbox"].append(np.stack([idx["inbox_token"][ipos:ipos + rows], idx["inbox_source"][ipos:ipos + rows],
                                      idx["inbox_slot"][ipos:ipos + rows]]))
        ipos += rows
        out["cindex"].append(idx["cindex"][cpos:cpos + per * rows].reshape(per, rows))
        cpos += per * rows
    return out


class Port(_Backend):
    prefix = "orc_"

    def __init__(self):
        super().__init__()
        self.lib = port_lib()


class Ref(_Backend):
    prefix = "ref_"

    def __init__(self):
        super().__init__()
        self.lib = ref_lib()


def seed_streams(seed: int):
    """cli.cpp:248-251: master Rng -> token, gate, expert seeds."""
    m = Rng(seed)
    return m.next(), m.next(), m.next()


def synthetic_layer(seed, n, dm, dh, ne, single=True, gated=False):
    """Reference CLI inputs (cli.cpp:248-256, :271): x, experts (w1 then w2
    per expert, core.cpp:47-50; w3 after w2 for the gated extension), gate."""
    ts, gs, es = seed_streams(seed)
    x = Rng(ts).random_matrix(n, dm, single)
    er = Rng(es)
    w1 = np.empty((ne, dm, dh))
    w2 = np.empty((ne, dh, dm))
    w3 = np.empty((ne, dm, dh)) if gated else None
    for e in range(ne):
        w1[e] = er.random_matrix(dm, dh, single)
        w2[e] = er.random_matrix(dh, dm, single)
        if gated:
            w3[e] = er.random_matrix(dm, dh, single)
    g = Rng(gs).random_matrix(ne, dm, single)
    return x, g, w1, w2, w3


def _u16(t):
    """bf16 storage (torch.bfloat16 tensor or uint16 array) -> contiguous uint16 numpy."""
    if t is None:
        return None
    if hasattr(t, "view") and hasattr(t, "dtype") and str(t.dtype) == "torch.bfloat16":
        import torch
        return np.ascontiguousarray(t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16))
    return np.ascontiguousarray(t, dtype=np.uint16)


def dense_rows_bf16(x, ids, w, w1, w2, rows, act="swiglu", w3=None, shared=None, threads=8):
    """dense_given_routing (+ shared experts) in fp64 for the sampled `rows`,
    operands in bf16 storage (occ_oracle.c orc_dense_rows_bf16): the
    full-size value oracle of the BASELINE layers.  ids [n, k] int32, w [n, k]
    f32 (the weights the layer ran with); w1/w3 [E, D, F], w2 [E, F, D];
    shared = dict(w1, w2, w3=None, gate=None) with [S, D, F_s] / [S, F_s, D] /
    [D].  Row chunks run on `threads` host threads (ctypes drops the GIL).
    Returns [len(rows), D] float64."""
    import threading
    L = port_lib()
    xu, w1u, w2u, w3u = _u16(x), _u16(w1), _u16(w2), _u16(w3)
    ids = _i32(ids)
    wf = np.ascontiguousarray(w, dtype=np.float32)
    n, dm = xu.shape
    k = ids.shape[1]
    ne, _, dh = w1u.shape
    ns, dhs, s1, s2, s3, sg = 0, 0, None, None, None, None
    if shared is not None:
        s1, s2 = _u16(shared["w1"]), _u16(shared["w2"])
        s3, sg = _u16(shared.get("w3")), _u16(shared.get("gate"))
        ns, dhs = s1.shape[0], s1.shape[2]
    rows = _i32(rows)
    out = np.empty((len(rows), dm), np.float64)
    chunks = [c for c in np.array_split(np.arange(len(rows)), max(1, min(threads, len(rows)))) if len(c)]
    gated = w3u is not None
    a = ACT["silu" if gated else act]

    def run(c):
        sub = np.ascontiguousarray(rows[c])
        o = np.empty((len(sub), dm), np.float64)
        L.orc_dense_rows_bf16(_ptr(xu), n, dm, _ptr(ids), _ptr(wf), k, ne, _ptr(w1u), _ptr(w2u), _ptr(w3u), dh, a,
                              ns, _ptr(s1), _ptr(s2), _ptr(s3), dhs, _ptr(sg), _ptr(sub), len(sub), _ptr(o))
        out[c] = o

    ts = [threading.Thread(target=run, args=(c,)) for c in chunks]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out
