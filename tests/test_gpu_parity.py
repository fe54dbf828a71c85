"""GPU parity: the sm_100a path (through the C-ABI) against the reference
compiled from its own sources (oracle/_ref) and the C restatement (oracle/).

Bars: bit-exact for routing ids/weights from fp64
scores, BRIM0/BRIM1 indices, exchange records, histogram, pruning and
placement; layer outputs (bf16 storage, fp32 accumulation) within
max_rel_error <= 1e-2 of the reference's fp64 result on identical
bf16-representable inputs (max|a-b| / max|b|, matrix.cpp:52-60).
"""
import numpy as np
import pytest
import torch

import paper_2505_13345_b200 as occ
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-2


def ref():
    return O.Ref() if O.ref_available() else O.Port()


def bf16_round(a):
    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy()


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def make_layer_inputs(seed, n, dm, dh, ne, gated=False):
    """Reference-seeded uniforms, weights scaled by 1/sqrt(fan_in), all
    rounded to bf16 so the device and the oracle see identical values."""
    x, g, w1, w2, w3 = O.synthetic_layer(seed, n, dm, dh, ne, single=True, gated=gated)
    x = bf16_round(x)
    g = bf16_round(g)
    w1 = bf16_round(w1 / np.sqrt(dm))
    w2 = bf16_round(w2 / np.sqrt(dh))
    w3 = bf16_round(w3 / np.sqrt(dm)) if gated else None
    return x, g, w1, w2, w3


def random_routing(n, ne, k, rng):
    ids = np.stack([rng.permutation(ne)[:k] for _ in range(n)]).astype(np.int32)
    w = rng.uniform(0.05, 1.0, size=(n, k))
    w = -np.sort(-w, axis=1)
    w = w / w.sum(1, keepdims=True)
    return ids, w


def cuda(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.to(dtype) if dtype is not None else t


# ------------------------------------------------------------------ routing --

@pytest.mark.parametrize("e,k", [(4, 2), (8, 2), (16, 5), (64, 8), (60, 4), (8, 8)])
@pytest.mark.parametrize("renorm", [True, False])
def test_topk_route_bit_exact(e, k, renorm):
    rng = np.random.default_rng(e * 31 + k)
    s = rng.uniform(size=(257, e))
    s[::7, 1] = s[::7, 0]            # exact ties -> lower index first (routing.cpp:71-74)
    s[::11, :] = 0.25                # fully tied rows
    ids, w = occ.topk_route(cuda(s), k, renorm)
    ri, rw = ref().topk_route(s, k, renorm)
    assert np.array_equal(ids.cpu().numpy(), ri)
    assert np.array_equal(w.cpu().numpy(), rw)  # bit-exact doubles


def test_topk_golden_vectors():
    # test_routing.cpp:64-99
    ids, _ = occ.topk_route(cuda(np.array([[0.1, 0.4, 0.3, 0.2]])), 4, False)
    assert ids.cpu().tolist() == [[1, 2, 3, 0]]
    ids, _ = occ.topk_route(cuda(np.array([[0.1, 0.4, 0.4, 0.1]])), 2, False)
    assert ids.cpu().tolist() == [[1, 2]]
    ids, w = occ.topk_route(cuda(np.array([[0.7, 0.1, 0.15, 0.05]])), 2, True)
    assert ids.cpu().tolist() == [[0, 2]]
    assert abs(w[0, 0].item() - 0.7 / 0.85) < 1e-15 and abs(w[0, 1].item() - 0.15 / 0.85) < 1e-15


def test_gate_scores_f64():
    x, g, *_ = O.synthetic_layer(21, 300, 48, 8, 16, single=False)
    s = occ.gate_scores_f64(cuda(x), cuda(g)).cpu().numpy()
    rs = ref().gate_scores(x, g)
    # logits sequential and FMA-free, softmax with the port of glibc's exp:
    # the scores are the reference's doubles bit for bit
    assert np.array_equal(s, rs)
    ids, _ = occ.topk_route(cuda(s), 4)
    ri, _ = ref().topk_route(rs, 4)
    assert np.array_equal(ids.cpu().numpy(), ri)


# (E, k, N_d, D, tokens, prune): C1, OLMoE at its full 65,536 tokens, Qwen-like
# 60 experts with router-score and similarity pruning to <= 2 devices.
EXACT_ROUTER_CASES = [(8, 2, 2, 512, 2048, None), (64, 8, 8, 2048, 65536, None),
                      (60, 4, 4, 2048, 4096, ("router", 2)), (60, 4, 4, 2048, 4096, ("similarity", 2)),
                      (64, 6, 8, 2048, 4096, ("router", 3))]


@pytest.mark.parametrize("ne,k,nd,dm,n,prune", EXACT_ROUTER_CASES)
def test_exact_router_bit_exact_from_raw_x(ne, k, nd, dm, n, prune):
    """forward_expert_parallel's routing (pipeline.cpp:509-512) from the raw
    bf16 tokens and gate: occ_route_exact's ids, fp64 weights and fp64 softmax
    scores equal gate_scores + topk_route (+ prune_routing) of the reference
    compiled from its own sources, bit for bit (routing.cpp:33-84,
    pruning.cpp:141-163)."""
    x, g, *_ = make_layer_inputs(17 + ne, n, dm, 8, ne)
    plist = np.random.default_rng(ne).permutation(ne).reshape(nd, ne // nd).astype(np.int32)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, 64),
                                    occ.Placement([list(map(int, r)) for r in plist]))
    R = ref()
    rs = R.gate_scores(x, g)
    ri, rw = R.topk_route(rs, k)
    spec = None
    if prune is not None:
        mode, budget = prune
        sim = None
        if mode == "similarity":
            sim = R.similarity_table(x[:512] @ g.T)[0]
            spec = occ.PruneSpec(mode, budget, table=sim)
        else:
            spec = occ.PruneSpec(mode, budget)
        ri, rw = R.prune_routing(rs, ri, rw, plist, mode, budget, sim_values=sim)
    ids, w, sc = layer.route_exact(cuda(x, torch.bfloat16), cuda(g, torch.bfloat16), prune=spec, want_scores=True)
    assert np.array_equal(sc.cpu().numpy(), rs)
    assert np.array_equal(ids.cpu().numpy(), ri)
    assert np.array_equal(w.cpu().numpy(), rw)
    # the layer's exact router mode routes with exactly these ids (weights in f32)
    layer.set_router_mode("exact")
    ids2, w2 = layer.route(cuda(x, torch.bfloat16), cuda(g, torch.bfloat16), prune=spec)
    assert np.array_equal(ids2.cpu().numpy(), ri)
    assert np.array_equal(w2.cpu().numpy(), rw.astype(np.float32))


def test_forward_expert_parallel_exact_router_vs_reference():
    """forward_expert_parallel (pipeline.cpp:503-517) end to end in the exact
    router mode at the C1 shape, against the reference's own
    forward_expert_parallel-equivalent (gate_scores + topk_route +
    forward_given_routing): identical CommReport (it depends only on the
    bit-exact routing) and outputs within the bf16 tolerance."""
    ne, k, nd, dm, dh, n = 8, 2, 2, 512, 1024, 512
    x, g, w1, w2, _ = make_layer_inputs(1, n, dm, dh, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    layer.set_router_mode("exact")
    out = layer.forward_expert_parallel(cuda(x, torch.bfloat16), cuda(g, torch.bfloat16))
    R = ref()
    ri, rw = R.topk_route(R.gate_scores(x, g), k)
    want, rep = R.forward_given_routing(x, ri, rw, w1, w2, np.arange(ne, dtype=np.int32).reshape(nd, -1),
                                        act="silu", single=False, bytes_per_scalar=2)
    got_rep = layer.comm_report(bytes_per_scalar=2)
    assert got_rep.mean_replicas == rep.mean_replicas
    assert got_rep.cross_device_bytes == rep.cross_device_bytes
    assert rel_err(out.double().cpu().numpy(), want) <= TOL


def test_production_router_matches_reference_ids():
    n, dm, ne, k = 2048, 512, 64, 8
    x, g, *_ = make_layer_inputs(5, n, dm, 8, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, 8, dm, 64))
    ids, w, sc = layer.route(cuda(x, torch.bfloat16), cuda(g, torch.bfloat16), want_scores=True)
    rs = ref().gate_scores(x, g)
    ri, rw = ref().topk_route(rs, k)
    ids = ids.cpu().numpy()
    mism = np.any(ids != ri, axis=1)
    # a flipped selection is only legal at a numerical near-tie of the reference scores
    for t in np.nonzero(mism)[0]:
        a = set(ids[t]) ^ set(ri[t])
        vals = sorted(rs[t, list(a)])
        assert vals[-1] - vals[0] < 1e-5 * rs[t].max(), (t, vals)
    assert mism.mean() < 0.01
    ok = ~mism
    assert np.max(np.abs(w.cpu().numpy()[ok] - rw[ok])) < 1e-5
    assert np.max(np.abs(sc.cpu().numpy() - rs)) < 1e-5


# --------------------------------------------------------------- dispatch ----

@pytest.mark.parametrize("nd,ne,k", [(1, 4, 2), (2, 4, 2), (2, 8, 2), (4, 8, 3), (8, 64, 8), (4, 16, 5)])
@pytest.mark.parametrize("srcmode", ["roundrobin", "random", "single"])
def test_dispatch_index_bit_exact(nd, ne, k, srcmode):
    rng = np.random.default_rng(nd * 100 + ne + k)
    n = 777
    ids, w = random_routing(n, ne, k, rng)
    src = {"roundrobin": np.arange(n) % nd, "random": rng.integers(0, nd, n), "single": np.zeros(n)}[srcmode]
    src = src.astype(np.int32)
    plist = np.arange(ne, dtype=np.int32).reshape(nd, ne // nd)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, 8, 8))
    brim0, counts = layer.build_dispatch_index(cuda(ids), cuda(src))
    brim0 = brim0.cpu().numpy()
    # reference: build_dispatch_index per source over its ascending token list
    R = O.ref_lib() if O.ref_available() else None
    pos = 0
    for s in range(nd):
        toks = np.nonzero(src == s)[0].astype(np.int32)
        want, nsfd = _ref_dispatch(ids, w, plist, toks, ne)
        got = brim0[pos:pos + nd * len(toks)].reshape(nd, len(toks))
        pos += nd * len(toks)
        assert np.array_equal(got, want), f"source {s}"
        assert counts.cpu().numpy()[s].sum() == nsfd


def _ref_dispatch(ids, w, plist, toks, ne):
    import ctypes as C
    nd = plist.shape[0]
    entries = np.empty(nd * len(toks), np.int32)
    nsfd = C.c_int()
    if O.ref_available():
        L = O.ref_lib()
        rc = L.ref_build_dispatch_index(O._ptr(ids), O._ptr(np.ascontiguousarray(w)), ids.shape[0], ids.shape[1],
                                        O._ptr(plist), nd, ne, O._ptr(toks), len(toks), O._ptr(entries), C.byref(nsfd))
        assert rc == 0
        return entries.reshape(nd, len(toks)), nsfd.value
    L = O.port_lib()
    dev_of = np.empty(ne, np.int32)
    L.orc_expert_to_device(O._ptr(plist), nd, ne // nd, O._ptr(dev_of))
    v = L.orc_build_dispatch_index(O._ptr(ids), ids.shape[1], O._ptr(dev_of), nd, O._ptr(toks), len(toks),
                                   O._ptr(entries))
    return entries.reshape(nd, len(toks)), v


def test_dispatch_golden_worked_example():
    # pipeline.hpp:17-27 / test_pipeline.cpp:90-95
    ids = np.array([[0, 1], [0, 2], [2, 3]], np.int32)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(4, 2, 2, 8, 8))
    brim0, counts = layer.build_dispatch_index(cuda(ids), cuda(np.zeros(3, np.int32)))
    assert brim0.cpu().tolist()[:6] == [0, 1, -1, -1, 2, 3]


# ---------------------------------------------------------------- forward ---

FWD_CASES = [
    # (ne, k, nd, dm, dh, act, n, placement)
    (8, 2, 2, 64, 128, "silu", 300, "trivial"),
    (8, 3, 4, 64, 64, "identity", 257, "trivial"),
    (8, 2, 1, 128, 256, "relu", 200, "trivial"),
    (16, 4, 4, 96, 160, "silu", 513, "shuffled"),
    (64, 8, 8, 128, 64, "silu", 400, "shuffled"),
    (4, 4, 2, 32, 32, "silu", 50, "trivial"),
    (8, 1, 8, 64, 64, "silu", 129, "trivial"),
    (8, 2, 2, 40, 72, "silu", 100, "shuffled"),       # D, F multiples of 8 only (TMA zero-fills the K tail)
    (8, 2, 2, 1024, 1800, "relu", 300, "trivial"),   # wide super-tiles with a ragged last N block
    # maximum sizes of the device path: E = 256 with 64 experts per device, top-k = 64, 64 devices
    (256, 16, 4, 64, 64, "silu", 300, "shuffled"),
    (128, 64, 2, 64, 64, "relu", 100, "shuffled"),
    (64, 64, 64, 32, 32, "identity", 70, "shuffled"),
]


def _placement(ne, nd, kind, seed=0):
    if kind == "trivial":
        return np.arange(ne, dtype=np.int32).reshape(nd, ne // nd)
    rng = np.random.default_rng(seed + ne)
    return rng.permutation(ne).astype(np.int32).reshape(nd, ne // nd)


@pytest.mark.parametrize("ne,k,nd,dm,dh,act,n,pk", FWD_CASES)
@pytest.mark.parametrize("dedup", [True, False])
def test_forward_given_routing(ne, k, nd, dm, dh, act, n, pk, dedup):
    x, g, w1, w2, _ = make_layer_inputs(ne * 7 + k, n, dm, dh, ne)
    rng = np.random.default_rng(n)
    ids, w = random_routing(n, ne, k, rng)
    w = w.astype(np.float32).astype(np.float64)  # f32 routing weights on the device
    plist = _placement(ne, nd, pk)
    src = (np.arange(n) % nd).astype(np.int32)
    want, rep, idx = ref().forward_given_routing(x, ids, w, w1, w2, plist, src, act=act, single=False,
                                                 bytes_per_scalar=2, want_index=True)
    cfg = occ.MoEConfig(ne, k, nd, dm, dh, activation=act, dedup=dedup)
    layer = occ.ExpertParallelLayer(cfg, occ.Placement([list(r) for r in plist]))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    out = layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32), cuda(src))
    got = out.double().cpu().numpy()
    err = rel_err(got, want)
    assert err <= TOL, err
    r = layer.comm_report(bytes_per_scalar=2)
    assert r.mean_replicas == rep.mean_replicas
    assert r.intra_share == rep.intra_share and r.inter_share == rep.inter_share
    if dedup:
        assert r.cross_device_bytes == rep.cross_device_bytes
        assert r.per_device_token_counts == [rep.per_device_rows[d] for d in range(nd)]
        tok, srcs, slot, cix, rows = layer.saved_index()
        tok, srcs, slot, cix = (t.cpu().numpy() for t in (tok, srcs, slot, cix))
        pos = cpos = 0
        P = ne // nd
        for d in range(nd):
            R = rows[d]
            assert np.array_equal(tok[pos:pos + R], idx["inbox"][d][0])
            assert np.array_equal(srcs[pos:pos + R], idx["inbox"][d][1])
            assert np.array_equal(slot[pos:pos + R], idx["inbox"][d][2])
            assert np.array_equal(cix[cpos:cpos + P * R].reshape(P, R), idx["cindex"][d])
            pos += R
            cpos += P * R
    else:
        assert r.n_sfd == n * k


@pytest.mark.parametrize("ne,k,nd,dm,dh,n", [(8, 2, 2, 128, 128, 300), (16, 4, 4, 64, 256, 257),
                                            (8, 2, 1, 256, 384, 1000)])
def test_forward_swiglu(ne, k, nd, dm, dh, n):
    x, g, w1, w2, w3 = make_layer_inputs(ne + dh, n, dm, dh, ne, gated=True)
    rng = np.random.default_rng(3)
    ids, w = random_routing(n, ne, k, rng)
    w = w.astype(np.float32).astype(np.float64)
    plist = _placement(ne, nd, "trivial")
    want, _ = O.Port().forward_given_routing(x, ids, w, w1, w2, plist, None, act="silu", single=False, w3=w3)
    # the SwiGLU restatement itself is pinned against an independent torch fp64 computation
    xt = torch.from_numpy(x)
    dense = torch.zeros_like(xt)
    for j in range(k):
        e = torch.from_numpy(ids[:, j]).long()
        a = torch.einsum("nd,ndf->nf", xt, torch.from_numpy(w1)[e])
        b = torch.einsum("nd,ndf->nf", xt, torch.from_numpy(w3)[e])
        h = torch.nn.functional.silu(a) * b
        dense += torch.from_numpy(w[:, j:j + 1]) * torch.einsum("nf,nfd->nd", h, torch.from_numpy(w2)[e])
    assert rel_err(want, dense.numpy()) < 1e-12
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="swiglu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16))
    out = layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    assert rel_err(out.double().cpu().numpy(), want) <= TOL


def make_shared(ns, dm, dh, gated, seed=0, gate=True):
    rng = np.random.default_rng(seed + 100)
    s1 = bf16_round(rng.uniform(-1, 1, (ns, dm, dh)) / np.sqrt(dm))
    s3 = bf16_round(rng.uniform(-1, 1, (ns, dm, dh)) / np.sqrt(dm)) if gated else None
    s2 = bf16_round(rng.uniform(-1, 1, (ns, dh, dm)) / np.sqrt(dh * ns))
    sg = bf16_round(rng.uniform(-1, 1, dm) * (2.0 / np.sqrt(dm))) if gate else None
    return s1, s2, s3, sg


@pytest.mark.parametrize("ne,k,nd,dm,dh,act,n,ns,dhs,gate", [
    (8, 2, 2, 128, 128, "swiglu", 300, 2, 128, False),   # DeepSeek-style: 2 shared experts, no gate
    (16, 4, 4, 128, 256, "swiglu", 513, 1, 512, True),   # Qwen-style: one wide shared expert + sigmoid gate
    (8, 2, 1, 64, 128, "silu", 100, 1, 64, True),        # 2-matrix experts
    (8, 2, 2, 256, 128, "relu", 1, 3, 96, False),        # one token, 3 shared experts of width 96
])
def test_forward_shared_experts(ne, k, nd, dm, dh, act, n, ns, dhs, gate):
    """Routed layer + shared experts (DeepSeek / Qwen extension) against the
    oracle: forward_given_routing restatement + orc_shared_experts."""
    gated = act == "swiglu"
    x, g, w1, w2, w3 = make_layer_inputs(ne + n + ns, n, dm, dh, ne, gated=gated)
    ids, w = random_routing(n, ne, k, np.random.default_rng(ns))
    w = w.astype(np.float32).astype(np.float64)
    plist = _placement(ne, nd, "shuffled", seed=1)
    s1, s2, s3, sg = make_shared(ns, dm, dhs, gated, seed=n, gate=gate)
    a = "silu" if gated else act
    want, _ = O.Port().forward_given_routing(x, ids, w, w1, w2, plist, None, act=a, single=False, w3=w3)
    want = O.Port().shared_experts(x, s1, s2, w3=s3, gate=sg, act=a, out=want)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act),
                                    occ.Placement([list(p) for p in plist]))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16) if gated else None)
    layer.load_shared_experts(cuda(s1, torch.bfloat16), cuda(s2, torch.bfloat16),
                              cuda(s3, torch.bfloat16) if gated else None,
                              cuda(sg, torch.bfloat16) if gate else None)
    out = layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    assert rel_err(out.double().cpu().numpy(), want) <= TOL
    # detaching the shared experts gives the routed layer back
    layer.load_shared_experts(cuda(s1[:0], torch.bfloat16), cuda(s2[:0], torch.bfloat16))
    plain, _ = O.Port().forward_given_routing(x, ids, w, w1, w2, plist, None, act=a, single=False, w3=w3)
    out2 = layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    assert rel_err(out2.double().cpu().numpy(), plain) <= TOL


def test_forward_bit_identical_reruns():
    # test_pipeline.cpp:490-509: deterministic (no atomics on the data path)
    ne, k, nd, dm, dh, n = 16, 4, 4, 128, 256, 1000
    x, g, w1, w2, _ = make_layer_inputs(79, n, dm, dh, ne)
    ids, w = random_routing(n, ne, k, np.random.default_rng(1))
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    args = (cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    a = layer.forward_given_routing(*args).clone()
    b = layer.forward_given_routing(*args)
    assert torch.equal(a, b)


def test_placement_changes_communication_not_values():
    # test_pipeline.cpp:447-462
    ne, k, nd, dm, dh, n = 8, 3, 4, 64, 128, 300
    x, g, w1, w2, _ = make_layer_inputs(77, n, dm, dh, ne)
    ids, w = random_routing(n, ne, k, np.random.default_rng(2))
    outs = []
    for pl in ([[0, 1], [2, 3], [4, 5], [6, 7]], [[7, 0], [3, 5], [1, 6], [2, 4]]):
        layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"), occ.Placement(pl))
        layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
        outs.append(layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32)).double())
    assert rel_err(outs[0].cpu().numpy(), outs[1].cpu().numpy()) < 5e-3


def test_invalid_routing_raises():
    layer = occ.ExpertParallelLayer(occ.MoEConfig(8, 2, 2, 64, 64))
    layer.load_experts(torch.zeros(8, 64, 64, device="cuda"), torch.zeros(8, 64, 64, device="cuda"))
    x = torch.zeros(4, 64, dtype=torch.bfloat16, device="cuda")
    w = torch.full((4, 2), 0.5, device="cuda")
    with pytest.raises(occ.RoutingError):
        layer.forward_given_routing(x, cuda(np.array([[0, 0]] * 4, np.int32)), w)  # duplicate id
    with pytest.raises(occ.RoutingError):
        layer.forward_given_routing(x, cuda(np.array([[0, 9]] * 4, np.int32)), w)  # out of range
    with pytest.raises(occ.RoutingError):
        layer.forward_given_routing(x, cuda(np.array([[0, 1]] * 4, np.int32)), torch.zeros(4, 2, device="cuda"))
    with pytest.raises(occ.ShapeError):
        layer.forward_given_routing(x, cuda(np.array([[0, 1]] * 4, np.int32)), w,
                                    cuda(np.array([0, 1, 2, 0], np.int32)))


def test_empty_batch():
    layer = occ.ExpertParallelLayer(occ.MoEConfig(8, 2, 2, 64, 64))
    layer.load_experts(torch.zeros(8, 64, 64, device="cuda"), torch.zeros(8, 64, 64, device="cuda"))
    out = layer.forward_given_routing(torch.zeros(0, 64, dtype=torch.bfloat16, device="cuda"),
                                      torch.zeros(0, 2, dtype=torch.int32, device="cuda"),
                                      torch.zeros(0, 2, device="cuda"))
    assert out.shape == (0, 64)


# ------------------------------------------------------ histogram / prune ---

@pytest.mark.parametrize("ne,k", [(3, 2), (12, 4), (64, 8), (60, 4), (8, 1)])
def test_histogram_bit_exact(ne, k):
    rng = np.random.default_rng(ne + k)
    ids, _ = random_routing(5000, ne, k, rng)
    got = occ.build_collab_graph(cuda(ids), ne).cpu().numpy()
    assert np.array_equal(got, ref().accumulate_collab(ids, ne))
    # accumulate: a second batch adds in place
    c = occ.build_collab_graph(cuda(ids), ne)
    occ.accumulate_collab(c, cuda(ids[:100]))
    assert np.array_equal(c.cpu().numpy(), ref().accumulate_collab(ids[:100], ne, got))


@pytest.mark.parametrize("mode", ["router", "similarity"])
@pytest.mark.parametrize("own", [False, True])
@pytest.mark.parametrize("ne,nd,k,budget", [(8, 4, 2, 1), (16, 4, 4, 2), (64, 8, 8, 2), (64, 8, 6, 3), (60, 4, 4, 2),
                                           # maximum sizes; (256, 16, 40, 2) cannot fit top-40 on 2 devices
                                           (256, 4, 64, 1), (256, 64, 16, 4), (128, 2, 64, 2), (256, 16, 40, 2)])
def test_prune_routing_bit_exact(mode, own, ne, nd, k, budget):
    if mode == "router" and own:
        pytest.skip("weight policy only applies to similarity replacement")
    rng = np.random.default_rng(ne * nd + k)
    s = rng.uniform(size=(300, ne))
    s = s / s.sum(1, keepdims=True)
    ri, rw = ref().topk_route(s, k)
    plist = _placement(ne, nd, "shuffled")
    sim, _ = ref().similarity_table(np.log(s))
    spec = occ.PruneSpec(mode, budget, sim if mode == "similarity" else None, "own" if own else "inherit")
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, 8, 8), occ.Placement([list(r) for r in plist]))
    try:
        want = ref().prune_routing(s, ri, rw, plist, mode, budget, sim_values=sim if mode == "similarity" else None,
                                   own_score=own)
    except O.OracleError as e:
        assert e.code == 5
        with pytest.raises(occ.CapacityError):
            layer.prune_routing(cuda(s), cuda(ri), cuda(rw), spec)
        return
    gi, gw = layer.prune_routing(cuda(s), cuda(ri), cuda(rw), spec)
    assert np.array_equal(gi.cpu().numpy(), want[0])
    assert np.array_equal(gw.cpu().numpy(), want[1])


def test_prune_golden_vectors():
    # test_pruning.cpp:73-79, :99-112
    layer = occ.ExpertParallelLayer(occ.MoEConfig(4, 2, 2, 8, 8))
    s = np.array([[0.3, 0.05, 0.5, 0.15]])
    ids, w = occ.topk_route(cuda(s), 2, False)
    gi, gw = layer.prune_routing(cuda(s), ids, w, occ.PruneSpec("router", 1))
    assert gi.cpu().tolist() == [[2, 3]]
    table = np.array([[1.0, 0.9, 0.1, 0.5], [0.9, 1.0, 0.2, 0.3], [0.1, 0.2, 1.0, 0.8], [0.5, 0.3, 0.8, 1.0]])
    ids = cuda(np.array([[2, 0]], np.int32))
    gi, gw = layer.prune_routing(cuda(s), ids, cuda(np.array([[0.5, 0.3]])), occ.PruneSpec("similarity", 1, table))
    assert gi.cpu().tolist() == [[2, 3]]


def test_router_with_pruning_respects_budget():
    ne, k, nd, dm, n = 64, 8, 8, 256, 1000
    x, g, *_ = make_layer_inputs(9, n, dm, 8, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, 64))
    ids, w = layer.route(cuda(x, torch.bfloat16), cuda(g, torch.bfloat16), occ.PruneSpec("router", 2))
    dev = ids.cpu().numpy() // (ne // nd)
    assert max(len(set(r)) for r in dev) <= 2
    assert torch.allclose(w.sum(1), torch.ones(n, device="cuda"), atol=1e-5)


@pytest.mark.parametrize("ne,k,nd,budget,renorm", [(64, 8, 8, 2, True), (60, 4, 4, 2, True), (16, 4, 4, 1, False),
                                                   (128, 6, 8, 3, True), (32, 2, 2, 1, True),
                                                   (128, 64, 2, 1, True), (256, 16, 4, 2, True), (256, 64, 8, 4, False)])
def test_router_epilogue_pruning_matches_oracle(ne, k, nd, budget, renorm):
    """Router-score pruning fused into the tcgen05 router's epilogue equals
    prune_routing (pruning.cpp:35-64, oracle restatement) applied to the same
    fp32 softmax rows, id for id; weights to fp32 rounding."""
    dm, n = 256, 2000
    x, g, *_ = make_layer_inputs(ne + k, n, dm, 8, ne)
    plist = _placement(ne, nd, "shuffled", seed=budget)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, 64, renormalize=renorm),
                                    occ.Placement([list(r) for r in plist]))
    xs, gs = cuda(x, torch.bfloat16), cuda(g, torch.bfloat16)
    ids, w = layer.route(xs, gs, occ.PruneSpec("router", budget))
    _, _, sc = layer.route(xs, gs, want_scores=True)
    s64 = sc.double().cpu().numpy()
    ids0, w0 = O.Port().topk_route(s64, k, renorm)
    want_ids, want_w = O.Port().prune_routing(s64, ids0, w0, plist, "router", budget, renormalize=renorm)
    assert np.array_equal(ids.cpu().numpy(), want_ids)
    assert np.allclose(w.double().cpu().numpy(), want_w, rtol=2e-6, atol=1e-7)


# --------------------------------------------------------- full-size checks --

def test_c1_full_size_vs_reference_rows():
    """C1 (8 experts top-2, d=512, d_ff=1024, 2048 tokens, 2 EP ranks):
    gate -> top-2 on the device, full forward; outputs compared on sampled
    rows against the reference dense oracle (rows are independent given
    routing, pipeline.cpp:548-560); indices compared at full size."""
    ne, k, nd, dm, dh, n = 8, 2, 2, 512, 1024, 2048
    x, g, w1, w2, _ = make_layer_inputs(1, n, dm, dh, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    xs = cuda(x, torch.bfloat16)
    ids, w = layer.route(xs, cuda(g, torch.bfloat16))
    out = layer.forward_given_routing(xs, ids, w).double().cpu().numpy()
    idn, wn = ids.cpu().numpy(), w.double().cpu().numpy()
    rows = np.arange(0, n, 8)
    want = O.Port().dense_given_routing(x, idn, wn, w1, w2, act="silu", single=False, rows=rows)
    assert rel_err(out[rows], want) <= TOL
    rep = layer.comm_report(bytes_per_scalar=2)
    P = O.Port()
    plist = np.arange(ne, dtype=np.int32).reshape(nd, ne // nd)
    # width-1 replay gives the reference's exact indices/accounting at full size
    _, rr = P.forward_given_routing(np.ones((n, 1)) * 0.5, idn, wn, np.ones((ne, 1, 8)), np.ones((ne, 8, 1)),
                                    plist, None, act="identity", single=False, bytes_per_scalar=2)
    assert rep.mean_replicas == rr.mean_replicas
    assert rep.crossing_rows == rr.crossing_rows
    assert rep.per_device_token_counts == [rr.per_device_rows[d] for d in range(nd)]


@pytest.mark.parametrize("name,ne,k,nd,n,prune", [
    ("olmoe", 64, 8, 8, 65536, None),          # BASELINE config 4 token count, EP=8
    ("deepseek", 64, 6, 8, 16384, None),       # config 3
    ("qwen_ep4_budget2", 60, 4, 4, 16384, 2),  # config 5 with collaboration pruning
    ("mixtral", 8, 2, 8, 16384, None),         # config 2
])
def test_full_size_indices_vs_reference(name, ne, k, nd, n, prune):
    """Integer parity at the BASELINE token counts: BRIM0 of every source,
    inbox records, BRIM1 and CommReport against the reference's own
    forward_given_routing replayed at width 1 (indices do not depend on D or
    F); routing from the fp64 top-k (+ pruning) path, itself
    bit-exact with the reference."""
    rng = np.random.default_rng(ne * 1000 + k)
    scores = rng.dirichlet(np.ones(ne), size=n)  # softmax-like rows
    plist = _placement(ne, nd, "shuffled", seed=k)
    ids, w = O.Port().topk_route(scores, k, True)
    if prune:
        ids, w = O.Port().prune_routing(scores, ids, w, plist, "router", prune)
    ids = ids.astype(np.int32)
    w = w.astype(np.float32).astype(np.float64)
    src = rng.integers(0, nd, n).astype(np.int32)
    _, rep, idx = ref().forward_given_routing(np.full((n, 1), 0.5), ids, w, np.ones((ne, 1, 8)),
                                              np.ones((ne, 8, 1)), plist, src, act="identity", single=False,
                                              bytes_per_scalar=2, want_index=True)
    dm, dh = 64, 128
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"),
                                    occ.Placement([list(r) for r in plist]))
    layer.load_experts(torch.zeros(ne, dm, dh, dtype=torch.bfloat16, device="cuda"),
                       torch.zeros(ne, dh, dm, dtype=torch.bfloat16, device="cuda"))
    brim0, counts = layer.build_dispatch_index(cuda(ids), cuda(src))
    brim0 = brim0.cpu().numpy()
    pos = 0
    for s_ in range(nd):
        want = idx["dindex"][s_]
        got = brim0[pos:pos + want.size].reshape(want.shape)
        pos += want.size
        assert np.array_equal(got, want), f"{name}: BRIM0 of source {s_}"
    x = torch.zeros(n, dm, dtype=torch.bfloat16, device="cuda")
    layer.forward_given_routing(x, cuda(ids), cuda(w, torch.float32), cuda(src))
    r = layer.comm_report(bytes_per_scalar=2)
    assert r.mean_replicas == rep.mean_replicas and r.crossing_rows == rep.crossing_rows
    assert r.intra_share == rep.intra_share and r.inter_share == rep.inter_share
    assert r.per_device_token_counts == [rep.per_device_rows[d] for d in range(nd)]
    tok, srcs, slot, cix, rows = layer.saved_index()
    tok, srcs, slot, cix = (t.cpu().numpy() for t in (tok, srcs, slot, cix))
    pos = cpos = 0
    P = ne // nd
    for d in range(nd):
        R = rows[d]
        assert np.array_equal(tok[pos:pos + R], idx["inbox"][d][0]), f"{name}: inbox tokens of device {d}"
        assert np.array_equal(srcs[pos:pos + R], idx["inbox"][d][1])
        assert np.array_equal(slot[pos:pos + R], idx["inbox"][d][2])
        assert np.array_equal(cix[cpos:cpos + P * R].reshape(P, R), idx["cindex"][d]), f"{name}: BRIM1 of device {d}"
        pos += R
        cpos += P * R


@pytest.mark.parametrize("chunks,mb", [(1, 1), (3, 1), (4, 1), (1, 2), (3, 2)])
def test_forward_host_pipeline_matches_device(chunks, mb):
    """occ_forward_host (pinned host in/out, chunked H2D/layer/D2H pipeline)
    gives bit-identical rows to the device-resident forward: rows are
    independent given routing and the kernels are order-deterministic."""
    ne, k, nd, dm, dh, n = 8, 2, 2, 256, 512, 1001
    x, g, w1, w2, _ = make_layer_inputs(5, n, dm, dh, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    xs = cuda(x, torch.bfloat16)
    gs = cuda(g, torch.bfloat16)
    want = layer.forward_expert_parallel(xs, gs).cpu()
    if mb > 1:  # the micro-batched forward inside the host pipeline
        layer.set_micro_batches(mb)
        layer.set_validate(False)
    xh = xs.cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    layer.forward_host(xh, gs, oh, chunks=chunks)
    torch.cuda.synchronize()
    assert torch.equal(oh, want)


def test_forward_host_graph_replay():
    """Validation off: occ_forward_host replays the layer as a CUDA graph per
    staging slot (captured once, re-captured when the batch shape or any
    workspace buffer changes); results stay bit-identical across calls,
    slots, new inputs, a batch-size change and a workspace regrow."""
    ne, k, nd, dm, dh = 8, 2, 2, 256, 512
    x, g, w1, w2, _ = make_layer_inputs(6, 1500, dm, dh, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    gs = cuda(g, torch.bfloat16)
    layer.set_validate(False)
    for n in (700, 700, 700, 300, 1500, 700):
        xs = cuda(x[:n], torch.bfloat16) * (1 + n % 7)  # new values each time
        want = layer.forward_expert_parallel(xs, gs).cpu()
        xh = xs.cpu().pin_memory()
        oh = torch.empty_like(xh).pin_memory()
        layer.forward_host(xh, gs, oh)
        torch.cuda.synchronize()
        assert torch.equal(oh, want), n


def test_forward_host_async_shrinking_batches():
    """wait=False with a batch size that shrinks and grows between calls (eager
    chunked path and graph replay): the two staging slots keep a fixed stride,
    so an in-flight call's inputs and outputs are never overwritten by the next
    call's copies (slot 1 used to start at n * D of the CURRENT
    call)."""
    ne, k, nd, dm, dh = 8, 2, 2, 256, 512
    x, g, w1, w2, _ = make_layer_inputs(9, 1200, dm, dh, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    gs = cuda(g, torch.bfloat16)
    for validate, chunks in ((True, 3), (False, 1), (False, 2)):
        layer.set_validate(validate)
        sizes = (1200, 900, 400, 1100, 250, 1200, 800)
        wants, hosts = [], []
        for i, n in enumerate(sizes):
            xs = cuda(x[:n], torch.bfloat16) * (1 + i % 5)
            wants.append(layer.forward_expert_parallel(xs, gs).cpu())
            hosts.append((xs.cpu().pin_memory(), torch.full((n, dm), float("nan"), dtype=torch.bfloat16).pin_memory()))
        torch.cuda.synchronize()
        for xh, oh in hosts:  # all enqueued back to back, no wait in between
            layer.forward_host(xh, gs, oh, chunks=chunks, wait=False)
        layer.host_wait()
        torch.cuda.synchronize()
        for i, ((xh, oh), want) in enumerate(zip(hosts, wants)):
            assert torch.equal(oh, want), (validate, chunks, i, sizes[i])


# ------------------------------------------- world_size > 1 (loopback) -----

@pytest.mark.parametrize("nd,ne,k,act,dedup,shared,peer", [(2, 8, 2, "silu", True, 0, False),
                                                           (4, 16, 4, "silu", True, 0, False),
                                                           (8, 64, 8, "relu", True, 0, False),
                                                           (4, 8, 3, "identity", False, 0, False),
                                                           (2, 8, 2, "swiglu", True, 0, False),
                                                           (4, 16, 4, "swiglu", True, 2, False),
                                                           (2, 8, 2, "relu", False, 1, False),
                                                           # fused exchange over peer memory
                                                           (2, 8, 2, "silu", True, 0, True),
                                                           (8, 64, 8, "relu", True, 0, True),
                                                           (4, 8, 3, "identity", False, 0, True),
                                                           (4, 16, 4, "swiglu", True, 2, True),
                                                           # maximum top-k, NCCL-free and peer
                                                           (2, 128, 64, "relu", True, 0, False),
                                                           (2, 128, 64, "silu", False, 0, True)])
@pytest.mark.parametrize("mb", [1, 2])
def test_multi_rank_forward_loopback(nd, ne, k, act, dedup, shared, peer, mb):
    """The world_size == N_d code path (per-rank plan, count all-gather, two
    variable all-to-alls, per-device BRIM1 + GEMMs + partial combine,
    combine) with the ranks as threads on one GPU, against the reference's
    single-process simulation with sources = owning rank; mb = 2 runs every
    forward as two micro-batches (the overlap path)."""
    import threading
    dm, dh = 128, 256
    n_per = [37, 64, 5, 100, 0, 64, 33, 1][:nd]
    n = sum(n_per)
    gated = act == "swiglu"
    x, g, w1, w2, w3 = make_layer_inputs(nd * 13 + k, n, dm, dh, ne, gated=gated)
    ids, w = random_routing(n, ne, k, np.random.default_rng(nd + k))
    w = w.astype(np.float32).astype(np.float64)
    plist = _placement(ne, nd, "shuffled", seed=nd)
    src = np.concatenate([np.full(c, r, np.int32) for r, c in enumerate(n_per)])
    if gated:
        want, rep = O.Port().forward_given_routing(x, ids, w, w1, w2, plist, src, act="silu", single=False, w3=w3,
                                                   bytes_per_scalar=2)
    else:
        want, rep = ref().forward_given_routing(x, ids, w, w1, w2, plist, src, act=act, single=False,
                                                bytes_per_scalar=2)
    if shared:  # shared experts at every source (extension), Qwen-style gate
        s1, s2, s3, sg = make_shared(shared, dm, 128, gated, seed=nd)
        want = O.Port().shared_experts(x, s1, s2, w3=s3, gate=sg, act="silu" if gated else act, out=want)
    outs = [None] * nd
    errs = []
    starts = np.concatenate([[0], np.cumsum(n_per)])
    key = np.random.default_rng().integers(1 << 30)
    # Ranks are threads sharing one GPU: a device-synchronising call on one
    # thread (cudaFree from a caching-allocator flush) while another rank's
    # arrival wait spins would stall until the wait times out, so all device
    # tensors are made up front and converted only after every rank is done.
    X = [cuda(x[starts[r]:starts[r + 1]], torch.bfloat16) for r in range(nd)]
    I = [cuda(ids[starts[r]:starts[r + 1]]) for r in range(nd)]
    Wt = [cuda(w[starts[r]:starts[r + 1]], torch.float32) for r in range(nd)]
    OUT = [torch.empty_like(X[r]) for r in range(nd)]
    done = threading.Barrier(nd)

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                cfg = occ.MoEConfig(ne, k, nd, dm, dh, activation=act, dedup=dedup)
                layer = occ.ExpertParallelLayer(cfg, occ.Placement([list(p) for p in plist]), world_size=nd, rank=r)
                loc = plist[r]
                layer.load_experts(cuda(w1[loc], torch.bfloat16), cuda(w2[loc], torch.bfloat16),
                                   cuda(w3[loc], torch.bfloat16) if gated else None)
                if shared:
                    layer.load_shared_experts(cuda(s1, torch.bfloat16), cuda(s2, torch.bfloat16),
                                              cuda(s3, torch.bfloat16) if gated else None, cuda(sg, torch.bfloat16))
                layer.comm_init_loopback(int(key))
                if peer:
                    layer.comm_enable_peer(128)
                if mb > 1:  # two micro-batches per forward: sibling handle + split communicator
                    layer.set_micro_batches(mb)
                for _rep in range(2 if peer else 1):  # peer mode: arrival flags advance per forward
                    layer.forward_given_routing(X[r], I[r], Wt[r], out=OUT[r])
                st.synchronize()
                rep_r = layer.comm_report(bytes_per_scalar=2)
                done.wait()
                outs[r] = (OUT[r].double().cpu().numpy(), rep_r)
        except Exception as e:  # surface thread failures
            errs.append(e)
            done.abort()

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(nd)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=120)
    assert not errs, errs
    got = np.concatenate([o[0] for o in outs])
    assert rel_err(got, want) <= TOL
    r0 = outs[0][1]
    if dedup:
        assert r0.cross_device_bytes == rep.cross_device_bytes
        assert r0.per_device_token_counts == [rep.per_device_rows[d] for d in range(nd)]


def test_loopback_peer_refused_under_lazy_loading():
    """Ranks as threads of one process share one context: with lazy kernel
    loading a rank's first launch of a kernel waits for another rank's
    spinning arrival wait, so the loopback peer exchange would stall until
    the wait's timeout.  occ_comm_enable_peer refuses it with a StateError
    that names CUDA_MODULE_LOADING=EAGER (checked in a fresh process)."""
    import os
    import subprocess
    import sys
    code = ("import paper_2505_13345_b200 as occ\n"
            "l = occ.ExpertParallelLayer(occ.MoEConfig(8, 2, 2, 128, 256), world_size=2, rank=0)\n"
            "l.comm_init_loopback(12345)\n"
            "try:\n    l.comm_enable_peer(16)\nexcept occ.StateError as e:\n    print('REFUSED', e)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_MODULE_LOADING="LAZY")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert "REFUSED" in out.stdout and "CUDA_MODULE_LOADING=EAGER" in out.stdout, out.stdout + out.stderr


# ------------------------------------------------------------------ backward --

@pytest.mark.parametrize("nd,ne,k,act,dedup,peer", [(2, 8, 2, "silu", True, False), (4, 16, 4, "relu", True, False),
                                                   (8, 64, 8, "silu", True, False), (4, 8, 3, "identity", False, False),
                                                   (8, 64, 8, "silu", True, True), (2, 8, 2, "relu", False, True),
                                                   (4, 16, 4, "swiglu", True, False)])
def test_multi_rank_backward_loopback(nd, ne, k, act, dedup, peer):
    """backward_vjps across world_size == N_d ranks (C4's EP=8 training step):
    the combine adjoint sent along the dispatch layout, expert-side adjoints on
    each rank's own experts, the scatter adjoint and routing-weight gradients
    returned along the inverse layout, dispatch adjoint at the source
    (backward.cpp:43-152).  Ranks are threads on one GPU (loopback transport;
    peer = the forward's fused peer-memory exchange).  Against the reference's
    backward_vjps with sources = owning rank (SwiGLU: the oracle restatement
    is the torch fp64 autograd of the same layer), within 2e-2."""
    import threading
    dm, dh = 128, 256
    n_per = [37, 64, 5, 100, 0, 64, 33, 1][:nd]
    n = sum(n_per)
    gated = act == "swiglu"
    x, g, w1, w2, w3 = make_layer_inputs(nd * 17 + k, n, dm, dh, ne, gated=gated)
    ids, w = random_routing(n, ne, k, np.random.default_rng(nd * 3 + k))
    w = w.astype(np.float32).astype(np.float64)
    plist = _placement(ne, nd, "shuffled", seed=nd + 1)
    src = np.concatenate([np.full(c, r, np.int32) for r, c in enumerate(n_per)])
    up = bf16_round(np.random.default_rng(2).uniform(-1, 1, (n, dm)))
    if gated:
        X = torch.tensor(x, requires_grad=True)
        W1, W2, W3 = (torch.tensor(a, requires_grad=True) for a in (w1, w2, w3))
        Wt = torch.tensor(w, requires_grad=True)
        Y = torch.zeros((n, dm), dtype=torch.float64)
        I = torch.from_numpy(ids).long()
        for e in range(ne):
            t, j = (I == e).nonzero(as_tuple=True)
            if len(t):
                h = torch.nn.functional.silu(X[t] @ W1[e]) * (X[t] @ W3[e])
                Y = Y.index_add(0, t, (h @ W2[e]) * Wt[t, j].unsqueeze(1))
        (Y * torch.from_numpy(up)).sum().backward()
        rgx, rgw1, rgw2, rgr, rgw3 = (a.grad.numpy() for a in (X, W1, W2, Wt, W3))
    else:
        rgx, rgw1, rgw2, rgr = O.ref_backward(x, ids, w, w1, w2, plist, src, up, act=act)
    grads = [None] * nd
    errs = []
    starts = np.concatenate([[0], np.cumsum(n_per)])
    key = np.random.default_rng().integers(1 << 30)
    sl = [slice(starts[r], starts[r + 1]) for r in range(nd)]  # device inputs up front (see the forward test)
    X = [cuda(x[q], torch.bfloat16) for q in sl]
    I = [cuda(ids[q]) for q in sl]
    Wt = [cuda(w[q], torch.float32) for q in sl]
    U = [cuda(up[q], torch.bfloat16) for q in sl]
    OUT = [torch.empty_like(t) for t in X]
    done = threading.Barrier(nd)

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                cfg = occ.MoEConfig(ne, k, nd, dm, dh, activation=act, dedup=dedup)
                layer = occ.ExpertParallelLayer(cfg, occ.Placement([list(p) for p in plist]), world_size=nd, rank=r)
                layer.set_training(True)
                loc = plist[r]
                layer.load_experts(cuda(w1[loc], torch.bfloat16), cuda(w2[loc], torch.bfloat16),
                                   cuda(w3[loc], torch.bfloat16) if gated else None)
                layer.comm_init_loopback(int(key))
                if peer:
                    layer.comm_enable_peer(128)
                for _rep in range(2):  # a second step reuses every buffer
                    layer.forward_given_routing(X[r], I[r], Wt[r], out=OUT[r])
                    gr = layer.backward(U[r])
                st.synchronize()
                done.wait()
                grads[r] = {kk: (v.cpu().numpy() if v is not None else None) for kk, v in gr.items()}
        except Exception as e:  # surface thread failures
            errs.append(e)
            done.abort()

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(nd)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=120)
    assert not errs, errs
    gx = np.concatenate([gg["x"] for gg in grads])
    gw = np.concatenate([gg["routing_weights"] for gg in grads])
    gw1 = np.zeros_like(rgw1)
    gw2 = np.zeros_like(rgw2)
    for r in range(nd):  # each rank holds its own experts' gradients, placement-list order
        gw1[plist[r]] = grads[r]["w1"]
        gw2[plist[r]] = grads[r]["w2"]
    e = {"x": rel_err(gx, rgx), "w1": rel_err(gw1, rgw1), "w2": rel_err(gw2, rgw2), "routing": rel_err(gw, rgr)}
    if gated:
        gw3 = np.zeros_like(rgw3)
        for r in range(nd):
            gw3[plist[r]] = grads[r]["w3"]
        e["w3"] = rel_err(gw3, rgw3)
    assert max(e.values()) <= 2e-2, e


BWD_CASES = [(8, 2, 2, 64, 128, "silu", 200), (8, 3, 4, 128, 256, "identity", 300), (16, 4, 4, 64, 320, "relu", 150),
             (8, 2, 1, 256, 512, "silu", 513),
             (128, 64, 2, 64, 64, "relu", 100),  # maximum top-k
             # wide-tile paths: forward / data-gradient GEMMs with K >= 1024 and weight gradients with
             # an even number of 256-column blocks
             (8, 2, 2, 1024, 1024, "silu", 300), (4, 1, 2, 512, 1024, "relu", 97)]


@pytest.mark.parametrize("ne,k,nd,dm,dh,act,n", BWD_CASES)
@pytest.mark.parametrize("dedup", [True, False])
def test_backward_matches_reference(ne, k, nd, dm, dh, act, n, dedup):
    """backward_vjps (backward.cpp:24-161) of the reference on identical
    bf16-representable inputs: every gradient block within 2e-2 normwise."""
    x, g, w1, w2, _ = make_layer_inputs(ne + n, n, dm, dh, ne)
    ids, w = random_routing(n, ne, k, np.random.default_rng(n))
    w = w.astype(np.float32).astype(np.float64)
    plist = _placement(ne, nd, "shuffled", seed=3)
    src = (np.arange(n) % nd).astype(np.int32)
    up = bf16_round(np.random.default_rng(1).uniform(-1, 1, (n, dm)))
    rgx, rgw1, rgw2, rgr = O.ref_backward(x, ids, w, w1, w2, plist, src, up, act=act)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act, dedup=dedup),
                                    occ.Placement([list(p) for p in plist]))
    layer.set_training(True)
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32), cuda(src))
    gr = layer.backward(cuda(up, torch.bfloat16))
    errs = {"x": rel_err(gr["x"].cpu().numpy(), rgx), "w1": rel_err(gr["w1"].cpu().numpy(), rgw1),
            "w2": rel_err(gr["w2"].cpu().numpy(), rgw2),
            "routing": rel_err(gr["routing_weights"].cpu().numpy(), rgr)}
    assert max(errs.values()) <= 2e-2, errs


@pytest.mark.parametrize("dm,dh", [(128, 256), (1024, 512)])  # (1024, 512): wide-tile GEMMs with saved pre-activations
def test_backward_swiglu_matches_autograd(dm, dh):
    """SwiGLU extension: against torch autograd in fp64 on the CPU."""
    ne, k, nd, n = 8, 2, 2, 300
    x, g, w1, w2, w3 = make_layer_inputs(11, n, dm, dh, ne, gated=True)
    ids, w = random_routing(n, ne, k, np.random.default_rng(5))
    w = w.astype(np.float32).astype(np.float64)
    up = bf16_round(np.random.default_rng(2).uniform(-1, 1, (n, dm)))
    T = lambda a: torch.tensor(a, dtype=torch.float64, requires_grad=True)
    tx, tw1, tw2, tw3, tw = T(x), T(w1), T(w2), T(w3), T(w)
    out = torch.zeros(n, dm, dtype=torch.float64)
    for j in range(k):
        e = torch.from_numpy(ids[:, j]).long()
        a = torch.einsum("nd,ndf->nf", tx, tw1[e])
        b = torch.einsum("nd,ndf->nf", tx, tw3[e])
        out = out + tw[:, j:j + 1] * torch.einsum("nf,nfd->nd", torch.nn.functional.silu(a) * b, tw2[e])
    (out * torch.from_numpy(up)).sum().backward()
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="swiglu"))
    layer.set_training(True)
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16))
    y = layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    assert rel_err(y.double().cpu().numpy(), out.detach().numpy()) <= TOL
    gr = layer.backward(cuda(up, torch.bfloat16))
    errs = {name: rel_err(gr[name].cpu().numpy(), ref_t.grad.numpy())
            for name, ref_t in (("x", tx), ("w1", tw1), ("w3", tw3), ("w2", tw2), ("routing_weights", tw))}
    assert max(errs.values()) <= 2e-2, errs


def test_backward_zero_upstream_and_state_error():
    ne, k, nd, dm, dh, n = 8, 2, 2, 64, 128, 64
    x, g, w1, w2, _ = make_layer_inputs(3, n, dm, dh, ne)
    ids, w = random_routing(n, ne, k, np.random.default_rng(0))
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    with pytest.raises(occ.StateError):  # backward.cpp:25 / test_pipeline.cpp:533-536
        layer.backward(torch.zeros(n, dm, device="cuda"))
    layer.set_training(True)
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    gr = layer.backward(torch.zeros(n, dm, device="cuda"))
    for name in ("x", "w1", "w2", "routing_weights"):
        assert not gr[name].any(), name
    # state invalidation: a new placement, new weights or a bare
    # dispatch plan drop the saved forward; training switched on after the
    # weights were loaded has no backward weight copies -> StateError, not a
    # device fault
    layer.build_dispatch_index(cuda(ids))
    with pytest.raises(occ.StateError):
        layer.backward(torch.zeros(n, dm, device="cuda"))
    late = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    late.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    late.set_training(True)
    late.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    with pytest.raises(occ.StateError):
        late.backward(torch.zeros(n, dm, device="cuda"))
    late.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))  # reload: copies built now
    late.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    assert not late.backward(torch.zeros(n, dm, device="cuda"))["x"].any()


def test_collaboration_aware_placement_on_gpu():
    """Profiling -> placement loop: device histogram of
    planted-block traces (bit-exact with the reference's accumulate_collab),
    reschedule_placement, and the device dispatch plan's E(C_T) drops by
    >= 10% vs the trivial layout (acceptance.cpp:218-244 criterion) at EP=8."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles"))
    from placement_gain import planted_block_ids
    ne, k, nd, n = 64, 8, 8, 8192
    ids_np, _ = planted_block_ids(n, ne, k, 8, 0.9, np.random.default_rng(11))
    ids = cuda(ids_np)
    counts = occ.build_collab_graph(ids, ne).cpu().numpy()
    assert np.array_equal(counts, ref().accumulate_collab(ids_np, ne))
    placement = occ.collaboration_aware_placement([ids], ne, nd)
    assert placement.devices == occ.reschedule_placement(ref().normalize_graph(counts), nd).devices
    ct = {}
    for name, pl in (("trivial", occ.trivial_placement(ne, nd)), ("rescheduled", placement)):
        layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, 64, 64), pl)
        layer.build_dispatch_index(ids)
        ct[name] = layer.comm_report(bytes_per_scalar=2).mean_replicas
    assert ct["rescheduled"] <= 0.9 * ct["trivial"], ct


@pytest.mark.parametrize("ne,k,nd,n", [(8, 2, 2, 2048), (64, 8, 8, 8192), (16, 4, 4, 999)])
def test_simulate_report_matches_reference(ne, k, nd, n):
    """`#moesim-report v1` from the GPU run == the same report rendered from
    the reference's own CommReport and accumulate_collab:
    every line, integers and doubles."""
    from types import SimpleNamespace
    from paper_2505_13345_b200 import report as R
    rng = np.random.default_rng(n + ne)
    ids, w = random_routing(n, ne, k, rng)
    w = w.astype(np.float32).astype(np.float64)
    plist = _placement(ne, nd, "shuffled", seed=2)
    _, rr = ref().forward_given_routing(np.full((n, 1), 0.5), ids, w, np.ones((ne, 1, 8)), np.ones((ne, 8, 1)),
                                        plist, None, act="identity", single=False, bytes_per_scalar=2)
    cfg = occ.MoEConfig(ne, k, nd, 64, 64, activation="silu")
    layer = occ.ExpertParallelLayer(cfg, occ.Placement([list(p) for p in plist]))
    layer.load_experts(torch.zeros(ne, 64, 64, dtype=torch.bfloat16, device="cuda"),
                       torch.zeros(ne, 64, 64, dtype=torch.bfloat16, device="cuda"))
    layer.forward_given_routing(torch.zeros(n, 64, dtype=torch.bfloat16, device="cuda"), cuda(ids),
                                cuda(w, torch.float32))
    got = R.simulate_report(layer, cuda(ids), bytes_per_scalar=2)
    ref_rep = SimpleNamespace(mean_replicas=rr.mean_replicas, cap_replicas=rr.cap_replicas,
                              intra_share=rr.intra_share, inter_share=rr.inter_share,
                              cross_device_bytes=rr.crossing_rows * 64 * 2,  # width-1 replay: bytes at D = 64
                              per_device_token_counts=[rr.per_device_rows[d] for d in range(nd)])
    want = R.render_simulate_report(cfg, ref_rep, ref().accumulate_collab(ids, ne), [list(p) for p in plist], n,
                                    bytes_per_scalar=2)
    diff = [(a, b) for a, b in zip(got.splitlines(), want.splitlines()) if a != b]
    assert not diff and len(got) == len(want), diff


@pytest.mark.parametrize("train,shared", [(False, False), (False, True), (True, False)])
def test_cuda_graph_replay_bit_identical(train, shared):
    """With validation off the whole step (route + forward [+ backward]) has no
    host synchronisation and captures into a CUDA graph; replays equal eager
    calls bit for bit (this is what bench.py times)."""
    ne, k, nd, dm, dh, n = 16, 4, 2, 128, 256, 700
    x, g, w1, w2, w3 = make_layer_inputs(5, n, dm, dh, ne, gated=True)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="swiglu"))
    if train:
        layer.set_training(True)
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16))
    if shared:
        s1, s2, s3, sg = make_shared(2, dm, 128, True, seed=3)
        layer.load_shared_experts(cuda(s1, torch.bfloat16), cuda(s2, torch.bfloat16), cuda(s3, torch.bfloat16),
                                  cuda(sg, torch.bfloat16))
    layer.set_validate(False)
    xs, gs = cuda(x, torch.bfloat16), cuda(g, torch.bfloat16)
    up = torch.empty_like(xs).uniform_(-1, 1)
    out = torch.empty_like(xs)
    res = {}

    def step():
        layer.forward_expert_parallel(xs, gs, out=out)
        if train:
            res["gx"] = layer.backward(up)["x"]

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    eager = out.clone()
    eager_gx = res["gx"].clone() if train else None
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    if train:
        assert torch.equal(res["gx"], eager_gx)


def test_train_step_host_pipeline_matches_device():
    """train_step_host (pinned host in/out, double-buffered copies) returns the
    same token gradients as forward_expert_parallel + backward on the device,
    step after step (the slots rotate)."""
    ne, k, nd, dm, dh, n = 8, 2, 2, 128, 256, 513
    x, g, w1, w2, w3 = make_layer_inputs(9, n, dm, dh, ne, gated=True)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="swiglu"))
    layer.set_training(True)
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16))
    gs = cuda(g, torch.bfloat16)
    rng = np.random.default_rng(4)
    hosts = []
    for i in range(3):
        xi = torch.from_numpy(bf16_round(rng.uniform(-1, 1, (n, dm)))).to(torch.bfloat16).pin_memory()
        ui = torch.from_numpy(bf16_round(rng.uniform(-1, 1, (n, dm)))).to(torch.bfloat16).pin_memory()
        gi = torch.empty((n, dm), dtype=torch.float32).pin_memory()
        hosts.append((xi, ui, gi))
    for xi, ui, gi in hosts:
        layer.train_step_host(xi, gs, ui, gi, wait=False)
    layer.host_wait()
    torch.cuda.synchronize()
    for xi, ui, gi in hosts:
        layer.forward_expert_parallel(xi.cuda(), gs)
        want = layer.backward(ui.cuda())["x"].cpu()
        assert torch.equal(gi, want)
    # mixed precision: bf16 token gradient = the fp32 one rounded once
    xi, ui, _ = hosts[0]
    gb = torch.empty((n, dm), dtype=torch.bfloat16).pin_memory()
    layer.train_step_host(xi, gs, ui, gb)
    layer.forward_expert_parallel(xi.cuda(), gs)
    want = layer.backward(ui.cuda())["x"].cpu()
    assert torch.equal(gb, want.to(torch.bfloat16))


@pytest.mark.parametrize("act,dm,dh", [("swiglu", 2048, 512), ("silu", 2048, 2048), ("relu", 1024, 1280)])
def test_wide_tile_gemm_path(act, dm, dh):
    """K >= 2048 with an even number of 256-row B blocks selects the 256 x 512
    super-tile GEMM (two accumulators sharing each A K-block); outputs match
    the oracle on sampled rows (rows are independent given routing).  Enough
    tokens for a full wave of tiles (the auto rule keeps narrow tiles for
    smaller batches)."""
    ne, k, nd, n = 8, 2, 2, 3000
    gated = act == "swiglu"
    x, g, w1, w2, w3 = make_layer_inputs(17, n, dm, dh, ne, gated=gated)
    ids, w = random_routing(n, ne, k, np.random.default_rng(17))
    w = w.astype(np.float32).astype(np.float64)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16) if gated else None)
    out = layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    rows = np.arange(0, n, 29)
    want = O.Port().dense_given_routing(x, ids, w, w1, w2, act="silu" if gated else act, single=False, rows=rows,
                                        w3=w3)
    assert rel_err(out.double().cpu().numpy()[rows], want) <= TOL


def test_wide_tile_forced_odd_blocks():
    """OCC_GEMM_WIDE=2 forces the wide kernel, including odd B-block counts
    (a last single-block super-tile): torch fp32 reference, fresh process."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, OCC_GEMM_WIDE="2")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "profiles", "probes", "wide_debug.py")], env=env,
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if " err " in l]
    assert len(lines) == 5, r.stdout
    for l in lines:
        assert float(l.split(" err ")[1].split()[0]) <= 1e-2, l


def test_dynamic_tile_schedule_bit_identical():
    """The dynamic tile scheduler (launch-order tile counter) only changes
    which CTA pair runs a tile, never a tile's math: forward, shared-expert
    and backward outputs of wide / narrow / weight-gradient GEMMs over many
    waves are bit-identical to the static walk (OCC_GEMM_DYN=0), each in a
    fresh process (the switch is read once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dig = []
    for dyn in ("0", "1"):
        r = subprocess.run([sys.executable, os.path.join(root, "profiles", "probes", "sched_digest.py")],
                           env=dict(os.environ, OCC_GEMM_DYN=dyn), capture_output=True, text=True, timeout=600,
                           cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        dig.append([l for l in r.stdout.splitlines() if l.startswith("digest")][0].split()[1])
    assert dig[0] == dig[1], dig


@pytest.mark.parametrize("ne,k,nd", [(256, 8, 4), (200, 64, 4), (130, 3, 5)])
def test_wide_gate_router_matches_oracle_topk(ne, k, nd):
    """Gates wider than 128 experts take the logits + router_select path:
    ids equal the reference top-k (routing.cpp:60-84) on the same fp32
    softmax rows."""
    dm, n = 128, 700
    x, g, *_ = make_layer_inputs(ne + k, n, dm, 8, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, 64))
    xs, gs = cuda(x, torch.bfloat16), cuda(g, torch.bfloat16)
    ids, w, sc = layer.route(xs, gs, want_scores=True)
    want_ids, want_w = O.Port().topk_route(sc.double().cpu().numpy(), k, True)
    assert np.array_equal(ids.cpu().numpy(), want_ids)
    assert np.allclose(w.double().cpu().numpy(), want_w, rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("ne,n", [(8, 777), (64, 4000), (60, 1)])
def test_similarity_table_on_gpu(ne, n):
    """SimilarityAccumulator (pruning.cpp:165-219) on the device: values
    bit-exact with the reference's build_similarity_table for fp64 logits;
    two batches equal one concatenated batch within rounding; f32 router
    logits from the tcgen05 router feed the same path."""
    rng = np.random.default_rng(ne + n)
    logits = rng.normal(size=(n, ne))
    logits[:, 0] = np.abs(logits[:, 0])
    want, want_rank = ref().similarity_table(logits)
    got = occ.build_similarity_table([cuda(logits)], ne)
    assert np.array_equal(got, want)
    if n > 1:
        h = n // 2
        got2 = occ.build_similarity_table([cuda(logits[:h]), cuda(logits[h:])], ne)
        assert np.allclose(got2, want, rtol=1e-12, atol=1e-14)
    dm = 128
    x, g, *_ = make_layer_inputs(ne, max(n, 2), dm, 8, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, 2, 1 if ne <= 64 else 2, dm, 64))
    lg = layer.router_logits(cuda(x, torch.bfloat16), cuda(g, torch.bfloat16))
    want_l = x.astype(np.float64) @ g.astype(np.float64).T
    assert rel_err(lg.double().cpu().numpy(), want_l) < 1e-5
    vals = occ.build_similarity_table([lg], ne)
    layer.set_similarity(vals)  # ranking built as the reference does


# ------------------------------------------- micro-batched (overlapped) forward --
@pytest.mark.parametrize("ne,k,nd,dm,dh,act,n,shared,sources", [
    (8, 2, 2, 128, 256, "silu", 1000, 0, False), (8, 2, 2, 128, 256, "silu", 1, 0, False),
    (16, 4, 4, 64, 128, "relu", 333, 0, True), (64, 6, 8, 256, 128, "swiglu", 777, 2, False),
    (8, 3, 1, 128, 256, "identity", 5, 1, False)])
def test_micro_batched_forward_bit_identical(ne, k, nd, dm, dh, act, n, shared, sources):
    """occ_set_micro_batches(2): the two halves on two streams give the unsplit
    forward's output bit for bit and the same CommReport (world_size 1; the
    world_size > 1 split is in test_multi_rank_forward_loopback)."""
    gated = act == "swiglu"
    x, g, w1, w2, w3 = make_layer_inputs(ne + n, n, dm, dh, ne, gated=gated)
    ids, w = random_routing(n, ne, k, np.random.default_rng(n))
    src = cuda(np.random.default_rng(1).integers(0, nd, n).astype(np.int32)) if sources else None
    res = {}
    for mb in (1, 2):
        layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act),
                                        occ.Placement([list(p) for p in _placement(ne, nd, "shuffled", seed=3)]))
        layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16) if gated else None)
        if shared:
            s1, s2, s3, sg = make_shared(shared, dm, 128, gated, seed=4)
            layer.load_shared_experts(cuda(s1, torch.bfloat16), cuda(s2, torch.bfloat16),
                                      cuda(s3, torch.bfloat16) if gated else None, cuda(sg, torch.bfloat16))
        if mb == 2:
            layer.set_micro_batches(2)
        xs = cuda(x, torch.bfloat16)
        a = layer.forward_given_routing(xs, cuda(ids), cuda(w, torch.float32), sources=src)
        b = layer.forward_expert_parallel(xs, cuda(g, torch.bfloat16), sources=src)
        rep = layer.comm_report(bytes_per_scalar=2)
        torch.cuda.synchronize()
        res[mb] = (a, b, rep)
    assert torch.equal(res[1][0], res[2][0])
    assert torch.equal(res[1][1], res[2][1])
    r1, r2 = res[1][2], res[2][2]
    assert (r1.mean_replicas, r1.cross_device_bytes, r1.per_device_token_counts, r1.intra_share) == \
        (r2.mean_replicas, r2.cross_device_bytes, r2.per_device_token_counts, r2.intra_share)


def test_micro_batches_guards():
    layer = occ.ExpertParallelLayer(occ.MoEConfig(8, 2, 2, 64, 64, activation="silu"))
    with pytest.raises(occ.api.MoesimError):
        layer.set_micro_batches(3)
    layer.set_micro_batches(2)
    with pytest.raises(occ.api.MoesimError):
        layer.set_training(True)
    layer.set_micro_batches(1)
    layer.set_training(True)


def test_degenerate_batches():
    """Zero tokens through every entry point: routed forward, micro-batched
    forward, host pipeline, training step and CommReport; one token with the
    maximum top-k."""
    ne, k, nd, dm, dh = 8, 2, 2, 64, 128
    x, g, w1, w2, _ = make_layer_inputs(3, 4, dm, dh, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    layer.set_training(True)
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    gs = cuda(g, torch.bfloat16)
    x0 = torch.zeros(0, dm, dtype=torch.bfloat16, device="cuda")
    assert layer.forward_expert_parallel(x0, gs).shape == (0, dm)
    gr = layer.backward(torch.zeros(0, dm, dtype=torch.bfloat16, device="cuda"))
    assert gr["x"].shape == (0, dm) and float(gr["w1"].abs().sum()) == 0.0
    r = layer.comm_report()
    assert r.mean_replicas == 0.0 and r.per_device_token_counts == [0, 0]
    layer.set_training(False)
    xh = x0.cpu().pin_memory()
    layer.forward_host(xh, gs, torch.empty_like(xh).pin_memory())
    layer.set_micro_batches(2)
    assert layer.forward_expert_parallel(x0, gs).shape == (0, dm)
    one = cuda(x[:1], torch.bfloat16)
    full = occ.ExpertParallelLayer(occ.MoEConfig(ne, ne, nd, dm, dh, activation="silu"))  # k = E: every expert
    full.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    ids = cuda(np.arange(ne, dtype=np.int32)[None, :])
    w = cuda(np.full((1, ne), 1.0 / ne, np.float32))
    got = full.forward_given_routing(one, ids, w).double().cpu().numpy()
    want, _ = ref().forward_given_routing(x[:1], np.arange(ne, dtype=np.int32)[None, :], np.full((1, ne), 1.0 / ne),
                                          w1, w2, _placement(ne, nd, "trivial"), np.zeros(1, np.int32), act="silu",
                                          single=False)
    assert rel_err(got, want) <= TOL


@pytest.mark.parametrize("ne,k,dm", [(8, 2, 40), (60, 4, 72), (130, 3, 200), (16, 16, 8), (64, 8, 4104)])
def test_router_ragged_widths(ne, k, dm):
    """Production router at token widths that are multiples of 8 but not of
    the 64-element K block (TMA zero-fills the tail): ids equal the reference
    top-k of its own softmax rows, which match fp64 softmax to f32 rounding."""
    n = 333
    x, g, *_ = make_layer_inputs(ne + dm, n, dm, 8, ne)
    nd = 1 if ne <= 64 else 5
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, 64))
    xs, gs = cuda(x, torch.bfloat16), cuda(g, torch.bfloat16)
    ids, w, sc = layer.route(xs, gs, want_scores=True)
    want_ids, _ = O.Port().topk_route(sc.double().cpu().numpy(), k, True)
    assert np.array_equal(ids.cpu().numpy(), want_ids)
    xb = xs.double().cpu().numpy()
    gb = gs.double().cpu().numpy()
    lg = xb @ gb.T
    p = np.exp(lg - lg.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    # f32 logits over K = D bf16 products: absolute error grows with D
    assert np.allclose(sc.double().cpu().numpy(), p, rtol=1e-3, atol=1e-5)


def test_placement_change_at_runtime():
    """occ_set_placement between forwards (the profiling -> placement loop
    applied to a live layer): the next forward equals a fresh layer built with
    the new placement, values and CommReport, with and without reloading the
    experts (world_size 1 keeps every expert resident)."""
    ne, k, nd, dm, dh, n = 16, 4, 4, 64, 128, 500
    x, g, w1, w2, _ = make_layer_inputs(21, n, dm, dh, ne)
    ids, w = random_routing(n, ne, k, np.random.default_rng(21))
    new = _placement(ne, nd, "shuffled", seed=9)
    args = (cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32))
    fresh = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"),
                                    occ.Placement([list(p) for p in new]))
    fresh.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    want = fresh.forward_given_routing(*args)
    want_rep = fresh.comm_report(bytes_per_scalar=2)
    for reload, mb in ((False, 1), (True, 1), (False, 2), (True, 2)):
        layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
        layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
        if mb > 1:
            layer.set_micro_batches(mb)
        layer.forward_given_routing(*args)
        layer.set_placement(occ.Placement([list(p) for p in new]))
        if reload:
            layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
        got = layer.forward_given_routing(*args)
        rep = layer.comm_report(bytes_per_scalar=2)
        assert torch.equal(got, want), reload
        assert (rep.mean_replicas, rep.cross_device_bytes, rep.per_device_token_counts) == \
            (want_rep.mean_replicas, want_rep.cross_device_bytes, want_rep.per_device_token_counts)


def test_repeated_forwards_stable():
    """Production loop: hundreds of forwards (eager, graph replay, host
    pipeline, micro-batched) give the first result bit for bit and the
    device's free memory does not drift (no per-call allocations leak)."""
    ne, k, nd, dm, dh, n = 16, 4, 4, 128, 256, 777
    x, g, w1, w2, w3 = make_layer_inputs(31, n, dm, dh, ne, gated=True)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="swiglu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16))
    xs, gs = cuda(x, torch.bfloat16), cuda(g, torch.bfloat16)
    want = layer.forward_expert_parallel(xs, gs).clone()
    layer.set_validate(False)
    out = torch.empty_like(xs)
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        layer.forward_expert_parallel(xs, gs, out=out)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(graph):
        layer.forward_expert_parallel(xs, gs, out=out)
    xh = xs.cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for i in range(300):
        if i % 3 == 0:
            graph.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, want), i
        elif i % 3 == 1:
            assert torch.equal(layer.forward_expert_parallel(xs, gs), want), i
        else:
            layer.forward_host(xh, gs, oh)
            torch.cuda.synchronize()
            assert torch.equal(oh, want.cpu()), i
    torch.cuda.synchronize()
    assert abs(torch.cuda.mem_get_info()[0] - free0) < (64 << 20)
    layer.set_micro_batches(2)
    for i in range(50):
        assert torch.equal(layer.forward_expert_parallel(xs, gs), want), i


def test_api_rejects_wrong_dtypes_and_shapes():
    """The C-ABI takes raw pointers: a float32 x / gate or int64 ids would be
    reinterpreted, so the Python mirror refuses them."""
    ne, k, nd, dm, dh, n = 8, 2, 2, 64, 128, 32
    x, g, w1, w2, _ = make_layer_inputs(4, n, dm, dh, ne)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    xb, gb = cuda(x, torch.bfloat16), cuda(g, torch.bfloat16)
    with pytest.raises(occ.ShapeError):
        layer.forward_expert_parallel(xb.float(), gb)
    with pytest.raises(occ.ShapeError):
        layer.forward_expert_parallel(xb, gb.float())
    with pytest.raises(occ.ShapeError):
        layer.route(xb, gb[:, :dm // 2])
    ids, w = layer.route(xb, gb)
    with pytest.raises(occ.ShapeError):
        layer.forward_given_routing(xb, ids.long(), w)
    with pytest.raises(occ.ShapeError):
        layer.forward_given_routing(xb, ids, w, sources=torch.zeros(n, dtype=torch.int64, device="cuda"))
    # non-contiguous but correctly typed inputs are accepted (copied, kept alive)
    xt = torch.empty((dm, n), dtype=torch.bfloat16, device="cuda").t()
    xt.copy_(xb)
    assert torch.equal(layer.forward_expert_parallel(xt, gb), layer.forward_expert_parallel(xb, gb))


STAGE_CASES = [(8, 2, 2, 256, 512, "silu", 700), (16, 4, 4, 128, 256, "swiglu", 1000),
               (64, 8, 8, 512, 256, "relu", 900), (8, 3, 1, 128, 128, "identity", 64)]


@pytest.mark.parametrize("ne,k,nd,dm,dh,act,n", STAGE_CASES)
def test_stage_entry_points_chain_equals_forward(ne, k, nd, dm, dh, act, n):
    """The stage-level C-ABI (pipeline.hpp:89-123) driven by the caller with
    its own exchange (torch indexing by the occ_exchange_layout offsets):
    build_dispatch_index -> dispatch (SfdBatch, pipeline.cpp:91-123) ->
    all_to_all_exchange (:125-176) -> build_compute_index (:52-89) +
    expert compute (:178-283) -> return exchange (:456-466) -> combine
    (:285-300).  The SfdBatch token map, the inbox order (source asc, counter
    asc) and BRIM1 equal the reference's own records; the chained output
    equals the fused occ_forward bit for bit (and so the reference within
    1e-2)."""
    gated = act == "swiglu"
    x, g, w1, w2, w3 = make_layer_inputs(ne + k + n, n, dm, dh, ne, gated=gated)
    ids, w = random_routing(n, ne, k, np.random.default_rng(n + 1))
    w32 = w.astype(np.float32)
    plist = _placement(ne, nd, "shuffled", seed=11)
    src = np.random.default_rng(n).integers(0, nd, n).astype(np.int32)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act),
                                    occ.Placement([list(map(int, p)) for p in plist]))
    layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16),
                       cuda(w3, torch.bfloat16) if gated else None)
    X, I, Wt, S = cuda(x, torch.bfloat16), cuda(ids), cuda(w32), cuda(src)
    want = layer.forward_given_routing(X, I, Wt, S)
    # reference records (indices are width-independent: a width-1 replay)
    _, _, ridx = ref().forward_given_routing(x[:, :1], ids, w32.astype(np.float64), w1[:, :1, :1], w2[:, :1, :1],
                                             plist, src, act="identity", single=False, want_index=True)
    brim0_all, counts = layer.build_dispatch_index(I, S)
    C = counts.cpu().numpy()
    pos, sfd = 0, []
    for s in range(nd):
        tok = np.nonzero(src == s)[0]
        b = brim0_all[pos:pos + nd * len(tok)]
        pos += nd * len(tok)
        assert np.array_equal(b.cpu().numpy().reshape(nd, len(tok)), ridx["dindex"][s])
        tt = cuda(tok.astype(np.int64))
        sx, si, sw, st = layer.dispatch(X[tt], I[tt], Wt[tt], b, n_sfd=int(C[s].sum()))
        # SfdBatch token map: Sfd row c holds the token whose counter is c
        want_tok = np.full(int(C[s].sum()), -1)
        bb = ridx["dindex"][s]
        for d in range(nd):
            for i in range(len(tok)):
                if bb[d, i] >= 0:
                    want_tok[bb[d, i]] = i
        assert np.array_equal(st.cpu().numpy(), want_tok)
        sfd.append((sx, si, sw, b, tt))
    # the caller's exchange: destination d receives, source asc, the contiguous
    # rows each source's device-major batch holds for it
    rets = {}
    for d in range(nd):
        parts, meta = [], []
        for s in range(nd):
            off = int(C[s, :d].sum())
            parts.append((sfd[s][0][off:off + C[s, d]], sfd[s][1][off:off + C[s, d]], sfd[s][2][off:off + C[s, d]]))
            meta.append((s, off, int(C[s, d])))
        in_x = torch.cat([p[0] for p in parts])
        in_i = torch.cat([p[1] for p in parts])
        in_w = torch.cat([p[2] for p in parts])
        rinbox = ridx["inbox"][d]
        got_src = np.concatenate([np.full(c, s) for s, _, c in meta]).astype(np.int64)
        got_slot = np.concatenate([np.arange(o, o + c) for _, o, c in meta]).astype(np.int64)
        assert np.array_equal(got_src, rinbox[1]) and np.array_equal(got_slot, rinbox[2])
        cix, nepd = layer.build_compute_index(d, in_i, in_w)
        assert np.array_equal(cix.cpu().numpy(), ridx["cindex"][d]) and nepd == int((ridx["cindex"][d] >= 0).sum())
        y = layer.expert_compute(d, in_x, in_i, in_w)
        r0 = 0
        for s, off, c in meta:
            rets[(s, d)] = (off, y[r0:r0 + c])
            r0 += c
    out = torch.empty_like(X)
    for s in range(nd):
        ns = int(C[s].sum())
        y_src = torch.empty((ns, dm), dtype=torch.bfloat16, device="cuda")
        for d in range(nd):
            off, rows = rets[(s, d)]
            y_src[off:off + rows.shape[0]] = rows
        out[sfd[s][4]] = layer.combine(y_src, sfd[s][3], sfd[s][4].shape[0])
    assert torch.equal(out, want)


def test_stage_entry_points_world_gt1_handle():
    """On a world_size > 1 handle (no communicator needed: the stages never
    communicate) the local BRIM0 of this rank's tokens equals the reference's
    per-source dispatch index, and expert_compute runs this rank's experts."""
    ne, k, nd, dm, dh, n = 16, 4, 4, 128, 256, 300
    x, g, w1, w2, _ = make_layer_inputs(77, n, dm, dh, ne)
    ids, w = random_routing(n, ne, k, np.random.default_rng(5))
    plist = _placement(ne, nd, "shuffled", seed=2)
    _, _, ridx = ref().forward_given_routing(x[:, :1], ids, w, w1[:, :1, :1], w2[:, :1, :1], plist,
                                             np.full(n, 2, np.int32), act="identity", single=False, want_index=True)
    rank = 2
    h = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"),
                                occ.Placement([list(map(int, p)) for p in plist]), world_size=nd, rank=rank)
    P = ne // nd
    h.load_experts(cuda(w1[plist[rank]], torch.bfloat16), cuda(w2[plist[rank]], torch.bfloat16))
    b, cnt = h.build_dispatch_index(cuda(ids))
    assert np.array_equal(b.cpu().numpy().reshape(nd, n), ridx["dindex"][rank])
    assert np.array_equal(cnt.cpu().numpy(), (ridx["dindex"][rank] >= 0).sum(1))
    # expert compute of this rank on the rows routed to it, vs a world_size 1 handle's device `rank`
    sx, si, sw, _ = h.dispatch(cuda(x, torch.bfloat16), cuda(ids), cuda(w.astype(np.float32)), b)
    off = int(cnt[:rank].sum())
    rows = slice(off, off + int(cnt[rank]))
    y = h.expert_compute(rank, sx[rows], si[rows], sw[rows])
    one = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"),
                                  occ.Placement([list(map(int, p)) for p in plist]))
    one.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16))
    assert torch.equal(y, one.expert_compute(rank, sx[rows], si[rows], sw[rows]))
    with pytest.raises(occ.ConfigError):
        h.expert_compute(0, sx[rows], si[rows], sw[rows])


@pytest.mark.parametrize("nd,ne,k", [(2, 8, 2), (8, 64, 8)])
def test_multi_rank_peer_forward_graph_replay_loopback(nd, ne, k):
    """world_size > 1 with the fused peer-memory exchange has no host
    synchronisation (counts exchanged through peer memory, received row count
    kept on the device, the arrival-flag sequence number advanced by a kernel),
    so each rank's forward captures into a CUDA graph; replays with new inputs
    equal the eager forward bit for bit (loopback ranks on one GPU)."""
    import threading
    dm, dh = 128, 256
    n_per = [37, 64, 5, 100, 0, 64, 33, 1][:nd]
    n = sum(n_per)
    x, g, w1, w2, _ = make_layer_inputs(nd * 5, n, dm, dh, ne)
    ids, w = random_routing(n, ne, k, np.random.default_rng(nd))
    plist = _placement(ne, nd, "shuffled", seed=nd + 7)
    starts = np.concatenate([[0], np.cumsum(n_per)])
    key = np.random.default_rng().integers(1 << 30)
    errs, ok = [], [False] * nd
    barrier = threading.Barrier(nd)

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"),
                                                occ.Placement([list(p) for p in plist]), world_size=nd, rank=r)
                loc = plist[r]
                layer.load_experts(cuda(w1[loc], torch.bfloat16), cuda(w2[loc], torch.bfloat16))
                layer.comm_init_loopback(int(key))
                layer.comm_enable_peer(128)
                layer.set_validate(False)
                a, b = starts[r], starts[r + 1]
                X = cuda(x[a:b], torch.bfloat16)
                I, W = cuda(ids[a:b]), cuda(w[a:b], torch.float32)
                out = torch.empty_like(X)
                layer.forward_given_routing(X, I, W, out=out)
                st.synchronize()
                barrier.wait()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=st, capture_error_mode="thread_local"):
                    layer.forward_given_routing(X, I, W, out=out)
                barrier.wait()
                for rep in range(3):
                    X.mul_(-1 if rep % 2 else 1.5)  # new values, same buffers
                    barrier.wait()
                    graph.replay()
                    st.synchronize()
                    got = out.clone()
                    barrier.wait()
                    want = layer.forward_given_routing(X, I, W)
                    st.synchronize()
                    barrier.wait()
                    assert torch.equal(got, want), (r, rep)
                ok[r] = True
        except Exception as e:  # surface thread failures
            errs.append(e)
            barrier.abort()

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(nd)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=180)
    assert not errs, errs
    assert all(ok)


@pytest.mark.parametrize("ne,k,nd,dm,dh,act,n,srcmode", [(8, 2, 2, 256, 512, "silu", 1000, "rr"),
                                                         (64, 8, 8, 256, 256, "swiglu", 3000, "random"),
                                                         (60, 4, 4, 128, 256, "relu", 777, "random"),
                                                         (8, 2, 1, 512, 1024, "silu", 4097, "rr"),
                                                         (16, 3, 4, 128, 128, "identity", 1, "rr"),
                                                         (64, 6, 8, 128, 128, "silu", 70000, "random")])
def test_fused_plan_kernel_equals_multi_kernel_chain(ne, k, nd, dm, dh, act, n, srcmode):
    """The one-GPU index chain as one cooperative kernel (occ_plan.cu, the
    default) equals the multi-kernel chain bit for bit: layer output, inbox
    records, BRIM1, CommReport, and the backward that consumes the saved
    grouping."""
    gated = act == "swiglu"
    x, g, w1, w2, w3 = make_layer_inputs(ne + n, n, dm, dh, ne, gated=gated)
    ids, w = random_routing(n, ne, k, np.random.default_rng(n))
    plist = _placement(ne, nd, "shuffled", seed=n)
    src = None if srcmode == "rr" else cuda(np.random.default_rng(1).integers(0, nd, n).astype(np.int32))
    up = cuda(np.random.default_rng(2).uniform(-1, 1, (n, dm)), torch.bfloat16)
    res = []
    for fused in (True, False):
        layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act),
                                        occ.Placement([list(map(int, p)) for p in plist]))
        layer.set_plan_kernels(fused)
        layer.set_training(True)
        layer.load_experts(cuda(w1, torch.bfloat16), cuda(w2, torch.bfloat16), cuda(w3, torch.bfloat16) if gated else None)
        out = layer.forward_given_routing(cuda(x, torch.bfloat16), cuda(ids), cuda(w, torch.float32), src)
        rep = layer.comm_report(bytes_per_scalar=2)
        idx = [t.cpu() for t in layer.saved_index()[:4]]
        gr = layer.backward(up)
        res.append((out.cpu(), rep, idx, {kk: v.cpu() for kk, v in gr.items() if v is not None}))
    (o1, r1, i1, g1), (o2, r2, i2, g2) = res
    assert torch.equal(o1, o2)
    assert r1 == r2
    for a, b in zip(i1, i2):
        assert torch.equal(a, b)
    for kk in g1:
        assert torch.equal(g1[kk], g2[kk]), kk
