"""CPU suite: the oracle restatement (oracle/occ_oracle.c) pinned against the
reference's golden vectors (tests/golden/golden.json, generated from the
reference itself) and, where the reference was compiled (oracle/_ref), live
against the reference on seeded random instances including the edge cases
the reference tests (empty batch, k = E, one device, one expert per device,
ties, capacity errors)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
P = O.Port()
have_ref = os.path.exists(O.REF_SO) or os.path.isdir("/root/reference/proj/src")
needs_ref = pytest.mark.skipif(not have_ref, reason="reference not compiled here")


def A(x, dt=np.float64):
    return np.asarray(x, dtype=dt)


@pytest.mark.parametrize("case", GOLD["topk"], ids=lambda c: c["cite"])
def test_topk_golden(case):
    ids, w = P.topk_route(A(case["scores"]), case["k"], case["renormalize"])
    assert ids.tolist() == case["ids"]
    assert np.array_equal(w, A(case["weights"]))


def test_gate_golden():
    c = GOLD["gate"][0]
    assert np.array_equal(P.gate_scores(A(c["x"]), A(c["gate"])), A(c["scores"]))


@pytest.mark.parametrize("case", GOLD["dispatch"], ids=lambda c: c["cite"])
def test_dispatch_golden(case):
    ids = A(case["ids"], np.int32)
    ne, nd = case["ne"], case["nd"]
    plist = np.arange(ne, dtype=np.int32).reshape(nd, ne // nd)
    _, rep, idx = P.forward_given_routing(np.zeros((len(ids), 8)), ids, np.full(ids.shape, 0.5), np.zeros((ne, 8, 8)),
                                          np.zeros((ne, 8, 8)), plist, A(case["sources"], np.int32),
                                          act="identity", single=False, want_index=True)
    assert [d.tolist() for d in idx["dindex"]] == case["dindex"]
    assert [rep.n_sfd_src[s] for s in range(nd)] == case["n_sfd"]


@pytest.mark.parametrize("case", GOLD["forward"], ids=lambda c: f"{c['ne']}e{c['k']}k{c['nd']}d-{c['act']}")
def test_forward_golden(case):
    y, rep, idx = P.forward_given_routing(A(case["x"]), A(case["ids"], np.int32), A(case["w"]), A(case["w1"]),
                                          A(case["w2"]), A(case["plist"], np.int32), A(case["sources"], np.int32),
                                          act=case["act"], single=case["single"], want_index=True)
    assert np.array_equal(y, A(case["y"]))  # bit-exact in double
    r = case["report"]
    assert rep.mean_replicas == r["mean_replicas"]
    assert (rep.intra_share, rep.inter_share) == (r["intra_share"], r["inter_share"])
    assert rep.cross_device_bytes == r["cross_device_bytes"]
    assert [d.tolist() for d in idx["dindex"]] == case["dindex"]
    assert [b.tolist() for b in idx["inbox"]] == case["inbox"]
    assert [c.tolist() for c in idx["cindex"]] == case["cindex"]


@pytest.mark.parametrize("case", GOLD["collab"], ids=lambda c: c["cite"])
def test_collab_golden(case):
    c = P.accumulate_collab(A(case["ids"], np.int32), case["ne"])
    assert c.tolist() == case["counts"]
    assert np.array_equal(P.normalize_graph(c), A(case["norm"]))


@pytest.mark.parametrize("case", GOLD["placement"], ids=lambda c: c["cite"])
def test_placement_golden(case):
    assert P.reschedule_placement(A(case["p"]), case["nd"]).tolist() == case["placement"]


@pytest.mark.parametrize("case", GOLD["prune"], ids=lambda c: c["cite"] + c["mode"])
def test_prune_golden(case):
    gi, gw = P.prune_routing(A(case["scores"]), A(case["ids"], np.int32), A(case["w"]), A(case["plist"], np.int32),
                             case["mode"], case["budget"], sim_values=None if case["sim"] is None else A(case["sim"]),
                             own_score=case["own"], renormalize=case["renorm"])
    assert gi.tolist() == case["out_ids"]
    assert np.array_equal(gw, A(case["out_w"]))


def test_rng_matches_mt19937_64():
    r = O.Rng(5489)
    # std::mt19937_64 default-seed 10000th output (C++ standard [rand.predef])
    for _ in range(9999):
        r.next()
    assert r.next() == 9981545732273789042


# ------------------------------------------------------- live vs reference --

@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_forward_matches_reference_live(seed):
    rng = np.random.default_rng(seed)
    nd = int(rng.integers(1, 5))
    per = int(rng.integers(1, 5))
    ne = nd * per
    k = int(rng.integers(1, ne + 1))
    n = int(rng.integers(0, 30))  # includes the empty batch
    dm, dh = int(rng.integers(1, 9)), int(rng.integers(1, 9))
    single = bool(seed % 2)
    act = ["identity", "silu", "relu"][seed % 3]
    x, g, w1, w2, _ = O.synthetic_layer(seed, n, dm, dh, ne, single=single)
    R = O.Ref()
    s = R.gate_scores(x, g) if n else np.zeros((0, ne))
    ids, w = R.topk_route(s, k) if n else (np.zeros((0, k), np.int32), np.zeros((0, k)))
    plist = rng.permutation(ne).astype(np.int32).reshape(nd, per)
    src = rng.integers(0, nd, n).astype(np.int32)
    a = P.forward_given_routing(x, ids, w, w1, w2, plist, src, act=act, single=single, want_index=True)
    b = R.forward_given_routing(x, ids, w, w1, w2, plist, src, act=act, single=single, want_index=True)
    assert np.array_equal(a[0], b[0])
    for key in ("mean_replicas", "intra_share", "inter_share", "cross_device_bytes"):
        assert getattr(a[1], key) == getattr(b[1], key)
    for key in ("dindex", "inbox", "cindex"):
        assert all(np.array_equal(u, v) for u, v in zip(a[2][key], b[2][key]))


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_routing_prune_placement_live(seed):
    R = O.Ref()
    rng = np.random.default_rng(100 + seed)
    nd = int(rng.integers(2, 5))
    per = int(rng.integers(2, 5))
    ne = nd * per
    k = int(rng.integers(1, per + 1))
    s = rng.uniform(size=(25, ne))
    s[::5, :2] = 0.5  # ties
    ids_p, w_p = P.topk_route(s, k)
    ids_r, w_r = R.topk_route(s, k)
    assert np.array_equal(ids_p, ids_r) and np.array_equal(w_p, w_r)
    plist = rng.permutation(ne).astype(np.int32).reshape(nd, per)
    sim_p, rk_p = P.similarity_table(s)
    sim_r, rk_r = R.similarity_table(s)
    assert np.array_equal(sim_p, sim_r) and np.array_equal(rk_p, rk_r)
    for mode in ("router", "similarity"):
        for own in (False, True):
            b = int(rng.integers(1, nd + 1))
            res = []
            for be in (P, R):
                try:
                    res.append(be.prune_routing(s, ids_p, w_p, plist, mode, b,
                                                sim_values=sim_p if mode == "similarity" else None, own_score=own))
                except O.OracleError as e:
                    res.append(e.code)
            if isinstance(res[0], int) or isinstance(res[1], int):
                assert res[0] == res[1]
            else:
                assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    c_p = P.accumulate_collab(ids_p, ne)
    assert np.array_equal(c_p, R.accumulate_collab(ids_p, ne))
    pn = P.normalize_graph(c_p)
    assert np.array_equal(pn, R.normalize_graph(c_p))
    assert np.array_equal(P.reschedule_placement(pn, nd), R.reschedule_placement(pn, nd))


@needs_ref
def test_capacity_error_matches_reference():
    # test_pruning.cpp:92-97
    s = np.array([[0.4, 0.3, 0.2, 0.1]])
    plist = np.arange(4, dtype=np.int32).reshape(2, 2)
    ids, w = P.topk_route(s, 3, False)
    for be in (P, O.Ref()):
        with pytest.raises(O.OracleError) as ei:
            be.prune_routing(s, ids, w, plist, "router", 1, renormalize=False)
        assert ei.value.code == 5


@pytest.mark.parametrize("gated,gate,act", [(True, False, "silu"), (True, True, "silu"), (False, True, "relu"),
                                            (False, False, "identity")])
def test_shared_experts_oracle_vs_torch(gated, gate, act):
    """orc_shared_experts (the DeepSeek/Qwen shared-expert extension, not in
    the reference) pinned against an independent torch fp64 computation."""
    import torch
    rng = np.random.default_rng(5)
    n, dm, dh, ns = 37, 24, 40, 2
    x = rng.uniform(-1, 1, (n, dm))
    w1 = rng.uniform(-1, 1, (ns, dm, dh)) / np.sqrt(dm)
    w3 = rng.uniform(-1, 1, (ns, dm, dh)) / np.sqrt(dm) if gated else None
    w2 = rng.uniform(-1, 1, (ns, dh, dm)) / np.sqrt(dh)
    g = rng.uniform(-1, 1, dm) if gate else None
    base = rng.uniform(-1, 1, (n, dm))
    got = P.shared_experts(x, w1, w2, w3=w3, gate=g, act=act, out=base)
    T = torch.from_numpy
    acc = torch.zeros(n, dm, dtype=torch.float64)
    fn = {"silu": torch.nn.functional.silu, "relu": torch.relu, "identity": lambda v: v}[act]
    for s in range(ns):
        a = T(x) @ T(w1[s])
        h = torch.nn.functional.silu(a) * (T(x) @ T(w3[s])) if gated else fn(a)
        acc += h @ T(w2[s])
    if gate:
        acc *= torch.sigmoid(T(x) @ T(g))[:, None]
    want = base + acc.numpy()
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12


@pytest.mark.parametrize("gated,act,shared,gate", [(True, "silu", 0, False), (False, "silu", 0, False),
                                                   (False, "relu", 2, False), (True, "silu", 2, True)])
def test_dense_rows_bf16_equals_scalar_restatement(gated, act, shared, gate):
    """orc_dense_rows_bf16 (the sampled-row value oracle of the BASELINE-size
    GPU tests: bf16 storage in, rows batched per expert) computes exactly the
    doubles of orc_dense_given_routing + orc_shared_experts (Precision::Double,
    pipeline.cpp:542-562) on the same bf16-representable inputs."""
    import torch
    n, dm, dh, ne, k, dhs = 40, 32, 48, 8, 3, 24
    rng = np.random.default_rng(7)
    bf = lambda a: torch.tensor(a, dtype=torch.float32).to(torch.bfloat16)
    x, w1, w2 = bf(rng.uniform(-1, 1, (n, dm))), bf(rng.uniform(-1, 1, (ne, dm, dh)) / 6), bf(rng.uniform(-1, 1, (ne, dh, dm)) / 7)
    w3 = bf(rng.uniform(-1, 1, (ne, dm, dh)) / 6) if gated else None
    ids = np.stack([rng.permutation(ne)[:k] for _ in range(n)]).astype(np.int32)
    w = rng.uniform(0.1, 1, (n, k)).astype(np.float32)
    rows = np.array([0, 5, 7, 8, 13, 21, 22, 39], np.int32)
    sh = None
    if shared:
        sh = {"w1": bf(rng.uniform(-1, 1, (shared, dm, dhs)) / 6), "w2": bf(rng.uniform(-1, 1, (shared, dhs, dm)) / 5),
              "w3": bf(rng.uniform(-1, 1, (shared, dm, dhs)) / 6) if gated else None,
              "gate": bf(rng.uniform(-1, 1, dm) / 6) if gate else None}
    got = O.dense_rows_bf16(x, ids, w, w1, w2, rows, act=act, w3=w3, shared=sh, threads=3)
    d = lambda t: None if t is None else t.double().numpy()
    P = O.Port()
    want = P.dense_given_routing(d(x), ids, w.astype(np.float64), d(w1), d(w2), act="silu" if gated else act,
                                 single=False, rows=rows, w3=d(w3))
    if sh:
        full = np.zeros((n, dm))
        full[rows] = want
        full = P.shared_experts(d(x), d(sh["w1"]), d(sh["w2"]), w3=d(sh["w3"]), gate=d(sh["gate"]),
                                act="silu" if gated else act, out=full)
        want = full[rows]
    assert np.array_equal(got, want)
