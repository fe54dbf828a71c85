"""Generate tests/golden/golden.json from the REFERENCE itself.

Runs the reference library compiled from /root/reference sources
(oracle/_ref/libmoesim_ref.so, see oracle/Makefile) on (a) the fixtures of
the reference's own unit tests (cited per case) and (b) seeded random
instances, and records inputs + outputs.  The committed JSON lets the CPU
suite pin the oracle restatement (and the GPU suite pin the device path)
where /root/reference is absent, e.g. on the GPU box.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

R = O.Ref()


def L(a):
    return np.asarray(a).tolist()


def topk_cases():
    out = []
    # test_routing.cpp:64-99
    for scores, k, ren, cite in [([[0.1, 0.4, 0.3, 0.2]], 4, False, "test_routing.cpp:64-73"),
                                 ([[0.1, 0.4, 0.4, 0.1]], 2, False, "test_routing.cpp:75-83"),
                                 ([[0.7, 0.1, 0.15, 0.05]], 2, True, "test_routing.cpp:85-99")]:
        ids, w = R.topk_route(np.array(scores), k, ren)
        out.append({"cite": cite, "scores": scores, "k": k, "renormalize": ren, "ids": L(ids), "weights": L(w)})
    rng = np.random.default_rng(2201)
    for e, k in [(8, 2), (64, 8), (60, 4), (16, 16)]:
        s = np.round(rng.uniform(size=(40, e)), 3)  # rounding creates ties
        ids, w = R.topk_route(s, k, True)
        out.append({"cite": "random, seed 2201", "scores": L(s), "k": k, "renormalize": True, "ids": L(ids),
                    "weights": L(w)})
    return out


def gate_cases():
    out = []
    x, g, *_ = O.synthetic_layer(21, 16, 24, 8, 8, single=False)
    out.append({"cite": "gate_scores routing.cpp:33-52, seed 21", "x": L(x), "gate": L(g),
                "scores": L(R.gate_scores(x, g))})
    return out


def dispatch_cases():
    out = []
    # test_pipeline.cpp:83-95 and pipeline.hpp:17-27 worked example
    for ids, ne, nd, cite in [([[0, 1], [2, 3], [1, 2]], 4, 1, "test_pipeline.cpp:83-88"),
                              ([[0, 1], [0, 2], [2, 3]], 4, 2, "test_pipeline.cpp:90-95")]:
        ids = np.array(ids, np.int32)
        w = np.full(ids.shape, 0.5)
        x = np.zeros((len(ids), 8))
        plist = np.arange(ne, dtype=np.int32).reshape(nd, ne // nd)
        _, rep, idx = R.forward_given_routing(x, ids, w, np.zeros((ne, 8, 8)), np.zeros((ne, 8, 8)), plist,
                                              np.zeros(len(ids), np.int32), act="identity", single=False,
                                              want_index=True)
        out.append({"cite": cite, "ids": L(ids), "ne": ne, "nd": nd, "sources": [0] * len(ids),
                    "dindex": [L(d) for d in idx["dindex"]], "n_sfd": [rep.n_sfd_src[s] for s in range(nd)]})
    return out


def forward_cases():
    out = []
    rng = np.random.default_rng(77)
    for (ne, k, nd, dm, dh, n, act, single) in [(8, 3, 4, 6, 10, 9, "identity", True), (8, 2, 2, 4, 6, 10, "silu", True),
                                                (4, 4, 2, 3, 5, 5, "relu", False), (16, 4, 4, 8, 8, 17, "silu", False)]:
        x, g, w1, w2, _ = O.synthetic_layer(int(rng.integers(1 << 30)), n, dm, dh, ne, single=single)
        s = R.gate_scores(x, g)
        ids, w = R.topk_route(s, k, True)
        plist = rng.permutation(ne).astype(np.int32).reshape(nd, ne // nd)
        src = (np.arange(n) % nd).astype(np.int32)
        y, rep, idx = R.forward_given_routing(x, ids, w, w1, w2, plist, src, act=act, single=single,
                                              bytes_per_scalar=4, want_index=True)
        out.append({"cite": "forward_given_routing pipeline.cpp:360-501", "ne": ne, "k": k, "nd": nd, "act": act,
                    "single": single, "x": L(x), "ids": L(ids), "w": L(w), "w1": L(w1), "w2": L(w2),
                    "plist": L(plist), "sources": L(src), "y": L(y),
                    "report": {"mean_replicas": rep.mean_replicas, "intra_share": rep.intra_share,
                               "inter_share": rep.inter_share, "cross_device_bytes": rep.cross_device_bytes,
                               "per_device_rows": [rep.per_device_rows[d] for d in range(nd)]},
                    "dindex": [L(d) for d in idx["dindex"]], "inbox": [L(b) for b in idx["inbox"]],
                    "cindex": [L(c) for c in idx["cindex"]]})
    return out


def collab_cases():
    out = []
    # test_collab.cpp:56-66, :81-87
    ids = np.array([[0, 1], [0, 1], [1, 2]], np.int32)
    c = R.accumulate_collab(ids, 3)
    out.append({"cite": "test_collab.cpp:56-66", "ids": L(ids), "ne": 3, "counts": L(c),
                "norm": L(R.normalize_graph(c))})
    rng = np.random.default_rng(31)
    ids = np.stack([rng.permutation(12)[:4] for _ in range(50)]).astype(np.int32)
    c = R.accumulate_collab(ids, 12)
    out.append({"cite": "random, seed 31", "ids": L(ids), "ne": 12, "counts": L(c), "norm": L(R.normalize_graph(c))})
    return out


def placement_cases():
    out = []
    # test_placement.cpp:50-56 worked example
    p = np.zeros((4, 4))
    for i, j, v in [(0, 1, 1.0), (0, 2, 0.2), (0, 3, 0.1), (1, 2, 0.3), (1, 3, 0.2), (2, 3, 0.9)]:
        p[i, j] = p[j, i] = v
    out.append({"cite": "test_placement.cpp:50-56", "p": L(p), "nd": 2, "placement": L(R.reschedule_placement(p, 2))})
    out.append({"cite": "test_placement.cpp:58-61", "p": L(np.zeros((4, 4))), "nd": 2,
                "placement": L(R.reschedule_placement(np.zeros((4, 4)), 2))})
    rng = np.random.default_rng(41)
    for nd, per in [(1, 4), (3, 1), (4, 16), (8, 8), (2, 5)]:
        ne = nd * per
        a = rng.uniform(size=(ne, ne))
        a = np.triu(a, 1)
        a = a + a.T
        out.append({"cite": "random, seed 41", "p": L(a), "nd": nd, "placement": L(R.reschedule_placement(a, nd))})
    return out


def prune_cases():
    out = []
    # test_pruning.cpp:73-79 (router worked example), :99-112 (similarity worked example)
    plist = np.arange(4, dtype=np.int32).reshape(2, 2)
    s = np.array([[0.3, 0.05, 0.5, 0.15]])
    ids, w = R.topk_route(s, 2, False)
    gi, gw = R.prune_routing(s, ids, w, plist, "router", 1, renormalize=False)
    out.append({"cite": "test_pruning.cpp:73-79", "scores": L(s), "ids": L(ids), "w": L(w), "plist": L(plist),
                "mode": "router", "budget": 1, "sim": None, "own": False, "renorm": False, "out_ids": L(gi),
                "out_w": L(gw)})
    table = np.array([[1.0, 0.9, 0.1, 0.5], [0.9, 1.0, 0.2, 0.3], [0.1, 0.2, 1.0, 0.8], [0.5, 0.3, 0.8, 1.0]])
    ids = np.array([[2, 0]], np.int32)
    w = np.array([[0.5, 0.3]])
    gi, gw = R.prune_routing(s, ids, w, plist, "similarity", 1, sim_values=table, renormalize=False)
    out.append({"cite": "test_pruning.cpp:99-112", "scores": L(s), "ids": L(ids), "w": L(w), "plist": L(plist),
                "mode": "similarity", "budget": 1, "sim": L(table), "own": False, "renorm": False, "out_ids": L(gi),
                "out_w": L(gw)})
    rng = np.random.default_rng(52)
    for mode, own, ne, nd, k, b in [("router", False, 16, 4, 4, 2), ("similarity", False, 16, 4, 4, 2),
                                    ("similarity", True, 16, 4, 3, 1), ("router", False, 64, 8, 8, 2)]:
        s = rng.uniform(size=(20, ne))
        s /= s.sum(1, keepdims=True)
        ids, w = R.topk_route(s, k, True)
        plist = rng.permutation(ne).astype(np.int32).reshape(nd, ne // nd)
        sim, _ = R.similarity_table(np.log(s))
        gi, gw = R.prune_routing(s, ids, w, plist, mode, b, sim_values=sim if mode == "similarity" else None,
                                 own_score=own)
        out.append({"cite": "random, seed 52", "scores": L(s), "ids": L(ids), "w": L(w), "plist": L(plist),
                    "mode": mode, "budget": b, "sim": L(sim) if mode == "similarity" else None, "own": own,
                    "renorm": True, "out_ids": L(gi), "out_w": L(gw)})
    return out


def main():
    g = {"generator": "tests/golden/make_golden.py over oracle/_ref/libmoesim_ref.so (reference sources)",
         "topk": topk_cases(), "gate": gate_cases(), "dispatch": dispatch_cases(), "forward": forward_cases(),
         "collab": collab_cases(), "placement": placement_cases(), "prune": prune_cases()}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
