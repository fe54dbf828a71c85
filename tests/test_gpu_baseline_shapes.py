"""Value parity at every BASELINE.json configuration, at its full size.

The layer runs exactly as bench.py runs it (same shapes, token counts,
activation, shared experts, pruning, production tcgen05 router, weight scaling)
through forward_expert_parallel; a sample of output rows is checked against the
fp64 oracle (oracle/occ_oracle.c orc_dense_rows_bf16 = dense_given_routing,
pipeline.cpp:542-562, + the shared-expert restatement) evaluated on the SAME
routing the layer used.  Rows are independent given routing
(pipeline.cpp:548-560), so a sample of rows of the full-size batch is a
full-size check of every kernel configuration the batch exercises (the
whole-expert raster bands of D, F >= 4096, the wide 256x512 tiles, the Qwen
shared expert at F_s = 5632, 64-expert groupings).  Bar: max_rel_error
(matrix.cpp:52-60) <= 1e-2 for the forward, 2e-2 for gradients.
The backward at OLMoE's real D/F runs against the reference's own
backward_vjps (2-matrix SiLU experts: the reference has no gated experts) and,
for the SwiGLU extension, against torch autograd in fp64.
"""
import time

import numpy as np
import pytest
import torch

import paper_2505_13345_b200 as occ
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-2
GTOL = 2e-2
SAMPLE = 48


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def uniform_bf16(shape, scale, gen):
    t = torch.empty(shape, dtype=torch.float32, device="cuda").uniform_(-1, 1, generator=gen)
    return t.mul_(scale).to(torch.bfloat16)


# (name, E, k, N_d simulated, D, F, act, tokens, shared (S, F_s, gated?), prune, placement)
CONFIGS = [
    ("c1", 8, 2, 2, 512, 1024, "silu", 2048, None, None, "trivial"),
    ("mixtral_ep1", 8, 2, 1, 4096, 14336, "swiglu", 16384, None, None, "trivial"),
    ("mixtral_ep8", 8, 2, 8, 4096, 14336, "swiglu", 16384, None, None, "shuffled"),
    ("deepseek", 64, 6, 8, 2048, 1408, "swiglu", 16384, (2, 1408, False), None, "shuffled"),
    ("qwen_ep4", 60, 4, 4, 2048, 1408, "swiglu", 16384, (1, 5632, True), ("router", 2), "shuffled"),
    ("olmoe", 64, 8, 8, 2048, 1024, "swiglu", 65536, None, None, "shuffled"),
]


@pytest.mark.parametrize("name,ne,k,nd,dm,dh,act,n,shared,prune,pl", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_baseline_shape_forward_values(name, ne, k, nd, dm, dh, act, n, shared, prune, pl):
    gen = torch.Generator(device="cuda").manual_seed(ne * 1000 + dm)
    gated = act == "swiglu"
    plist = np.arange(ne, dtype=np.int32).reshape(nd, ne // nd)
    if pl == "shuffled":
        plist = np.random.default_rng(ne + nd).permutation(ne).astype(np.int32).reshape(nd, ne // nd)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act),
                                    occ.Placement([list(map(int, r)) for r in plist]))
    w1 = uniform_bf16((ne, dm, dh), dm ** -0.5, gen)
    w3 = uniform_bf16((ne, dm, dh), dm ** -0.5, gen) if gated else None
    w2 = uniform_bf16((ne, dh, dm), dh ** -0.5, gen)
    layer.load_experts(w1, w2, w3)
    sh = None
    if shared:
        ns, fs, with_gate = shared
        sh = {"w1": uniform_bf16((ns, dm, fs), dm ** -0.5, gen),
              "w3": uniform_bf16((ns, dm, fs), dm ** -0.5, gen) if gated else None,
              "w2": uniform_bf16((ns, fs, dm), (ns * fs) ** -0.5, gen),
              "gate": uniform_bf16((dm,), dm ** -0.5, gen) if with_gate else None}
        layer.load_shared_experts(sh["w1"], sh["w2"], sh["w3"], sh["gate"])
    x = uniform_bf16((n, dm), 1.0, gen)
    gate = uniform_bf16((ne, dm), 3.0 / dm ** 0.5, gen)
    spec = occ.PruneSpec(prune[0], prune[1]) if prune else None
    layer.set_validate(False)  # the bench's asynchronous mode
    out = layer.forward_expert_parallel(x, gate, prune=spec)
    ids, w = layer.route(x, gate, prune=spec)  # deterministic: the routing the forward used
    torch.cuda.synchronize()
    if prune:  # collaboration pruning really capped every token's device span
        dev_of = torch.from_numpy(np.argsort(plist.reshape(-1)) // (ne // nd)).cuda()
        span = torch.stack([(dev_of[ids.long()] == d).any(1) for d in range(nd)], 1).sum(1)
        assert int(span.max()) <= prune[1]
    rng = np.random.default_rng(n + ne)
    rows = np.unique(np.concatenate([[0, n - 1], rng.choice(n, SAMPLE, replace=False)])).astype(np.int32)
    t0 = time.time()
    want = O.dense_rows_bf16(x, ids.cpu().numpy(), w.cpu().numpy(), w1, w2, rows, act=act, w3=w3, shared=sh)
    oracle_s = time.time() - t0
    got = out[torch.from_numpy(rows).cuda().long()].double().cpu().numpy()
    err = rel_err(got, want)
    print(f"{name}: n={n} rows={len(rows)} max_rel_error={err:.3e} oracle {oracle_s:.1f}s (8 host threads)")
    assert err <= TOL, err


def test_olmoe_shape_backward_vs_reference():
    """C4's backward at OLMoE's real D = 2048 / F = 1024, 64 experts top-8 over
    8 simulated devices, against the reference's backward_vjps
    (backward.cpp:24-161) in fp64 on identical bf16-representable inputs
    (2-matrix SiLU experts; reduced token count: the reference is a scalar CPU
    loop)."""
    ne, k, nd, dm, dh, n = 64, 8, 8, 2048, 1024, 64
    rng = np.random.default_rng(64)
    bf = lambda a: torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy()
    x = bf(rng.uniform(-1, 1, (n, dm)))
    w1 = bf(rng.uniform(-1, 1, (ne, dm, dh)).astype(np.float32) * dm ** -0.5)
    w2 = bf(rng.uniform(-1, 1, (ne, dh, dm)).astype(np.float32) * dh ** -0.5)
    ids = np.stack([rng.permutation(ne)[:k] for _ in range(n)]).astype(np.int32)
    w = rng.uniform(0.05, 1.0, (n, k))
    w = (w / w.sum(1, keepdims=True)).astype(np.float32).astype(np.float64)
    plist = rng.permutation(ne).astype(np.int32).reshape(nd, ne // nd)
    src = (np.arange(n) % nd).astype(np.int32)
    up = bf(rng.uniform(-1, 1, (n, dm)))
    t0 = time.time()
    rgx, rgw1, rgw2, rgr = O.ref_backward(x, ids, w, w1, w2, plist, src, up, act="silu")
    ref_s = time.time() - t0
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"),
                                    occ.Placement([list(map(int, r)) for r in plist]))
    layer.set_training(True)
    layer.load_experts(torch.from_numpy(w1).cuda().to(torch.bfloat16), torch.from_numpy(w2).cuda().to(torch.bfloat16))
    layer.forward_given_routing(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(ids).cuda(),
                                torch.from_numpy(w).cuda().float(), torch.from_numpy(src).cuda())
    gr = layer.backward(torch.from_numpy(up).cuda().to(torch.bfloat16))
    used = np.unique(ids)
    errs = {"x": rel_err(gr["x"].cpu().numpy(), rgx),
            "w1": rel_err(gr["w1"].cpu().numpy()[used], rgw1[used]),
            "w2": rel_err(gr["w2"].cpu().numpy()[used], rgw2[used]),
            "routing": rel_err(gr["routing_weights"].cpu().numpy(), rgr)}
    print(f"olmoe backward: {errs} (reference {ref_s:.1f}s)")
    assert max(errs.values()) <= GTOL, errs


def test_olmoe_shape_swiglu_backward_vs_autograd():
    """The SwiGLU extension's backward at OLMoE's D/F (64 experts top-8, EP=8
    simulated) against torch autograd in fp64 on the CPU (the reference has no
    gated experts)."""
    ne, k, nd, dm, dh, n = 64, 8, 8, 2048, 1024, 192
    gen = torch.Generator().manual_seed(5)
    bf = lambda shape, s: (torch.rand(shape, generator=gen) * 2 - 1).mul_(s).to(torch.bfloat16)
    x, up = bf((n, dm), 1.0), bf((n, dm), 1.0)
    w1, w3, w2 = bf((ne, dm, dh), dm ** -0.5), bf((ne, dm, dh), dm ** -0.5), bf((ne, dh, dm), dh ** -0.5)
    ids = torch.stack([torch.randperm(ne, generator=gen)[:k] for _ in range(n)]).int()
    w = torch.rand((n, k), generator=gen) + 0.05
    w = (w / w.sum(1, keepdim=True)).float()
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="swiglu"))
    layer.set_training(True)
    layer.load_experts(w1.cuda(), w2.cuda(), w3.cuda())
    layer.forward_given_routing(x.cuda(), ids.cuda(), w.cuda())
    gr = layer.backward(up.cuda())
    X = x.double().requires_grad_()
    W1, W3, W2 = (t.double().requires_grad_() for t in (w1, w3, w2))
    Wt = w.double().requires_grad_()
    Y = torch.zeros((n, dm), dtype=torch.float64)
    for e in ids.unique().tolist():
        t, j = (ids == e).nonzero(as_tuple=True)
        xe = X[t]
        h = torch.nn.functional.silu(xe @ W1[e]) * (xe @ W3[e])
        Y = Y.index_add(0, t, (h @ W2[e]) * Wt[t, j].unsqueeze(1))
    (Y * up.double()).sum().backward()
    used = ids.unique().long()
    errs = {"x": rel_err(gr["x"].cpu(), X.grad), "w1": rel_err(gr["w1"].cpu()[used], W1.grad[used]),
            "w3": rel_err(gr["w3"].cpu()[used], W3.grad[used]), "w2": rel_err(gr["w2"].cpu()[used], W2.grad[used]),
            "routing": rel_err(gr["routing_weights"].cpu(), Wt.grad)}
    print(f"olmoe swiglu backward: {errs}")
    assert max(errs.values()) <= GTOL, errs
