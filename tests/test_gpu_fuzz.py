"""GPU fuzz: random layer configurations (experts, top-k, EP degree, widths,
token counts, activation, dedup / replicate-k, placement, shared experts)
through forward_given_routing against the oracle restatement; shapes cover
both GEMM kernels (256 x 256 and 256 x 512 super-tiles), ragged tails and
single-token batches."""
import numpy as np
import pytest
import torch

import paper_2505_13345_b200 as occ
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("seed", range(48))
def test_random_layer_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    nd = int(rng.choice([1, 2, 4]))
    per = int(rng.choice([1, 2, 3, 4, 8]))
    ne = nd * per
    k = int(rng.integers(1, min(ne, 6) + 1))
    act = str(rng.choice(["silu", "relu", "identity", "swiglu"]))
    gated = act == "swiglu"
    dm = int(rng.choice([64, 96, 256, 1024]))
    dh = int(rng.choice([128, 256, 512, 1024])) if gated else int(rng.choice([72, 128, 320, 1024]))
    n = int(rng.choice([1, 37, 256, 513]))
    dedup = bool(rng.integers(0, 2))
    shared = int(rng.choice([0, 0, 1, 2]))
    x = _bf16(rng.uniform(-1, 1, (n, dm)))
    w1 = _bf16(rng.uniform(-1, 1, (ne, dm, dh)) / np.sqrt(dm))
    w3 = _bf16(rng.uniform(-1, 1, (ne, dm, dh)) / np.sqrt(dm)) if gated else None
    w2 = _bf16(rng.uniform(-1, 1, (ne, dh, dm)) / np.sqrt(dh))
    ids = np.stack([rng.permutation(ne)[:k] for _ in range(n)]).astype(np.int32)
    w = rng.uniform(0.05, 1.0, (n, k))
    w = (w / w.sum(1, keepdims=True)).astype(np.float32).astype(np.float64)
    plist = rng.permutation(ne).astype(np.int32).reshape(nd, per)
    src = rng.integers(0, nd, n).astype(np.int32)
    a = "silu" if gated else act
    want, _ = O.Port().forward_given_routing(x, ids, w, w1, w2, plist, src, act=a, single=False, w3=w3)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act, dedup=dedup),
                                    occ.Placement([list(r) for r in plist]))
    C = lambda v, dt=None: (lambda t: t.to(dt) if dt is not None else t)(torch.from_numpy(np.ascontiguousarray(v)).cuda())
    layer.load_experts(C(w1, torch.bfloat16), C(w2, torch.bfloat16), C(w3, torch.bfloat16) if gated else None)
    if shared:
        fs = 128 if gated else 64
        s1 = _bf16(rng.uniform(-1, 1, (shared, dm, fs)) / np.sqrt(dm))
        s3 = _bf16(rng.uniform(-1, 1, (shared, dm, fs)) / np.sqrt(dm)) if gated else None
        s2 = _bf16(rng.uniform(-1, 1, (shared, fs, dm)) / np.sqrt(fs * shared))
        sg = _bf16(rng.uniform(-1, 1, dm) / np.sqrt(dm)) if seed % 2 else None
        layer.load_shared_experts(C(s1, torch.bfloat16), C(s2, torch.bfloat16),
                                  C(s3, torch.bfloat16) if gated else None,
                                  C(sg, torch.bfloat16) if sg is not None else None)
        want = O.Port().shared_experts(x, s1, s2, w3=s3, gate=sg, act=a, out=want)
    out = layer.forward_given_routing(C(x, torch.bfloat16), C(ids), C(w, torch.float32), C(src))
    got = out.double().cpu().numpy()
    err = float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))
    assert err <= 1e-2, (seed, dict(nd=nd, ne=ne, k=k, act=act, dm=dm, dh=dh, n=n, dedup=dedup, shared=shared), err)


@pytest.mark.parametrize("seed", range(16))
def test_random_wide_routing_vs_oracle(seed):
    """Large routing shapes up to the device path's limits: E <= 256, up to
    64 experts per device, top-k up to 64, up to 64 devices."""
    rng = np.random.default_rng(5000 + seed)
    while True:
        nd = int(rng.choice([1, 2, 4, 8, 16, 64]))
        per = int(rng.choice([1, 4, 16, 32, 64]))
        if nd * per <= 256:
            break
    ne = nd * per
    k = int(rng.integers(1, min(ne, 64) + 1))
    act = str(rng.choice(["silu", "relu", "identity"]))
    dm, dh = int(rng.choice([32, 64, 128])), int(rng.choice([32, 64, 128]))
    n = int(rng.choice([1, 100, 300]))
    dedup = bool(rng.integers(0, 2))
    x = _bf16(rng.uniform(-1, 1, (n, dm)))
    w1 = _bf16(rng.uniform(-1, 1, (ne, dm, dh)) / np.sqrt(dm))
    w2 = _bf16(rng.uniform(-1, 1, (ne, dh, dm)) / np.sqrt(dh))
    ids = np.stack([rng.permutation(ne)[:k] for _ in range(n)]).astype(np.int32)
    w = rng.uniform(0.05, 1.0, (n, k))
    w = (w / w.sum(1, keepdims=True)).astype(np.float32).astype(np.float64)
    plist = rng.permutation(ne).astype(np.int32).reshape(nd, per)
    src = rng.integers(0, nd, n).astype(np.int32)
    want, rep = O.Port().forward_given_routing(x, ids, w, w1, w2, plist, src, act=act, single=False,
                                               bytes_per_scalar=2)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act, dedup=dedup),
                                    occ.Placement([list(r) for r in plist]))
    C = lambda v, dt=None: (lambda t: t.to(dt) if dt is not None else t)(torch.from_numpy(np.ascontiguousarray(v)).cuda())
    layer.load_experts(C(w1, torch.bfloat16), C(w2, torch.bfloat16))
    out = layer.forward_given_routing(C(x, torch.bfloat16), C(ids), C(w, torch.float32), C(src))
    got = out.double().cpu().numpy()
    err = float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))
    assert err <= 1e-2, (seed, ne, k, nd, dedup, err)
    r = layer.comm_report(bytes_per_scalar=2)
    assert r.mean_replicas == rep.mean_replicas
    if dedup:
        assert r.cross_device_bytes == rep.cross_device_bytes
