"""Multi-process expert parallelism on one GPU: world_size processes, each an
EP rank with its own handle, bootstrapped by occ_comm_init_host over
torch.distributed (gloo) -- no NCCL, which refuses two ranks on one device --
with the fused exchange over CUDA IPC peer mappings between the processes
(occ_comm_enable_peer).  Outputs against the reference's forward_given_routing
with sources = owning rank (all_to_all_exchange semantics,
pipeline.cpp:125-176 / :456-466), gradients against its backward_vjps, and the
peer-mode forward captured as a CUDA graph replaying bit-identically."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bf16(a):
    import torch
    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("world,ne,k", [(2, 8, 2), (4, 16, 4)])
def test_multi_process_ipc_peer_exchange(tmp_path, world, ne, k):
    dm, dh = 128, 256
    n_per = np.array([37, 64, 5, 100][:world])
    n = int(n_per.sum())
    rng = np.random.default_rng(world)
    x = _bf16(rng.uniform(-1, 1, (n, dm)))
    w1 = _bf16(rng.uniform(-1, 1, (ne, dm, dh)) / np.sqrt(dm))
    w2 = _bf16(rng.uniform(-1, 1, (ne, dh, dm)) / np.sqrt(dh))
    ids = np.stack([rng.permutation(ne)[:k] for _ in range(n)]).astype(np.int32)
    w = rng.uniform(0.05, 1, (n, k))
    w = (w / w.sum(1, keepdims=True)).astype(np.float32).astype(np.float64)
    plist = rng.permutation(ne).astype(np.int32).reshape(world, ne // world)
    up = _bf16(rng.uniform(-1, 1, (n, dm)))
    np.savez(tmp_path / "inputs.npz", x=x, ids=ids, w=w, w1=w1, w2=w2, plist=plist, up=up, n_per=n_per)
    port = _free_port()
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "ipc_worker.py"), str(r), str(world),
                               str(port), str(tmp_path)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out.decode(errors="replace"))
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    src = np.concatenate([np.full(c, r, np.int32) for r, c in enumerate(n_per)])
    R = O.Ref() if O.ref_available() else O.Port()
    want, rep = R.forward_given_routing(x, ids, w, w1, w2, plist, src, act="silu", single=False, bytes_per_scalar=2)
    rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
    host = np.concatenate([r["out_host"] for r in res])
    assert rel(host, want) <= 1e-2
    for key in ("out_peer0", "out_peer1", "out_graph0", "out_graph1", "out_graph2"):
        got = np.concatenate([r[key] for r in res])
        assert np.array_equal(got, host), key  # same kernels and order: identical to the host-staged path
    assert int(res[0]["cross_bytes"]) == rep.cross_device_bytes
    rgx, rgw1, rgw2, rgr = O.ref_backward(x, ids, w, w1, w2, plist, src, up, act="silu")
    gx = np.concatenate([r["g_x"] for r in res])
    gr = np.concatenate([r["g_routing_weights"] for r in res])
    gw1, gw2 = np.zeros_like(rgw1), np.zeros_like(rgw2)
    for r in range(world):
        gw1[plist[r]] = res[r]["g_w1"]
        gw2[plist[r]] = res[r]["g_w2"]
    errs = {"x": rel(gx, rgx), "w1": rel(gw1, rgw1), "w2": rel(gw2, rgw2), "routing": rel(gr, rgr)}
    assert max(errs.values()) <= 2e-2, errs
