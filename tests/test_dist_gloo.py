"""Multi-process (world_size 2 and 4, gloo, CPU) test of the world_size > 1
exchange protocol.

Each process is one EP device owning a contiguous token shard.  It forms its
Sfd batch (BRIM0 of its tokens), all-gathers the per-source count rows, asks
the product's host layout function (occ_exchange_layout, the code that sizes
the NCCL all-to-alls in forward_multi) where every peer's rows go, runs the
dispatch all-to-all and the return all-to-all with point-to-point gloo
messages, and checks that
  * the received inbox equals the reference's all_to_all_exchange inbox for
    this device (token, source, source slot; pipeline.cpp:125-176), and
  * the return exchange delivers every inbox row back to its source's Sfd
    slot, so combine (pipeline.cpp:285-300) sums the right rows.
The BRIM0 stand-in on CPU is the oracle; the device plan kernel that
produces it on the GPU is pinned bit-exact separately
(tests/test_gpu_parity.py::test_dispatch_index_bit_exact)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(world, ne, k, n_per, seed):
    rng = np.random.default_rng(seed)
    n = sum(n_per)
    ids = np.stack([rng.permutation(ne)[:k] for _ in range(n)]).astype(np.int32)
    w = np.full((n, k), 1.0 / k)
    plist = rng.permutation(ne).astype(np.int32).reshape(world, ne // world)
    src = np.concatenate([np.full(c, r, np.int32) for r, c in enumerate(n_per)])
    return ids, w, plist, src


def _worker(rank, world, port, ne, k, n_per, seed, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2505_13345_b200 as occ
        from oracle import oracle as O
        ids, w, plist, src = _problem(world, ne, k, n_per, seed)
        n = ids.shape[0]
        # reference single-process simulation of the whole layer's index state
        _, rep, idx = O.Port().forward_given_routing(np.zeros((n, 1)), ids, w, np.zeros((ne, 1, 1)),
                                                     np.zeros((ne, 1, 1)), plist, src, act="identity",
                                                     single=False, want_index=True)
        toks = np.nonzero(src == rank)[0]
        brim0 = idx["dindex"][rank]                              # nd x n_r, this source
        n_sfd = int((brim0 >= 0).sum())
        sfd_tok = np.empty(n_sfd, np.int64)
        for d in range(world):
            for i, t in enumerate(toks):
                if brim0[d, i] >= 0:
                    sfd_tok[brim0[d, i]] = t
        row = torch.tensor([(brim0[d] >= 0).sum() for d in range(world)], dtype=torch.int32)
        rows = [torch.zeros(world, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(rows, row)
        C = torch.stack(rows).numpy()                            # C[s][d]
        so, sc, ro, rc = occ.exchange_layout(C, rank)
        # dispatch: payload = (token, source, slot)
        send = torch.tensor(np.stack([sfd_tok, np.full(n_sfd, rank), np.arange(n_sfd)], 1), dtype=torch.int64)
        recv = torch.full((int(rc.sum()), 3), -1, dtype=torch.int64)
        _alltoallv(send, so, sc, recv, ro, rc, rank, world)
        want = idx["inbox"][rank].T                              # (token, source, slot) per inbox row
        ok_inbox = recv.numpy().tolist() == want.tolist()
        # return: each inbox row carries token*16 + device back to its source slot
        ret = (recv[:, 0] * 16 + rank).reshape(-1, 1).contiguous()
        y_src = torch.full((n_sfd, 1), -1, dtype=torch.int64)
        _alltoallv(ret, ro, rc, y_src, so, sc, rank, world)
        combined = np.zeros(len(toks), np.int64)
        expect = np.zeros(len(toks), np.int64)
        dev_of = np.empty(ne, int)
        for d, lst in enumerate(plist):
            dev_of[lst] = d
        for i, t in enumerate(toks):
            for d in range(world):
                if brim0[d, i] >= 0:
                    combined[i] += y_src[brim0[d, i], 0].item()
            expect[i] = sum(t * 16 + d for d in sorted(set(dev_of[ids[t]])))
        q.put((rank, ok_inbox, bool(np.array_equal(combined, expect)), int(rc.sum()),
               int(rep.per_device_rows[rank])))
        dist.destroy_process_group()
    except Exception as e:  # report to the parent
        q.put((rank, repr(e), False, -1, -1))


def _alltoallv(send, so, sc, recv, ro, rc, rank, world):
    reqs = []
    for p in range(world):
        if p == rank:
            if sc[p]:
                recv[ro[p]:ro[p] + rc[p]] = send[so[p]:so[p] + sc[p]]
            continue
        if sc[p]:
            reqs.append(dist.isend(send[so[p]:so[p] + sc[p]].contiguous(), p))
        if rc[p]:
            buf = torch.empty((int(rc[p]),) + tuple(recv.shape[1:]), dtype=recv.dtype)
            reqs.append((dist.irecv(buf, p), buf, p))
    for r in reqs:
        if isinstance(r, tuple):
            r[0].wait()
            recv[ro[r[2]]:ro[r[2]] + rc[r[2]]] = r[1]
        else:
            r.wait()


@pytest.mark.parametrize("world,ne,k,n_per", [(2, 8, 2, [40, 25]), (4, 16, 4, [10, 0, 33, 7]),
                                             (2, 64, 8, [64, 64])])
def test_exchange_protocol_multiprocess(world, ne, k, n_per):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ne, k, n_per, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_inbox, ok_comb, got_rows, want_rows in sorted(res):
        assert ok_inbox is True, (rank, ok_inbox)
        assert ok_comb, rank
        assert got_rows == want_rows


def test_exchange_layout_golden():
    import paper_2505_13345_b200 as occ
    C = np.array([[3, 1, 0], [2, 0, 5], [1, 1, 1]])
    so, sc, ro, rc = occ.exchange_layout(C, 1)
    assert so.tolist() == [0, 2, 2] and sc.tolist() == [2, 0, 5]
    assert ro.tolist() == [0, 1, 1] and rc.tolist() == [1, 0, 1]


def _allgather_worker(rank, world, port, q):
    """One rank: the host all-gather callback of occ_comm_init_host (the
    transport that bootstraps the IPC mapping without NCCL), called the way the
    library calls it -- raw pointers through the C function-pointer type."""
    import ctypes as C
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_13345_b200.api import host_allgather_fn
    fn = host_allgather_fn()
    ok = True
    for nbytes in (1, 8, 100, 64 * (world + 3), 0):
        send = (C.c_uint8 * max(nbytes, 1))(*[(rank * 37 + i) % 251 for i in range(max(nbytes, 1))])
        recv = (C.c_uint8 * max(world * nbytes, 1))()
        rc = fn(None, C.addressof(send), nbytes, C.addressof(recv))
        want = [(r * 37 + i) % 251 for r in range(world) for i in range(nbytes)]
        ok &= rc == 0 and list(recv)[:world * nbytes] == want
    dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.parametrize("world", [2, 3])
def test_host_allgather_callback_multiprocess(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_allgather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
