"""One rank of the multi-process test (tests/test_gpu_ipc.py): world_size
processes share ONE GPU, bootstrapped over torch.distributed / gloo through
occ_comm_init_host (no NCCL, which refuses two ranks on one GPU), and run
(a) the forward over the host transport, (b) the fused peer-memory forward
over CUDA IPC mappings (twice: the arrival flags advance), (c) a training
step (forward + backward).  Writes its results to <out>/rank<r>.npz.
Usage: python ipc_worker.py <rank> <world> <port> <out_dir>"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_13345_b200 as occ  # noqa: E402


def main():
    rank, world, port, out_dir = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    d = np.load(os.path.join(out_dir, "inputs.npz"))
    x, ids, w, w1, w2, plist, up, n_per = (d[k] for k in ("x", "ids", "w", "w1", "w2", "plist", "up", "n_per"))
    ne, k = w1.shape[0], ids.shape[1]
    dm, dh = x.shape[1], w1.shape[2]
    starts = np.concatenate([[0], np.cumsum(n_per)])
    a, b = starts[rank], starts[rank + 1]
    bf = lambda arr: torch.from_numpy(np.ascontiguousarray(arr)).cuda().to(torch.bfloat16)
    X, I, W = bf(x[a:b]), torch.from_numpy(ids[a:b]).cuda(), torch.from_numpy(w[a:b]).cuda().float()
    res = {}
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, world, dm, dh, activation="silu"),
                                    occ.Placement([list(map(int, p)) for p in plist]), world_size=world, rank=rank)
    layer.set_training(True)
    layer.load_experts(bf(w1[plist[rank]]), bf(w2[plist[rank]]))
    layer.comm_init_host()
    # (a) host-staged all-to-alls + (c) backward
    res["out_host"] = layer.forward_given_routing(X, I, W).float().cpu().numpy()
    g = layer.backward(bf(up[a:b]))
    for key in ("x", "w1", "w2", "routing_weights"):
        res["g_" + key] = g[key].float().cpu().numpy()
    # (b) fused exchange over CUDA IPC peer mappings between the processes
    layer.comm_enable_peer(int(n_per.max()))
    for rep in range(2):
        res[f"out_peer{rep}"] = layer.forward_given_routing(X, I, W).float().cpu().numpy()
    rep_ = layer.comm_report(bytes_per_scalar=2)
    res["cross_bytes"] = np.array(rep_.cross_device_bytes)
    # (b') peer mode with validation off replays as a CUDA graph, bit-identical
    layer.set_validate(False)
    stream = torch.cuda.Stream()
    out_g = torch.empty_like(X)
    with torch.cuda.stream(stream):
        layer.forward_given_routing(X, I, W, out=out_g)  # warm (eager)
        stream.synchronize()
        graph = torch.cuda.CUDAGraph()
        dist.barrier()
        with torch.cuda.graph(graph, stream=stream):
            layer.forward_given_routing(X, I, W, out=out_g)
    dist.barrier()
    for rep in range(3):
        out_g.zero_()
        graph.replay()
        torch.cuda.synchronize()
        res[f"out_graph{rep}"] = out_g.float().cpu().numpy()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
