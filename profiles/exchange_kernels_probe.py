"""Exchange-side kernels at a Mixtral-like shape with world_size = 2 loopback
ranks (threads on one GPU): the dispatch pack (`pack_kernel`: each token row
read once, written to its Sfd send rows with the routing metadata), the
intra-device partial combine and the final combine of the returned rows.
Non-peer transport (host barriers, no spin waits), so it is safe under ncu:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      -k regex:"pack_kernel|partial_combine|combine_kernel" python profiles/exchange_kernels_probe.py

With --peer the fused peer-memory path runs instead (timed with CUDA events
around whole forwards).  Under ncu, which serialises the ranks' kernels, run
--peer --once with OCC_PEER_TIMEOUT_MS=200: each arrival wait then gives up
after 0.2 s (the forward's values are garbage, the kernels' traffic is real)."""
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")  # peer mode between threads (tests/conftest.py)
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13345_b200 as occ  # noqa: E402


def main():
    peer = "--peer" in sys.argv
    iters = 1 if "--once" in sys.argv else 10
    nd, ne, k, dm, dh, n = 2, 8, 2, 4096, 1024, 16384
    torch.manual_seed(0)
    plist = np.arange(ne).reshape(nd, ne // nd)
    w1 = (torch.rand(ne, dm, dh, device="cuda") * 2 - 1).mul_(dm ** -0.5).bfloat16()
    w2 = (torch.rand(ne, dh, dm, device="cuda") * 2 - 1).mul_(dh ** -0.5).bfloat16()
    X = [(torch.rand(n, dm, device="cuda") * 2 - 1).bfloat16() for _ in range(nd)]
    G = (torch.rand(ne, dm, device="cuda") * 2 - 1).mul_(3 / dm ** 0.5).bfloat16()
    OUT = [torch.empty_like(x) for x in X]
    key = int(np.random.default_rng().integers(1 << 30))
    times = [None] * nd
    bar = threading.Barrier(nd)

    def rank(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation="silu"),
                                            occ.Placement([list(map(int, p)) for p in plist]), world_size=nd, rank=r)
            loc = plist[r]
            layer.load_experts(w1[loc].contiguous(), w2[loc].contiguous())
            layer.comm_init_loopback(key)
            if peer:
                layer.comm_enable_peer(n)
            layer.set_validate(False)
            for _ in range(1 if iters == 1 else 3):
                layer.forward_expert_parallel(X[r], G, out=OUT[r])
            st.synchronize()
            bar.wait()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(iters):
                layer.forward_expert_parallel(X[r], G, out=OUT[r])
            e1.record(st)
            st.synchronize()
            times[r] = e0.elapsed_time(e1) / iters
            bar.wait()

    ths = [threading.Thread(target=rank, args=(r,)) for r in range(nd)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    print(f"world={nd} peer={peer} n_per_rank={n} D={dm}: forward ms per rank {times}")


if __name__ == "__main__":
    main()
