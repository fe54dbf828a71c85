"""Profiling -> placement loop on the GPU (paper Table 1):
planted-block routing traces (trace_gen.cpp:69-101 semantics, p_in = 0.9,
hidden blocks unaligned with the trivial layout) at the OLMoE shape (64
experts top-8, 65,536 tokens, EP=8); device co-activation histogram ->
reschedule_placement -> the device dispatch plan's E(C_T) and all-to-all
bytes/token, trivial vs rescheduled placement (and vs naive top-k).
Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13345_b200 as occ  # noqa: E402


def planted_block_ids(n, ne, k, blocks, p_in, rng):
    """Vectorised planted-block routing: each token has a home block; each of
    its k distinct experts is drawn from the home block with prob. p_in."""
    perm = rng.permutation(ne)
    block_of = np.empty(ne, np.int64)
    block_of[perm] = np.arange(ne) // (ne // blocks)
    members = [np.nonzero(block_of == b)[0] for b in range(blocks)]
    others = [np.nonzero(block_of != b)[0] for b in range(blocks)]
    home = rng.integers(0, blocks, n)
    n_home = rng.binomial(k, p_in, n)
    ids = np.empty((n, k), np.int32)
    for b in range(blocks):
        sel = np.nonzero(home == b)[0]
        ih = np.argsort(rng.random((len(sel), len(members[b]))), axis=1)
        io = np.argsort(rng.random((len(sel), len(others[b]))), axis=1)
        hm, ot = members[b][ih], others[b][io]
        for j in range(k):
            use_home = j < n_home[sel]
            ids[sel, j] = np.where(use_home, hm[:, min(j, hm.shape[1] - 1)], ot[:, j])
    return ids, block_of


def main(ne=64, k=8, nd=8, n=65536, blocks=8, p_in=0.9, batches=4, seed=2505):
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", 0)
    profile = [torch.from_numpy(planted_block_ids(n, ne, k, blocks, p_in, np.random.default_rng(seed))[0]).to(dev)]
    for b in range(1, batches):
        profile.append(torch.from_numpy(planted_block_ids(n, ne, k, blocks, p_in, np.random.default_rng(seed))[0]
                                        [rng.permutation(n)]).to(dev))
    t0 = time.perf_counter()
    placement = occ.collaboration_aware_placement(profile, ne, nd)
    torch.cuda.synchronize()
    t_place = time.perf_counter() - t0
    # evaluate on a held-out batch from the same distribution
    ids = torch.from_numpy(planted_block_ids(n, ne, k, blocks, p_in, np.random.default_rng(seed))[0][::-1].copy()).to(dev)
    src = torch.from_numpy(rng.integers(0, nd, n).astype(np.int32)).to(dev)
    out = {}
    for name, pl in (("trivial", occ.trivial_placement(ne, nd)), ("rescheduled", placement)):
        layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, 2048, 1024), pl)
        layer.build_dispatch_index(ids, src)
        r = layer.comm_report(bytes_per_scalar=2)
        out[name] = {"mean_replicas": r.mean_replicas, "crossing_rows_per_token": r.crossing_rows / n,
                     "dedup_bytes_per_token": r.crossing_rows * 2048 * 2 / n,
                     "naive_bytes_per_token": r.naive_crossing_rows * 2048 * 2 / n,
                     "intra_share": r.intra_share}
    line = {"experiment": "collaboration-aware placement on GPU (planted-block traces)",
            "config": {"experts": ne, "top_k": k, "ep": nd, "tokens": n, "d_model": 2048, "blocks": blocks,
                       "p_in": p_in, "profile_batches": batches},
            "placement_s": t_place, **out,
            "ct_reduction": 1 - out["rescheduled"]["mean_replicas"] / out["trivial"]["mean_replicas"],
            "bytes_vs_naive_rescheduled": out["rescheduled"]["dedup_bytes_per_token"]
            / out["rescheduled"]["naive_bytes_per_token"]}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
