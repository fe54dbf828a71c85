"""LRU model of the grouped GEMMs' L2 reuse under a tile schedule (offline;
no GPU).  Tiles of the wide kernel (256 x 512 super-tiles; A m-tile 256 rows,
B super-block 512 rows, one 64-deep K block per step) are walked in the
kernel's raster order (tile_coords: per expert, bands of `band` m-tiles,
n-block-major inside a band); tile t starts at (t // pairs) * KB K-steps
(waves in phase: what the dynamic scheduler keeps, and the best case of the
static walk before the pairs drift) or at t * KB / pairs (uniformly
staggered pairs).  Measured against ncu: Mixtral GEMM-1 in phase 2.51 GB vs
2.67 GB with the dynamic scheduler (6.07 GB static, drifted).  Every K step
a tile reads its A and B K-slices; the C tile is written when it ends.  A byte-capacity LRU (default 80 MB, measured
by profiles/probes/l2_capacity_probe.cu) counts the bytes that miss.

python profiles/l2_schedule_sim.py [mixtral1|mixtral2|deepseek2|olmoe1|olmoe2] [band] [cap_MB]"""
import sys
from collections import OrderedDict

SHAPES = {  # experts, rows/expert, K, N (output cols), pairs
    "mixtral1": (8, 4096, 4096, 28672),
    "mixtral2": (8, 4096, 14336, 4096),
    "deepseek2": (64, 1536, 1408, 2048),
    "olmoe1": (64, 8192, 2048, 2048),
    "olmoe2": (64, 8192, 1024, 2048),
}


def simulate(shape, band, cap_mb, staggered=False, pairs=74):
    E, rows, K, N = SHAPES[shape]
    mt, nbw, KB = rows // 256, N // 512, K // 64
    tiles = []
    for e in range(E):
        for b0 in range(0, mt, band):
            bm = min(band, mt - b0)
            for nb in range(nbw):
                for m in range(bm):
                    tiles.append((e, b0 + m, nb))
    events = []
    for t, (e, m, nb) in enumerate(tiles):
        s = t * KB / pairs if staggered else (t // pairs) * KB
        for kb in range(KB):
            events.append((s + kb, t, kb))
    events.sort()
    a_bytes, b_bytes, c_bytes = 256 * 128, 512 * 128, 256 * 512 * 2
    cap = cap_mb * (1 << 20)
    lru, used, miss = OrderedDict(), 0, 0

    def touch(key, nbytes, count=True):
        nonlocal used, miss
        if key in lru:
            lru.move_to_end(key)
            return
        if count:
            miss += nbytes
        lru[key] = nbytes
        used += nbytes
        while used > cap:
            _, nb_ = lru.popitem(last=False)
            used -= nb_

    for _, t, kb in events:
        e, m, nb = tiles[t]
        touch(("A", e, m, kb), a_bytes)
        touch(("B", e, nb, kb), b_bytes)
        if kb == KB - 1:
            touch(("C", t), c_bytes, count=False)
    algo = E * (rows * K * 2 + N * K * 2)
    return miss / 1e9, algo / 1e9


if __name__ == "__main__":
    shape = sys.argv[1] if len(sys.argv) > 1 else "mixtral2"
    bands = [int(sys.argv[2])] if len(sys.argv) > 2 else [2, 4, 8, 16]
    cap = float(sys.argv[3]) if len(sys.argv) > 3 else 80
    for band in bands:
        for stg in (False, True):
            got, algo = simulate(shape, band, cap, stg)
            print(f"{shape} band {band:2d} {'staggered' if stg else 'in phase '} cap {cap:.0f} MB: "
                  f"DRAM read {got:.2f} GB (algorithmic {algo:.2f} GB, {got / algo:.2f}x)")
