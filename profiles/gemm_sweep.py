"""Mixtral-layer forward timed per stage (CUDA events), for raster/band
experiments: OCC_GEMM_BAND=<m-tiles per band> python profiles/gemm_sweep.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13345_b200 as occ  # noqa: E402


def main(steps=10, E=8, k=2, D=4096, F=14336, n=16384):
    dev = torch.device("cuda", 0)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(E, k, 1, D, F, activation="swiglu"))
    w1 = torch.empty((E, D, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5)
    w3 = torch.empty_like(w1).uniform_(-1, 1).mul_(D ** -0.5)
    w2 = torch.empty((E, F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(F ** -0.5)
    layer.load_experts(w1, w2, w3)
    del w1, w2, w3
    gate = torch.empty((E, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(3.0 / D ** 0.5)
    x = torch.empty((n, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    out = torch.empty_like(x)
    layer.set_validate(False)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        layer.forward_expert_parallel(x, gate, out=out)
    layer.set_profiling(True)
    acc = {}
    for _ in range(steps):
        flush.zero_()
        layer.forward_expert_parallel(x, gate, out=out)
        for kk, v in layer.stage_ms().items():
            acc.setdefault(kk, []).append(v)
    print(json.dumps({"band": os.environ.get("OCC_GEMM_BAND"),
                      **{kk: sorted(v)[len(v) // 2] for kk, v in acc.items() if kk.startswith("gemm")}}))


if __name__ == "__main__":
    main()
