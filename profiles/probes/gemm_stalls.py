"""Stall-cycle breakdown of the grouped GEMMs (OCC_GEMM_DEBUG=1 makes the
library print producer / MMA / epilogue wait cycles per launch to stderr).
Usage: OCC_GEMM_DEBUG=1 python profiles/probes/gemm_stalls.py deepseek"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2505_13345_b200 as occ  # noqa: E402

CASES = {"deepseek": (64, 6, 2048, 1408, 16384), "olmoe": (64, 8, 2048, 1024, 65536),
         "mixtral": (8, 2, 4096, 14336, 16384)}


def main(name):
    E, k, D, F, n = CASES[name]
    dev = torch.device("cuda", 0)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(E, k, 1, D, F, activation="swiglu"))
    w1 = torch.empty((E, D, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5)
    layer.load_experts(w1, torch.empty((E, F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(F ** -0.5),
                       torch.empty_like(w1).uniform_(-1, 1).mul_(D ** -0.5))
    x = torch.empty((n, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    ids = torch.argsort(torch.rand(n, E, device=dev), dim=1)[:, :k].to(torch.int32)
    w = torch.full((n, k), 1.0 / k, device=dev)
    layer.set_validate(False)
    for _ in range(4):
        layer.forward_given_routing(x, ids, w)
    torch.cuda.synchronize()
    print("---", name, "WIDE", os.environ.get("OCC_GEMM_WIDE", "1"), file=sys.stderr, flush=True)
    layer.forward_given_routing(x, ids, w)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1])
