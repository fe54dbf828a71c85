"""Forward + backward of one MoE layer (training mode), stage by stage, for
profiling the backward kernels: python profiles/bwd_micro.py [E k D F n]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13345_b200 as occ  # noqa: E402


def main(E=64, k=8, D=2048, F=1024, n=65536, iters=4):
    dev = torch.device("cuda", 0)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(E, k, 1, D, F, activation="swiglu"))
    layer.set_training(True)
    w1 = torch.empty((E, D, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5)
    w3 = torch.empty_like(w1).uniform_(-1, 1).mul_(D ** -0.5)
    w2 = torch.empty((E, F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(F ** -0.5)
    layer.load_experts(w1, w2, w3)
    x = torch.empty((n, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    up = torch.empty_like(x).uniform_(-1, 1)
    ids = torch.argsort(torch.rand(n, E, device=dev), dim=1)[:, :k].to(torch.int32)
    w = torch.full((n, k), 1.0 / k, device=dev)
    layer.set_validate(False)
    for _ in range(iters):
        layer.forward_given_routing(x, ids, w)
        layer.backward(up)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    layer.backward(up)
    e1.record()
    torch.cuda.synchronize()
    print(f"backward {e0.elapsed_time(e1):.3f} ms")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
