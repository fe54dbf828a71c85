"""Digest of layer outputs (forward, shared experts, training forward + every
backward gradient) over shapes that take the wide / narrow / weight-gradient
GEMM kernels through several waves.  The tile -> CTA-pair assignment must not
change a single bit (each tile's math is the same whoever runs it), so
OCC_GEMM_DYN=0 (static walk) and =1 (dynamic tile scheduler) print the same
digest (tests/test_gpu_parity.py::test_dynamic_tile_schedule_bit_identical).
python profiles/probes/sched_digest.py"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2505_13345_b200 as occ  # noqa: E402


def layer_io(E, k, D, F, n, act, seed, shared=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda *s, scale=1.0: (torch.rand(*s, device="cuda", generator=g) * 2 - 1).mul_(scale).bfloat16()
    w1, w2 = r(E, D, F, scale=D ** -0.5), r(E, F, D, scale=F ** -0.5)
    w3 = r(E, D, F, scale=D ** -0.5) if act == "swiglu" else None
    x = r(n, D)
    ids = torch.argsort(torch.rand(n, E, device="cuda", generator=g), dim=1)[:, :k].to(torch.int32)
    w = torch.rand(n, k, device="cuda", generator=g) + 0.05
    w = (w / w.sum(1, keepdim=True)).float()
    sh = None
    if shared:  # S shared experts of width 128: w1/w3 [S, D, 128], w2 [S, 128, D]
        sh = (r(shared, D, 128, scale=D ** -0.5), r(shared, 128, D, scale=(128 * shared) ** -0.5),
              r(shared, D, 128, scale=D ** -0.5) if act == "swiglu" else None)
    return w1, w2, w3, x, ids, w, sh


def main():
    h = hashlib.sha256()
    cases = [  # E, k, D, F, n, act, train, shared
        (8, 2, 1024, 2048, 8192, "swiglu", False, 0),   # wide GEMM-1 / GEMM-2, many waves
        (16, 4, 512, 1408, 4096, "swiglu", False, 0),   # odd B-block count: narrow GEMM-1
        (8, 2, 1024, 1024, 4096, "silu", True, 0),      # training forward + backward (wide wgrad)
        (16, 4, 512, 768, 3000, "swiglu", True, 0),     # backward, narrow wgrad (odd 256-col blocks)
        (16, 4, 512, 256, 2048, "swiglu", False, 2),    # shared experts
    ]
    for i, (E, k, D, F, n, act, train, shared) in enumerate(cases):
        w1, w2, w3, x, ids, w, sh = layer_io(E, k, D, F, n, act, seed=i + 1, shared=shared)
        layer = occ.ExpertParallelLayer(occ.MoEConfig(E, k, 1, D, F, activation=act))
        if train:
            layer.set_training(True)
        layer.load_experts(w1, w2, w3)
        if sh:
            layer.load_shared_experts(sh[0], sh[1], sh[2])
        out = layer.forward_given_routing(x, ids, w)
        h.update(out.view(torch.int16).cpu().numpy().tobytes())
        if train:
            up = torch.ones_like(x)
            gr = layer.backward(up)
            for kk in ("x", "w1", "w3", "w2", "routing_weights"):
                if gr.get(kk) is not None:
                    h.update(gr[kk].contiguous().view(torch.int32).cpu().numpy().tobytes())
    torch.cuda.synchronize()
    print("digest", h.hexdigest(), "dyn", os.environ.get("OCC_GEMM_DYN", "1"))


if __name__ == "__main__":
    main()
