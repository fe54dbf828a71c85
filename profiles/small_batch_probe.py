"""Small-batch (C1 / decode-like) probe: per-stage CUDA-event times of the
one-GPU forward at a given shape, and the GEMM role-stall counters
(OCC_GEMM_DEBUG).  Run one configuration per process (env switches are read
once):  python profiles/small_batch_probe.py [ne k nd dm dh act n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13345_b200 as occ  # noqa: E402


def main():
    a = sys.argv[1:] or ["8", "2", "2", "512", "1024", "silu", "2048"]
    ne, k, nd, dm, dh = map(int, a[:5])
    act, n = a[5], int(a[6])
    torch.manual_seed(0)
    dev = torch.device("cuda")
    layer = occ.ExpertParallelLayer(occ.MoEConfig(ne, k, nd, dm, dh, activation=act))
    g = act == "swiglu"
    w1 = (torch.rand(ne, dm, dh, device=dev) * 2 - 1).mul_(dm ** -0.5).bfloat16()
    w3 = (torch.rand(ne, dm, dh, device=dev) * 2 - 1).mul_(dm ** -0.5).bfloat16() if g else None
    w2 = (torch.rand(ne, dh, dm, device=dev) * 2 - 1).mul_(dh ** -0.5).bfloat16()
    layer.load_experts(w1, w2, w3)
    x = (torch.rand(n, dm, device=dev) * 2 - 1).bfloat16()
    gate = (torch.rand(ne, dm, device=dev) * 2 - 1).mul_(3 / dm ** 0.5).bfloat16()
    layer.set_validate(False)
    out = torch.empty_like(x)
    if os.environ.get("OCC_GEMM_DEBUG") or os.environ.get("OCC_GEMM_TIMELINE"):  # synchronising: eager only
        for _ in range(3):
            layer.forward_expert_parallel(x, gate, out=out)
        torch.cuda.synchronize()
        return
    for _ in range(5):
        layer.forward_expert_parallel(x, gate, out=out)
    torch.cuda.synchronize()
    layer.set_profiling(True)
    acc = {}
    for _ in range(20):
        layer.forward_expert_parallel(x, gate, out=out)
        for kk, v in layer.stage_ms().items():
            acc.setdefault(kk, []).append(v)
    layer.set_profiling(False)
    st = {kk: sorted(v)[len(v) // 2] * 1e3 for kk, v in acc.items()}
    # whole step as a CUDA graph
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        layer.forward_expert_parallel(x, gate, out=out)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        layer.forward_expert_parallel(x, gate, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        gr.replay()
    e0.record()
    for _ in range(50):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    env = {kk: v for kk, v in os.environ.items() if kk.startswith("OCC_")}
    print(f"shape={a} env={env} graph_us={e0.elapsed_time(e1) / 50 * 1e3:.1f} stages_us=" +
          " ".join(f"{kk}:{v:.1f}" for kk, v in st.items()))


if __name__ == "__main__":
    main()
