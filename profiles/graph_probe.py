"""CUDA-graph capture of the whole layer step (route + plan + dispatch +
grouped FFN + combine [+ backward]): checks the replay is bit-identical to
eager calls and times both (CUDA events, median of 50)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13345_b200 as occ  # noqa: E402

CASES = {"c1": (8, 2, 512, 1024, 2048, "silu", 2, False), "mixtral": (8, 2, 4096, 14336, 16384, "swiglu", 1, False),
         "deepseek": (64, 6, 2048, 1408, 16384, "swiglu", 1, False), "small": (64, 8, 2048, 1024, 256, "swiglu", 1, False),
         "olmoe_train_small": (64, 8, 2048, 1024, 4096, "swiglu", 1, True)}


def run(name):
    E, k, D, F, n, act, nd, train = CASES[name]
    dev = torch.device("cuda", 0)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(E, k, nd, D, F, activation=act))
    if train:
        layer.set_training(True)
    w1 = torch.empty((E, D, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5)
    w3 = torch.empty_like(w1).uniform_(-1, 1).mul_(D ** -0.5) if act == "swiglu" else None
    w2 = torch.empty((E, F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(F ** -0.5)
    layer.load_experts(w1, w2, w3)
    gate = torch.empty((E, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(3.0 / D ** 0.5)
    x = torch.empty((n, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    up = torch.empty_like(x).uniform_(-1, 1)
    out = torch.empty_like(x)
    layer.set_validate(False)
    res = {}

    def step():
        layer.forward_expert_parallel(x, gate, out=out)
        if train:
            res["g"] = layer.backward(up)["x"]

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    eager = out.clone()
    g = torch.cuda.CUDAGraph()
    l0 = occ.launch_count()
    with torch.cuda.graph(g):
        step()
    per_step = occ.launch_count() - l0
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    same = bool(torch.equal(out, eager))

    def timeit(fn, reps=50):
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return sorted(ts)[len(ts) // 2]
    print(json.dumps({"case": name, "kernels_per_step": per_step, "replay_bit_identical": same,
                      "eager_ms": timeit(step), "graph_ms": timeit(g.replay)}), flush=True)


if __name__ == "__main__":
    for nm in (sys.argv[1].split(",") if len(sys.argv) > 1 else CASES):
        run(nm)
