"""Sustained (power-capped) comparison on one box: our Mixtral-layer GEMM-1 /
GEMM-2 (grouped, routed rows) vs cuBLAS on a dense GEMM of the same shape and
FLOPs, each run back to back for ~4 s (the regime MEASURED_PEAKS calls
`bf16_tflops_sustained`), CUDA events over the whole loop, SM clock sampled."""
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13345_b200 as occ  # noqa: E402


def clocked(fn, seconds=4.0):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < 0.3:
        fn()
        n += 1
    torch.cuda.synchronize()
    per = (time.perf_counter() - t0) / n
    reps = max(3, int(seconds / per))
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "100"],
                           stdout=subprocess.PIPE, text=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    smi.terminate()
    clk = sorted(float(l) for l in smi.communicate()[0].split() if l.strip())
    return e0.elapsed_time(e1) / reps, (clk[len(clk) // 2] if clk else None)


def main(E=8, k=2, D=4096, F=14336, n=16384):
    dev = torch.device("cuda", 0)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(E, k, 1, D, F, activation="swiglu"))
    w1 = torch.empty((E, D, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(D ** -0.5)
    w3 = torch.empty_like(w1).uniform_(-1, 1).mul_(D ** -0.5)
    w2 = torch.empty((E, F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(F ** -0.5)
    layer.load_experts(w1, w2, w3)
    del w1, w2, w3
    x = torch.empty((n, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    ids = torch.argsort(torch.rand(n, E, device=dev), dim=1)[:, :k].to(torch.int32)
    w = torch.full((n, k), 0.5, device=dev)
    layer.set_validate(False)
    f_layer = 2.0 * n * k * D * 3 * F  # GEMM-1 + GEMM-2 FLOPs of the layer
    t_layer, clk_l = clocked(lambda: layer.forward_given_routing(x, ids, w))
    a = torch.empty((n * k, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    b = torch.empty((D, 2 * F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    a2 = torch.empty((n * k, F), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    b2 = torch.empty((F, D), dtype=torch.bfloat16, device=dev).uniform_(-1, 1)

    def cublas_pair():
        torch.matmul(a, b)
        torch.matmul(a2, b2)
    t_cub, clk_c = clocked(cublas_pair)
    print(json.dumps({"what": "4 s back-to-back loops, power-capped",
                      "ours_layer_ms": t_layer, "ours_layer_tflops_incl_non_gemm": f_layer / t_layer / 1e9,
                      "ours_sm_mhz": clk_l, "cublas_two_dense_gemms_ms": t_cub,
                      "cublas_tflops": f_layer / t_cub / 1e9, "cublas_sm_mhz": clk_c}))


if __name__ == "__main__":
    main()
