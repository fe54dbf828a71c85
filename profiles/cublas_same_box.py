"""Same-box tensor-core reference for the grouped GEMMs: cuBLAS (torch.matmul)
on dense GEMMs with the FLOPs and operand shapes of the Mixtral-layer GEMM-1
(x @ [w1|w3]: M=32768 routed rows, N=2F=28672, K=4096) and GEMM-2
(h @ w2: M=32768, N=4096, K=14336), timed with CUDA events, burst (best of 10)
and back to back for ~3 s (sustained), with the SM clock sampled. Used to
separate box-to-box power/clock variance from kernel quality (profiles/)."""
import json
import subprocess
import time

import torch


def timed(fn, iters):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    dev = torch.device("cuda", 0)
    out = {}
    for name, (m, n, k) in {"gemm1_shape": (32768, 28672, 4096), "gemm2_shape": (32768, 4096, 14336),
                            "square8192": (8192, 8192, 8192)}.items():
        a = torch.randn(m, k, device=dev, dtype=torch.bfloat16)
        b = torch.randn(k, n, device=dev, dtype=torch.bfloat16)
        f = lambda: torch.matmul(a, b)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        best = min(timed(f, 1) for _ in range(10))
        n_sus = max(3, int(3000 / best))
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                "-lms", "100"], stdout=subprocess.PIPE, text=True)
        time.sleep(0.05)
        sus = timed(f, n_sus)
        smi.terminate()
        clk = [float(l.split(",")[0]) for l in smi.communicate()[0].splitlines() if l.strip()]
        fl = 2.0 * m * n * k
        out[name] = {"mnk": [m, n, k], "burst_ms": best, "burst_tflops": fl / best / 1e9,
                     "sustained_ms": sus, "sustained_tflops": fl / sus / 1e9,
                     "sm_mhz_median": sorted(clk)[len(clk) // 2] if clk else None}
        del a, b
    print(json.dumps(out))


if __name__ == "__main__":
    main()
