#!/bin/bash
# C1 / small-batch latency: graph step + per-stage times, plan phase timeline,
# GEMM per-chunk epilogue timeline.
cd "$(dirname "$0")/../.."
python profiles/small_batch_probe.py
python profiles/small_batch_probe.py 64 6 8 2048 1408 swiglu 128
python profiles/small_batch_probe.py 8 2 1 4096 14336 swiglu 512
python profiles/small_batch_probe.py 64 8 8 2048 1024 swiglu 2048
OCC_PLAN_DEBUG=1 python profiles/small_batch_probe.py 2>&1 | grep "plan dbg" | tail -1
OCC_GEMM_TIMELINE=1 python profiles/small_batch_probe.py 2>&1 | grep "gemm tl" | tail -2
