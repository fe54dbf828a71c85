#!/bin/bash
# One-box perf snapshot used between changes: small-batch graph steps, the
# short-K grouped GEMMs against same-box cuBLAS, GEMM timeline of the C1
# layer, and the default bench line.
cd "$(dirname "$0")/../.."
python profiles/small_batch_probe.py
python profiles/small_batch_probe.py 64 6 8 2048 1408 swiglu 128
python profiles/small_batch_probe.py 8 2 1 4096 14336 swiglu 512
python profiles/small_batch_probe.py 64 8 8 2048 1024 swiglu 2048
OCC_GEMM_TIMELINE=1 python profiles/small_batch_probe.py 2>&1 | grep "gemm tl" | tail -2
python profiles/gemm_micro.py deepseek,olmoe,mixtral random 2>&1 | grep '^{'
python bench.py --steps 10 --warmup 3 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', round(d['value']), d['ms_per_step'], d['roofline']['frac'], d['roofline']['gemm2']['frac'], d['clocks'], d['stages_ms'])"
