#!/bin/bash
# C1 latency sweep: plan-kernel grid sizes (OCC_PLAN_BLOCKS, phase timeline via
# OCC_PLAN_DEBUG) and epilogue-staging variants (OCC_LIB_EXPERIMENT).
cd "$(dirname "$0")/../.."
for b in 0 16 37 74 148 296; do
  echo "== plan blocks $b"
  OCC_PLAN_BLOCKS=$b OCC_PLAN_DEBUG=1 python profiles/small_batch_probe.py 2>&1 | grep "plan dbg" | tail -1
  OCC_PLAN_BLOCKS=$b python profiles/small_batch_probe.py
done
for v in "$@"; do
  echo "== variant $v"
  OCC_LIB_EXPERIMENT=profiles/variants/libocc_$v.so python profiles/small_batch_probe.py
  OCC_LIB_EXPERIMENT=profiles/variants/libocc_$v.so OCC_GEMM_TIMELINE=1 python profiles/small_batch_probe.py 2>&1 | grep "gemm tl" | tail -2
  OCC_LIB_EXPERIMENT=profiles/variants/libocc_$v.so python profiles/gemm_micro.py deepseek,olmoe random 2>&1 | tail -2
done
echo "== base gemm_micro"
python profiles/gemm_micro.py deepseek,olmoe random 2>&1 | tail -2
