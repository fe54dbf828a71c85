#!/bin/bash
# A/B of GEMM environment switches: DRAM bytes per launch under ncu (Mixtral
# and DeepSeek layers) and CUDA-event TFLOP/s (gemm_micro, variants
# interleaved so clock drift hits all alike).
# usage: gemm_env_ab.sh OUTDIR "VAR=a VAR=b ..." [cases]
cd "$(dirname "$0")/../.."
OUT=$1; VARIANTS=$2; CASES=${3:-mixtral,deepseek}; mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct"
for v in $VARIANTS; do
  env $v ncu --metrics $M --clock-control none -k regex:gemm_kernel -c 2 --csv --log-file $OUT/mix_$v.csv \
    python profiles/small_batch_probe.py 8 2 1 4096 14336 swiglu 16384 > /dev/null 2>&1
  env $v ncu --metrics $M --clock-control none -k regex:gemm_kernel -c 2 --csv --log-file $OUT/ds_$v.csv \
    python profiles/small_batch_probe.py 64 6 1 2048 1408 swiglu 16384 > /dev/null 2>&1
  echo "== $v"; python profiles/ncu_brief.py $OUT/mix_$v.csv; python profiles/ncu_brief.py $OUT/ds_$v.csv
done
for rep in 1 2 3; do
  for v in $VARIANTS; do
    echo "== time $v rep $rep"
    env $v OCC_MICRO_CUBLAS=0 python profiles/gemm_micro.py $CASES random 2>&1 | grep '^{' | \
      python -c "import json,sys; [print(d['case'], round(d['gemm1_tflops']), round(d['gemm2_tflops'])) for d in map(json.loads, sys.stdin)]"
  done
done
