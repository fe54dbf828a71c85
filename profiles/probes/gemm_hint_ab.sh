#!/bin/bash
# L2 eviction-policy A/B for the grouped GEMMs (OCC_GEMM_HINT bits: 1 B loads
# evict_first, 2 C stores evict_first, 4 A loads evict_last): DRAM bytes per
# launch under ncu (Mixtral layer) and CUDA-event TFLOP/s (gemm_micro, hints
# interleaved so clock drift hits all alike).   usage: gemm_hint_ab.sh OUTDIR "hints"
cd "$(dirname "$0")/../.."
OUT=$1; HINTS=${2:-"0 1 2 3 7"}; mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct"
for h in $HINTS; do
  OCC_GEMM_HINT=$h ncu --metrics $M --clock-control none -k regex:gemm_kernel -c 2 --csv --log-file $OUT/mix_h$h.csv \
    python profiles/small_batch_probe.py 8 2 1 4096 14336 swiglu 16384 > /dev/null 2>&1
  OCC_GEMM_HINT=$h ncu --metrics $M --clock-control none -k regex:gemm_kernel -c 2 --csv --log-file $OUT/ds_h$h.csv \
    python profiles/small_batch_probe.py 64 6 1 2048 1408 swiglu 16384 > /dev/null 2>&1
  echo "== hint $h"; python profiles/ncu_brief.py $OUT/mix_h$h.csv; python profiles/ncu_brief.py $OUT/ds_h$h.csv
done
for rep in 1 2; do
  for h in $HINTS; do
    echo "== time hint $h rep $rep"
    OCC_MICRO_CUBLAS=0 OCC_GEMM_HINT=$h python profiles/gemm_micro.py mixtral,deepseek random 2>&1 | grep '^{' | \
      python -c "import json,sys; [print(d['case'], round(d['gemm1_tflops']), round(d['gemm2_tflops'])) for d in map(json.loads, sys.stdin)]"
  done
done
