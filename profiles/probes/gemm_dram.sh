#!/bin/bash
# DRAM traffic of the grouped GEMMs (Mixtral layer, 16,384 tokens) under TMA
# L2-promotion variants, and the L2 capacity / cross-die sharing probe.
# usage: gemm_dram.sh OUTDIR
cd "$(dirname "$0")/../.."
OUT=$1; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o $OUT/l2_capacity_probe profiles/probes/l2_capacity_probe.cu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct"
for mb in 32 48 64 80 96 112 128; do
  for sh in 0 74; do
    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k two_pass -c 1 --csv $OUT/l2_capacity_probe $mb $sh 2>/dev/null \
      | grep -E "dram__bytes_read|gpu__time" | awk -F'","' -v mb=$mb -v sh=$sh '{print "probe", mb, "MB shift", sh, $(NF-2), $(NF-1), $NF}'
  done
done
for pr in 3 2 0; do
  OCC_TMAP_PROMO=$pr ncu --metrics $M --clock-control none -k regex:wide_gemm -c 2 --csv --log-file $OUT/gemm_promo$pr.csv \
    python profiles/small_batch_probe.py 8 2 1 4096 14336 swiglu 16384 > /dev/null 2>&1
  echo "== promo $pr"; python profiles/ncu_brief.py $OUT/gemm_promo$pr.csv | tail -4
done
