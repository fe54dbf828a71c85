#!/bin/bash
# Round-2 evidence pass on one B200: GPU suite, smoke, bench lines for every
# BASELINE workload, the bench's launch list, one --set full capture of
# GEMM-1, and the C1 launch list + GEMM timeline.   usage: r02_final.sh OUTDIR
cd "$(dirname "$0")/../.."
OUT=$1; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/gputests.log 2>&1; echo rc=$? >> $OUT/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench_mixtral.log 2>&1
for w in c1 deepseek olmoe qwen; do timeout 600 python bench.py --workload $w > $OUT/bench_$w.log 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 > $OUT/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wide_gemm_kernel -c 1 -o $OUT/gemm1_full \
  python profiles/probes/gemm_stalls.py mixtral > /dev/null 2>&1
python profiles/summarize_ncu.py $OUT/gemm1_full.ncu-rep > $OUT/gemm1_full_summary.md 2>&1
ncu -i $OUT/gemm1_full.ncu-rep --page raw --csv > $OUT/gemm1_full_raw.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file $OUT/c1_launches.csv \
  python profiles/small_batch_probe.py > /dev/null 2>&1
OCC_GEMM_TIMELINE=1 python profiles/small_batch_probe.py 2>&1 | grep "gemm tl" | tail -2 > $OUT/c1_gemm_timeline.txt
python profiles/small_batch_probe.py > $OUT/c1_probe.txt 2>&1
