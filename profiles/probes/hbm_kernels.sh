#!/bin/bash
# HBM-bound layer kernels, cold-cache ncu per launch (time + DRAM bytes) and
# in-step stage times: the one-GPU Mixtral layer (combine_fused, scatter,
# router) and the two-rank loopback exchange (pack, partial combine, combine).
# usage: hbm_kernels.sh OUTDIR [variant ...]   (variant: profiles/variants/libocc_<v>.so)
cd "$(dirname "$0")/../.."
OUT=$1; shift; mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for v in base "$@"; do
  if [ "$v" = base ]; then unset OCC_LIB_EXPERIMENT; else export OCC_LIB_EXPERIMENT=profiles/variants/libocc_$v.so; fi
  ncu --metrics $M --clock-control none -k regex:"combine_fused|scatter_rows|router_tc" -c 6 --csv \
      --log-file $OUT/hbm_$v.csv python bench.py --steps 1 --warmup 1 > /dev/null 2>&1
  ncu --metrics $M --clock-control none -k regex:"pack_kernel|partial_combine|combine_kernel" -c 12 --csv \
      --log-file $OUT/xch_$v.csv python profiles/exchange_kernels_probe.py --once > /dev/null 2>&1
  OCC_PEER_TIMEOUT_MS=300 ncu --metrics $M --clock-control none -k regex:"peer_pack|peer_return|combine_kernel" -c 12 --csv \
      --log-file $OUT/peer_$v.csv python profiles/exchange_kernels_probe.py --peer --once > /dev/null 2>&1
  echo "== $v"
  python profiles/ncu_brief.py $OUT/hbm_$v.csv | awk '{print $0}' | tail -3
  python profiles/ncu_brief.py $OUT/xch_$v.csv | tail -6
  python profiles/ncu_brief.py $OUT/peer_$v.csv | tail -6
  python bench.py --steps 10 --warmup 3 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stages', {k: round(v*1e3,1) for k,v in d['stages_ms'].items()}, 'ms', d['ms_per_step'])"
done
unset OCC_LIB_EXPERIMENT
