# A/B of wide-kernel epilogue variants (profiles/build_variant.sh), gemm_micro random routing
cd $GRAFT_REPO_ROOT
VARS=${VARS:-"nosplit default split_ldc2 split_ldc1"}
for r in 1 2; do
for v in $VARS; do
  if [ $v = default ]; then L=""; else L=profiles/variants/libocc_$v.so; fi
  echo "== $v round $r"
  OCC_LIB_EXPERIMENT=$L OCC_MICRO_CUBLAS=0 timeout 200 python profiles/gemm_micro.py deepseek,olmoe,mixtral random 2>&1 | grep case | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['case'], round(d['gemm1_tflops']), round(d['gemm2_tflops']))"
done; done
