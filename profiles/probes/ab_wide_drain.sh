cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in old default ldc2 ldc4 sw_only; do
  if [ $v = default ]; then L=""; else L=profiles/variants/libocc_$v.so; fi
  echo "== $v round $r"
  OCC_LIB_EXPERIMENT=$L OCC_MICRO_CUBLAS=0 timeout 200 python profiles/gemm_micro.py deepseek,olmoe,mixtral random 2>&1 | grep case | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['case'], round(d['gemm1_tflops']), round(d['gemm2_tflops']))"
done; done
