# runtime split policy vs the compile-time no-split build (gemm_micro random routing)
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in nosplit auto ws0 ws2; do
  L=""; E=""
  case $v in nosplit) L=profiles/variants/libocc_nosplit.so;; ws0) E=0;; ws2) E=2;; esac
  echo "== $v round $r"
  OCC_GEMM_WSPLIT=$E OCC_LIB_EXPERIMENT=$L OCC_MICRO_CUBLAS=0 timeout 200 python profiles/gemm_micro.py deepseek,olmoe,mixtral random 2>&1 | grep case | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['case'], round(d['gemm1_tflops']), round(d['gemm2_tflops']))"
done; done
