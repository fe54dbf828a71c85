#!/bin/bash
# A/B builds for profiling: libocc with extra -D flags on one source file
# (default occ_gemm.cu; VARIANT_SRC=occ_kernels.cu ... to pick another), written
# to profiles/variants/libocc_<name>.so (git-ignored, travels with gpurun);
# select with OCC_LIB_EXPERIMENT=profiles/variants/libocc_<name>.so.
# usage: [VARIANT_SRC=file.cu] profiles/build_variant.sh <name> -DFOO=1 ...
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
CSRC=$HERE/../paper_2505_13345_b200/csrc
SRC=${VARIANT_SRC:-occ_gemm.cu}
OBJ=${SRC%.cu}.o
NAME=$1; shift
OUT=$HERE/variants; mkdir -p $OUT/$NAME
NCCL=$(python3 -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -I$NCCL/include"
nvcc $FL "$@" -c $CSRC/$SRC -o $OUT/$NAME/$OBJ
OBJS=$(ls $CSRC/build/*.o | grep -v "/$OBJ\$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libocc_$NAME.so $OUT/$NAME/$OBJ $OBJS -lcudart \
    -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib
echo $OUT/libocc_$NAME.so
