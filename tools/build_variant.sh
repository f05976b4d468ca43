#!/bin/bash
# Build an alternative libcoopbatch_b200.so with extra -D flags for sample.cu
# (the other objects come from the in-tree build): for tools/ab.sh.
#   bash tools/build_variant.sh NAME "-DCB_PURE_STAGES=2 -DCB_MARK_CTAS=6"
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2310_12403_b200/csrc
OUT=$ROOT/build_variants/$NAME
mkdir -p $OUT
make -s -C $SRC >/dev/null
NV="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-ffp-contract=off -Xptxas -O3 --expt-relaxed-constexpr -I$ROOT/include"
nvcc $NV $FLAGS -I$SRC -c ${SAMPLE_SRC:-$SRC/sample.cu} -o $OUT/sample.o
OBJS=$(ls $SRC/build/*.o | grep -v '/sample.o')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libcoopbatch_b200.so $OUT/sample.o $OBJS -cudart static -Xlinker -z,defs -lpthread -ldl -lrt
echo "$FLAGS" > $OUT/FLAGS
