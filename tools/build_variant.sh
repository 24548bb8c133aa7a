#!/bin/bash
# build_variant.sh NAME SRC.cu [ORIG.cu]: link a variant library whose ORIG
# object (default ctransform.cu) is replaced by SRC compiled with the
# Makefile's flags -> paper_1905_12154_b200/variants/libbfm_NAME.so (select
# it at run time with BFM_LIB_OVERRIDE)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_1905_12154_b200/csrc
NAME=$1; SRC=$2; ORIG=${3:-ctransform.cu}
mkdir -p $ROOT/paper_1905_12154_b200/variants /tmp/variants
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v ${VINC:+-I$VINC} -I$CS -I$ROOT/include -c $SRC -o /tmp/variants/$NAME.o 2> /tmp/variants/$NAME.log
OBJS=$(ls $CS/*.o | grep -v "/${ORIG%.cu}.o")
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $ROOT/paper_1905_12154_b200/variants/libbfm_$NAME.so $OBJS /tmp/variants/$NAME.o -lpthread -ldl
grep -E "registers|spill" /tmp/variants/$NAME.log | tail -4
