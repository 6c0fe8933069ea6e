#!/bin/bash
# Build a variant of the library with extra nvcc defines for A/B timing:
#   tools/variant_build.sh TAG -DFOO=1 ...   -> _variants/libimpact_b200_TAG.so
# (select with IMP_LIB_PATH=...; the JIT construction module is unaffected)
set -e
TAG=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/_variants/obj_$TAG; mkdir -p $OBJ
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
C=$ROOT/paper_2401_03555_b200/csrc
for u in imdp sweep build export; do nvcc $F "$@" -c $C/$u.cu -o $OBJ/$u.o & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/_variants/libimpact_b200_$TAG.so $OBJ/*.o \
  -L/usr/local/cuda/lib64 -lcudart -lnvrtc -Xlinker -rpath,/usr/local/cuda/lib64
rm -rf $OBJ
echo $ROOT/_variants/libimpact_b200_$TAG.so
