#!/bin/bash
# A/B build of libdgnn.so with extra nvcc flags for sample.cu (the other objects from the normal
# build): tools/build_variant.sh TAG -DDGNN_PART_THREADS=256 ...  ->  paper_2405_05231_b200/build/ab/libdgnn_TAG.so
# (select it at run time with DGNN_LIB=...).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_2405_05231_b200
TAG=$1; shift
python "$PKG/build.py" > /dev/null
mkdir -p "$PKG/build/ab"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
$NVCC -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC,-O2 \
    -Xptxas -O3 -I "$ROOT/include" "$@" -c "$PKG/csrc/sample.cu" -o "$PKG/build/ab/sample_$TAG.o"
OBJS=$(ls "$PKG"/build/*.cu.o | grep -v '/sample.cu.o$')
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o "$PKG/build/ab/libdgnn_$TAG.so" $OBJS "$PKG/build/ab/sample_$TAG.o" -lcudart
echo "$PKG/build/ab/libdgnn_$TAG.so"
