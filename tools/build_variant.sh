#!/bin/bash
# Build an experimental variant of libnao_b200.so with extra -D flags for one source:
#   tools/build_variant.sh <source stem> <out.so> -DFOO=1 ...
# (objects of the other sources come from build/obj of the normal build)
set -e
cd "$(dirname "$0")/.."
stem=$1; out=$2; shift 2
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NVCC $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include "$@" \
    -c paper_2510_16028_b200/csrc/$stem.cu -o build/var_$stem.o
objs=$(ls build/obj/*.o | grep -v "/$stem.o")
$NVCC $ARCH -shared -cudart shared -o "$out" $objs build/var_$stem.o -Xlinker -rpath,/usr/local/cuda/lib64
echo "$out"
