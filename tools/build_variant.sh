#!/bin/bash
# Build a variant of libwinoleg_b200.so with extra nvcc defines into gpurun_variants/<name>.so
# (measurement of kernel variants via WL_LIB_PATH).  Usage: tools/build_variant.sh name "-DFOO=1 ..."
set -e
cd "$(dirname "$0")/../paper_2004_11077_b200/csrc"
D=/tmp/variant_$1; mkdir -p $D
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c -o $D/wl_forward.o wl_forward.cu
nvcc $ARCH -shared -o ../../gpurun_variants/$1.so $D/wl_forward.o wl_backward.o wl_float.o wl_direct.o -lcudart -lcublas
echo built gpurun_variants/$1.so
