#!/bin/bash
# Build a variant of libwinoleg_b200.so into gpurun_variants/<name>.so: the translation units listed in
# $3 (default: all forward TUs) are recompiled with the extra nvcc defines $2, the rest reuse the
# in-tree objects.  Usage: tools/build_variant.sh name "-DFOO=1 ..." "wl_fwd_gemm wl_fwd_out_256"
set -e
cd "$(dirname "$0")/../paper_2004_11077_b200/csrc"
make -s -j8 > /dev/null
D=/tmp/variant_$1; mkdir -p $D ../../gpurun_variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
TUS=${3:-"wl_fwd wl_fwd_gemm wl_fwd_in_32 wl_fwd_in_64 wl_fwd_in_128 wl_fwd_in_256 wl_fwd_in_512 wl_fwd_out_64 wl_fwd_out_128 wl_fwd_out_256 wl_fwd_out_512"}
OBJS=""
for o in *.o; do
  b=${o%.o}
  if echo " $TUS " | grep -q " $b "; then
    nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c -o $D/$b.o $b.cu &
    OBJS="$OBJS $D/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
wait
nvcc $ARCH -shared -o ../../gpurun_variants/$1.so $OBJS -lcudart
echo built gpurun_variants/$1.so
