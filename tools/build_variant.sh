#!/bin/bash
# Build an A/B variant of the C-ABI library with extra nvcc flags:
#   tools/build_variant.sh NAME -DMACRO=VALUE ...
# -> paper_2503_05046_b200/_native/variants/NAME.so; select it at run time with
#    MPMRB_LIB_PATH=paper_2503_05046_b200/_native/variants/NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_2503_05046_b200/_native/variants/$name
mkdir -p "$out"
objs=()
for src in capi binning scan mpm contact solver sim reorder cloth seed; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr "$@" -c paper_2503_05046_b200/csrc/$src.cu -o "$out/$src.o" &
  objs+=("$out/$src.o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out.so" "${objs[@]}" -lcudart
rm -rf "$out"
echo "$out.so"
