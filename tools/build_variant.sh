#!/bin/bash
# Build an A/B variant of the library with extra nvcc flags:
#   tools/build_variant.sh NAME -DFOO=1 ...   ->  build/variants/NAME.so
# and load it with RFPK_LIB=build/variants/NAME.so (paper_0901_1696_b200/_capi.py).
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
obj=$root/build/variants/$name
mkdir -p "$obj"
cd "$root/paper_0901_1696_b200/csrc"
for f in gemm blas rfp capi batched tile_potrf; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c $f.cu -o "$obj/$f.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build/variants/$name.so" "$obj"/*.o -lcudart
