#!/bin/bash
# Build an A/B variant of libfrobinv.so with extra nvcc flags into tools/ab/libfrobinv_$1.so
#   bash tools/build_variant.sh s4 -DFROB_GEMM_STAGES=4
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p tools/ab/$name
objs=""
for src in lu.cu lu2.cu tma.cu frob.cu batched.cu hpd.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr "$@" -c paper_2208_01239_b200/csrc/$src -o tools/ab/$name/${src%.cu}.o &
  objs="$objs tools/ab/$name/${src%.cu}.o"
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o tools/ab/libfrobinv_$name.so $objs -lcudart
echo tools/ab/libfrobinv_$name.so
