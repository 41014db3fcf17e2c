#!/bin/bash
# libfrobinv with the kernel timeline tracer (-DFROB_TL) -> tools/libfrobinv_tl.so (not the product)
set -e
cd "$(dirname "$0")/../paper_2208_01239_b200/csrc"
for f in lu.cu lu2.cu tma.cu frob.cu batched.cu hpd.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -DFROB_TL -c $f -o /tmp/tl_${f%.cu}.o &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../../tools/libfrobinv_tl.so /tmp/tl_*.o -lcudart
