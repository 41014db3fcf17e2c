#!/bin/bash
# full ncu capture of one n x n x n frob_dgemm (the kernel and shape of the three Frobenius GEMMs)
mkdir -p gpurun_out
n=${1:-16384}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 2 -c 1 \
  -o gpurun_out/full_gemm$n python tools/gemm_one.py $n > gpurun_out/ncu_gemm$n.log 2>&1; echo gemm$n=$?
python tools/ncu_summary.py gpurun_out/full_gemm$n.ncu-rep > gpurun_out/ncu_full_gemm$n.txt 2>&1
ncu -i gpurun_out/full_gemm$n.ncu-rep --page raw --csv > gpurun_out/raw_full_gemm$n.csv 2>&1
ncu -i gpurun_out/full_gemm$n.ncu-rep --page source --csv > gpurun_out/src_full_gemm$n.csv 2>&1
