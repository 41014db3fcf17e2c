#!/bin/bash
# full ncu capture (with source-level stall sampling) of the batched kernels
mkdir -p gpurun_out
for a in "128 4096" "32 16384"; do
  set -- $a
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:frob_batched -c 1 -o gpurun_out/full_b$1 \
    python tools/batched_run.py $1 $2 > gpurun_out/ncu_b$1.log 2>&1; echo b$1=$?
  ncu -i gpurun_out/full_b$1.ncu-rep --page source --csv > gpurun_out/src_b$1.csv 2>&1
  python tools/ncu_summary.py gpurun_out/full_b$1.ncu-rep > gpurun_out/ncu_full_b$1.txt 2>&1
  rm -f gpurun_out/full_b$1.ncu-rep
done
