#!/bin/bash
# ncu evidence pass (run under gpurun, one GPU): launch list of the default bench command and
# full captures of the top kernels.  Numbers printed under ncu are never bench values.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config2.csv \
  python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
for k in lu_panel2 lu_update2; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 -o gpurun_out/full_$k \
    python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1; echo $k=$?
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 8 -c 1 -o gpurun_out/full_gemm \
  python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; echo gemm=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 40 -c 1 -o gpurun_out/full_gemm4096 \
  python bench.py --config 5 --n 4096 --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_gemm4096.log 2>&1; echo gemm4096=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:frob_batched -c 2 -o gpurun_out/full_batched \
  python tools/batched_run.py 128 1184 > gpurun_out/ncu_batched.log 2>&1; echo batched=$?
