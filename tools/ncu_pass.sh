#!/bin/bash
# ncu evidence pass (run under gpurun, one GPU): launch list of the default bench command and
# full captures of the top kernels.  Numbers printed under ncu are never bench values.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config2.csv \
  python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
cap() {  # tag, kernel regex, skip count, bench args...
  tag=$1; k=$2; sk=$3; shift 3
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $sk -c 1 -o gpurun_out/full_$tag \
    python bench.py "$@" --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1; echo $tag=$?
}
cap lu_panel2c lu_panel2c 20
cap lu_panel2 'lu_panel2_kernel' 40
cap lu_update2m lu_update2m 20
cap gemm gemm_kernel 8
cap gemm4096 gemm_kernel 40 --config 5 --n 4096
cap lu_update2m_4096 lu_update2m 20 --config 5 --n 4096
cap lu_panel2c_4096 lu_panel2c 20 --config 5 --n 4096
timeout 600 ncu --set full --import-source on --clock-control none -k regex:frob_batched -c 2 -o gpurun_out/full_batched \
  python tools/batched_run.py 128 1184 > gpurun_out/ncu_batched.log 2>&1; echo batched=$?
# summaries here (the .ncu-rep files are too large to bring back)
for f in gpurun_out/full_*.ncu-rep; do
  t=$(basename $f .ncu-rep); python tools/ncu_summary.py $f > gpurun_out/ncu_${t}.txt 2>&1
  ncu -i $f --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/raw_${t}.csv 2>&1
done
if [ -z "$KEEP_REP" ]; then rm -f gpurun_out/full_*.ncu-rep; fi
