#!/bin/bash
# Round-2 ncu evidence pass (run under gpurun, one GPU).  Numbers printed under ncu are never bench
# values.  1) launch list of the default bench command (config 5, n = 16384); 2) full captures of the
# dominant kernel (gemm_kernel<double> at the n x n x n shape of the three Frobenius GEMMs), the
# blocked LU's panel and trailing GEMM at n = 16384, and the batched kernels (n = 32, 128).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config5.csv \
  python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
full() {  # tag, kernel regex, skip, count, command...
  tag=$1; k=$2; sk=$3; c=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $sk -c $c -o gpurun_out/full_$tag \
    "$@" > gpurun_out/ncu_$tag.log 2>&1; echo $tag=$?
}
full gemm16384 gemm_kernel 3 1 python tools/gemm_one.py 16384
full getrf16384_panel lu_panel_kernel 300 1 python tools/getrf_one.py 16384 1
full getrf16384_gemm gemm_kernel 40 3 python tools/getrf_one.py 16384 1
full batched32 frob_batched_kernel 0 1 python tools/batched_run.py 32 65536
full batched128 frob_batched128 0 1 python tools/batched_run.py 128 16384
for f in gpurun_out/full_*.ncu-rep; do
  t=$(basename $f .ncu-rep); python tools/ncu_summary.py $f > gpurun_out/ncu_${t}.txt 2>&1
  ncu -i $f --page raw --csv > gpurun_out/raw_${t}.csv 2>&1
done
python tools/ncu_launches.py gpurun_out/launches_config5.csv > gpurun_out/launches_config5.md 2>&1
if [ -z "$KEEP_REP" ]; then rm -f gpurun_out/full_*.ncu-rep; fi
