#!/bin/bash
# Full measurement pass (run under gpurun): every config's bench line -> gpurun_out/bench_*.json
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/gpu_info.txt 2>&1
lscpu | head -20 > gpurun_out/cpu_info.txt 2>&1
run() { tag=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "$tag rc=$?"; cut -c1-200 gpurun_out/bench_$tag.json; }
run config5_n16384 --steps 20 --warmup 5
run reference_config5 --impl reference --steps 3 --warmup 1
run config1 --config 1 --steps 50 --warmup 10 --no-cpu-baseline
run config2 --config 2 --steps 20 --warmup 5 --no-cpu-baseline
run config3 --config 3 --steps 5 --warmup 3 --no-cpu-baseline
run config4 --config 4 --steps 3 --warmup 3 --no-cpu-baseline
run config5_n2048 --config 5 --n 2048 --steps 10 --warmup 3 --no-cpu-baseline
run config5_n4096 --config 5 --n 4096 --steps 5 --warmup 3 --no-cpu-baseline
run config5_n8192 --config 5 --n 8192 --steps 3 --warmup 3 --no-cpu-baseline
