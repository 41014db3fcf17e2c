#!/bin/bash
# One GPU iteration: parity tests, bench line, ncu launch list (run under gpurun).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.txt 2> gpurun_out/bench.err; cat gpurun_out/bench.txt; tail -3 gpurun_out/bench.err
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu=$?
python tools/launches.py gpurun_out/launches.csv | head -14
fi
