#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo "parity $?"; tail -1 gpurun_out/parity.log
timeout 300 python scripts/prof_setup.py poisson 100 3 > gpurun_out/prof_p100_sw.json 2>&1; echo "p100 $?"
timeout 300 python scripts/prof_setup.py fe 40 2 > gpurun_out/prof_fe40_sw.json 2>&1; echo "fe40 $?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_sw.json 2> gpurun_out/bench_sw.log; echo "bench $?"
