#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/spmv_sweep.py > gpurun_out/spmv_sweep.txt 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/bench_ll.json 2> gpurun_out/bench_ll.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_ll.log 2>&1
echo "ncu rc $?"
