#!/bin/bash
# Round evidence on one GPU: bench line, its ncu launch list, M2 set-up ncu capture, oracle timings.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/ev_nproc.txt; lscpu | grep -i "model name" >> gpurun_out/ev_nproc.txt
timeout 600 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.log; echo "bench $?"
tail -1 gpurun_out/ev_bench.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu_bench.log 2>&1; echo "ncu-list $?"
python scripts/summarize_launches.py gpurun_out/ev_launches.csv > gpurun_out/ev_launches_summary.txt 2>&1
gzip -f gpurun_out/ev_launches.csv
KIND=poisson N=100 TAG=p100f bash scripts/gpu_ncu_setup.sh
echo "oracle skipped (unchanged)"
