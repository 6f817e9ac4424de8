#!/bin/bash
# One GPU call: all-config measurement, a bench line, and the ncu launch list of the same bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python scripts/measure_configs.py ${CONFIGS:-M1 M2 M3 M4} > gpurun_out/configs.json 2> gpurun_out/configs.log; echo "measure $?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "bench $?"
tail -1 gpurun_out/bench.json
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo "ncu $?"
python scripts/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
rm -f gpurun_out/launches.csv.gz; gzip -f gpurun_out/launches.csv
fi
