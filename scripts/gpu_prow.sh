#!/bin/bash
# Parity of every set-up plan, then FE / hetero set-up profiles and the M3/M4 measurements.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo "parity $?"
tail -3 gpurun_out/parity.log
timeout 300 python scripts/prof_setup.py fe 20 2 > gpurun_out/prof_fe20.json 2>&1; echo "fe20 $?"
timeout 300 python scripts/prof_setup.py fe 40 2 > gpurun_out/prof_fe40.json 2>&1; echo "fe40 $?"
timeout 300 python scripts/prof_setup.py hetero 100 2 > gpurun_out/prof_het100.json 2>&1; echo "het100 $?"
timeout 1200 python scripts/measure_configs.py ${CONFIGS:-M3 M4} > gpurun_out/configs2.json 2> gpurun_out/configs2.log; echo "measure $?"
