#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo "parity $?"; tail -1 gpurun_out/parity.log
rm -f gpurun_out/dist_measure.jsonl
CONFIGS="M3" NLIST="4" REPS=3 bash scripts/gpu_dist_measure.sh
CONFIGS="M5" NLIST="4 2" REPS=2 bash scripts/gpu_dist_measure.sh
