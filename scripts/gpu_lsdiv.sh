#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
KIND=poisson N=100 TAG=p100e bash scripts/gpu_ncu_setup.sh
timeout 1200 python scripts/measure_configs.py M3 M4 > gpurun_out/configs3.json 2> gpurun_out/configs3.log; echo "measure $?"
