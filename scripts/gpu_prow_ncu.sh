#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo "parity $?"
tail -3 gpurun_out/parity.log
KIND=fe N=40 TAG=${TAG:-fe40b} bash scripts/gpu_ncu_setup.sh
