#!/bin/bash
cd "$(dirname "$0")/.."
python scripts/prof_setup.py fe 20 2 > gpurun_out/prof_fe20.json 2>&1; echo "fe20 $?"
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/pytest_full.log 2>&1; echo "full $?"
tail -5 gpurun_out/pytest_full.log
