#!/bin/bash
cd "$(dirname "$0")/.."
bash scripts/gpu_check.sh
python scripts/prof_setup.py poisson 100 2 > gpurun_out/prof_p100_ls16.json 2>&1; echo "ls16 $?"
