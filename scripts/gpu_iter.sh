#!/bin/bash
# parity tests + set-up profile on M2 (default plan and variants) and a small FE case
cd "$(dirname "$0")/.."
bash scripts/gpu_check.sh
python scripts/prof_setup.py poisson 100 2 > gpurun_out/prof_p100.json 2>&1; echo "p100 $?"
AFSAI_HITS=0 python scripts/prof_setup.py poisson 100 2 > gpurun_out/prof_p100_scan.json 2>&1; echo "p100 scan $?"
python scripts/prof_setup.py fe 20 2 > gpurun_out/prof_fe20.json 2>&1; echo "fe20 $?"
