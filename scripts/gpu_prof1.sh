#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/prof_setup.py poisson 100 2 > gpurun_out/prof_p100.json 2>&1; echo "p100 $?"
python scripts/prof_setup.py fe 20 2 > gpurun_out/prof_fe20.json 2>&1; echo "fe20 $?"
python scripts/prof_setup.py poisson 40 2 > gpurun_out/prof_p40.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:afsai_setup_rows -s 1 -c 1 -o gpurun_out/setup_p40 \
   python scripts/prof_setup.py poisson 40 2 > gpurun_out/ncu_setup.log 2>&1; echo "ncu $?"
