#!/bin/bash
# ncu --set full capture of the set-up rows kernel; the .ncu-rep is kept under gpurun_out/ (KIND, N, TAG)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${N:-48}; KIND=${KIND:-poisson}; TAG=${TAG:-v}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:afsai_setup_rows -s 1 -c 1 \
   -o gpurun_out/setup_$TAG -f python scripts/prof_setup.py $KIND $N 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc $?"
ls -la gpurun_out/setup_$TAG.ncu-rep
