#!/bin/bash
# ncu --set full of the set-up kernel (KIND = poisson | hetero | fe, size N); text summaries only
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/ncu
N=${N:-40}
KIND=${KIND:-poisson}
TAG=${TAG:-v}
python scripts/prof_setup.py $KIND $N 2 > gpurun_out/prof_${KIND}${N}_$TAG.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:afsai_setup_rows -s 1 -c 1 \
   -o /tmp/ncu/setup_$TAG -f python scripts/prof_setup.py $KIND $N 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc $?"
python scripts/ncu_lines.py /tmp/ncu/setup_$TAG.ncu-rep "" 80 > gpurun_out/ncu_lines_$TAG.txt 2>&1
ncu -i /tmp/ncu/setup_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv 2>&1
ncu -i /tmp/ncu/setup_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_details_$TAG.csv 2>&1
ncu -i /tmp/ncu/setup_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_$TAG.csv 2>&1
ls -la gpurun_out/ncu_sass_$TAG.csv
