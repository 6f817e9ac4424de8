#!/bin/bash
# ncu --set full of the set-up kernel on Poisson N^3 for several LPR; text summaries only
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/ncu
N=${N:-32}
for L in ${LPRS:-32 8}; do
  AFSAI_LPR=$L python scripts/prof_setup.py poisson $N 2 > gpurun_out/prof_p${N}_l$L.json 2>&1 && \
  AFSAI_LPR=$L ncu --set full --clock-control none --import-source on -k regex:afsai_setup_rows -s 1 -c 1 \
     -o /tmp/ncu/setup_l$L -f python scripts/prof_setup.py poisson $N 2 > gpurun_out/ncu_l$L.log 2>&1
  echo "L$L rc $?"
  python scripts/ncu_lines.py /tmp/ncu/setup_l$L.ncu-rep "" 60 > gpurun_out/ncu_lines_l$L.txt 2>&1
  ncu -i /tmp/ncu/setup_l$L.ncu-rep --page details --csv > gpurun_out/ncu_details_l$L.csv 2>&1
  ncu -i /tmp/ncu/setup_l$L.ncu-rep --page raw --csv > gpurun_out/ncu_raw_l$L.csv 2>&1
done
ls -la /tmp/ncu
