#!/bin/bash
cd "$(dirname "$0")/.."
for L in 32 16; do
  AFSAI_LPR=$L python scripts/prof_setup.py poisson 100 2 > gpurun_out/prof_p100_l$L.json 2>&1; echo "L$L $?"
done
