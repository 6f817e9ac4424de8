#!/bin/bash
# miniwarp width sweep of the PCG SpMVs on one workload (scripts/pcg_kernel_times.py)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
WL=${WL:-M3}
OUT=${OUT:-gpurun_out/spmv_sweep_$WL.jsonl}
for WA in 1 2 4; do for WG in 2 4 8; do
  AFSAI_SPMV_WIDTH_A=$WA AFSAI_SPMV_WIDTH_G=$WG AFSAI_SPMV_WIDTH_GT=$WG python scripts/pcg_kernel_times.py $WL >> $OUT 2>&1
done; done
