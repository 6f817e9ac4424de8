#!/bin/bash
# Executed fp64 instruction counts of the set-up kernels' main pass (M3, and M4 for the
# FE pattern-row kernel) against the counted algorithmic FMAs (afsai_setup_stats_t).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M="smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,gpu__time_duration.sum"
for cfg in "hetero 200" "fe 79"; do
  set -- $cfg
  timeout 1800 ncu --metrics $M --clock-control none -k regex:afsai_setup_rows -c 8 --csv \
     --log-file gpurun_out/dfma_$1$2.csv python scripts/prof_setup.py $1 $2 1 > gpurun_out/dfma_$1$2.json 2> gpurun_out/dfma_$1$2.err
  echo "$cfg rc $?"
done
