#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_all.txt
lscpu | grep -i "model name\|^CPU(s)" > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
CUDA_VISIBLE_DEVICES=0 timeout 900 python scripts/measure_configs.py M1 M2 > gpurun_out/configs_m12.json 2> gpurun_out/configs_m12.log; echo "m12 $?"
rm -f gpurun_out/dist_measure.jsonl
CONFIGS="M3 M4 M5" NLIST="1 2 4" REPS=3 bash scripts/gpu_dist_measure.sh
