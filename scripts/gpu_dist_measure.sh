#!/bin/bash
# Multi-GPU measurements (run with gpurun --gpus N): CONFIGS on 1..N GPUs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
free -g | head -2 > gpurun_out/host_mem.txt
NG=$(nvidia-smi -L | wc -l)
for C in ${CONFIGS:-M3}; do
  for P in ${NLIST:-1 2 4}; do
    [ $P -gt $NG ] && continue
    if [ $P = 1 ]; then
      timeout 1500 python scripts/measure_dist.py $C ${REPS:-3} >> gpurun_out/dist_measure.jsonl 2>> gpurun_out/dist_measure.err
    else
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
        --master-port $((29500 + P)) scripts/measure_dist.py $C ${REPS:-3} >> gpurun_out/dist_measure.jsonl 2>> gpurun_out/dist_measure.err
    fi
    echo "$C x$P rc=$?"
  done
done
