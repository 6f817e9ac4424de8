#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; : > gpurun_out/m3x4dbg.txt
for t in 1 2 3; do
  AFSAI_DEBUG_LIB=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + t)) scripts/measure_dist.py M3 3 > /tmp/o.json 2> /tmp/o$t.err
  echo "try $t rc=$? $(grep -o '"T_p_ms": [0-9.]*' /tmp/o.json)" >> gpurun_out/m3x4dbg.txt
  grep -a "afsai bounds\|failed at" /tmp/o$t.err | head -8 >> gpurun_out/m3x4dbg.txt
done
cat gpurun_out/m3x4dbg.txt
