#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; : > gpurun_out/m3x4.txt
run() {
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) scripts/measure_dist.py M3 3 > /tmp/o.json 2> /tmp/o.err
  echo "$* rc=$? $(grep -o '"T_p_ms": [0-9.]*' /tmp/o.json) $(grep -o 'failed at [^:]*:[0-9]*' /tmp/o.err | head -1)" >> gpurun_out/m3x4.txt
}
run X=1
run AFSAI_NOPROBE=1
run AFSAI_LOCKSTEP=0
run NCCL_P2P_DISABLE=1
run AFSAI_POOL_KEEP0=1
run X=2
cat gpurun_out/m3x4.txt
