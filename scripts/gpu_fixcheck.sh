#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo "parity $?"; tail -1 gpurun_out/parity.log
for P in 1 2 3; do timeout 300 python scripts/repro_block.py M3 4 $P 4 2>&1 | tail -1 | cut -c1-160; done
for t in 1 2 3; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800 + t)) scripts/measure_dist.py M3 3 > /tmp/o.json 2> /tmp/o$t.err
  echo "M3x4 try $t rc=$? $(grep -o '"T_p_ms": [0-9.]*' /tmp/o.json)"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29810 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench4 $?"
tail -1 gpurun_out/bench4.json | cut -c1-400
