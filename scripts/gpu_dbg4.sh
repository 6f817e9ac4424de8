#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 scripts/dist_check.py > gpurun_out/dbg4_check.json 2> gpurun_out/dbg4_check.err; echo "check4 $?"
AFSAI_NOPROBE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 scripts/measure_dist.py M3 1 > gpurun_out/dbg4_noprobe.json 2> gpurun_out/dbg4_noprobe.err; echo "noprobe $?"
CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 scripts/measure_dist.py M3 1 > gpurun_out/dbg4_blocking.json 2> gpurun_out/dbg4_blocking.err; echo "blocking $?"
