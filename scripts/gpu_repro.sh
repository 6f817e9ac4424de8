#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; : > gpurun_out/repro.jsonl
for P in 0 1 2 3; do timeout 300 python scripts/repro_block.py M3 4 $P >> gpurun_out/repro.jsonl 2>>gpurun_out/repro.err; done
AFSAI_NOPROBE=1 timeout 300 python scripts/repro_block.py M3 4 2 >> gpurun_out/repro.jsonl 2>>gpurun_out/repro.err
AFSAI_TABLE=256 timeout 300 python scripts/repro_block.py M3 4 2 >> gpurun_out/repro.jsonl 2>>gpurun_out/repro.err
AFSAI_LOCKSTEP=0 timeout 300 python scripts/repro_block.py M3 4 2 >> gpurun_out/repro.jsonl 2>>gpurun_out/repro.err
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/repro_block.py M3 4 2 >> gpurun_out/repro.jsonl 2>>gpurun_out/repro.err
cat gpurun_out/repro.jsonl
