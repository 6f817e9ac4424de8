#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out; : > gpurun_out/repro2.jsonl
for P in 1 2; do timeout 300 python scripts/repro_block.py M3 4 $P 4 >> gpurun_out/repro2.jsonl 2>>gpurun_out/repro2.err; done
AFSAI_DEBUG_LIB=1 timeout 300 python scripts/repro_block.py M3 4 1 4 >> gpurun_out/repro2.jsonl 2>>gpurun_out/repro2.err
timeout 300 python scripts/repro_block.py M2 1 0 4 >> gpurun_out/repro2.jsonl 2>>gpurun_out/repro2.err
timeout 300 python scripts/repro_block.py M3 1 0 3 >> gpurun_out/repro2.jsonl 2>>gpurun_out/repro2.err
cat gpurun_out/repro2.jsonl; grep -a "afsai bounds" gpurun_out/repro2.err | head
