#!/bin/bash
# M5 (the largest config) strong scaling after the FE kernel changes, plus the parity suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r02g}
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > gpurun_out/${TAG}_parity.log
for N in 1 4; do
  RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29800 + N))"
  [ $N = 1 ] && RUN=python
  timeout 1500 $RUN bench.py --gpus $N --workload M5 --steps 2 --warmup 1 --e2e-runs 1 --no-cpu-baseline \
    > gpurun_out/${TAG}_M5_$N.json 2> gpurun_out/${TAG}_M5_$N.log
  echo "M5 N=$N rc $?"
done
timeout 900 python bench.py --workload M4 --precision fp32 --steps 2 --warmup 1 --e2e-runs 1 --no-cpu-baseline \
  > gpurun_out/${TAG}_M4_fp32.json 2> gpurun_out/${TAG}_M4_fp32.log
cat gpurun_out/${TAG}_parity.log
for f in gpurun_out/${TAG}_M5_*.json gpurun_out/${TAG}_M4_fp32.json; do
  echo "$f: $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), "M G-nnz/s", round(d["ms_per_step"],1), "ms/step setup", round(d["setup_ms"],1), d["setup_phase_ms"], "iters", d["pcg_iters"], "solve", round(d["solve_ms"],1))' 2>/dev/null)"
done
