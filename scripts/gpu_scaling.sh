#!/bin/bash
# Strong scaling (M3 = bench default, M5 = the largest config) and box-scale weak scaling
# (121^3 rows per GPU) of bench.py on 1..NMAX GPUs of one box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NMAX=${NMAX:-4}
TAG=${TAG:-r02}
for N in 1 2 4 8; do
  [ $N -gt $NMAX ] && break
  RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29600 + N))"
  [ $N = 1 ] && RUN=python
  timeout 900 $RUN bench.py --gpus $N --workload M3 --no-cpu-baseline > gpurun_out/${TAG}_scale_M3_$N.json 2> gpurun_out/${TAG}_scale_M3_$N.log
  echo "M3 N=$N rc $?"
  timeout 900 $RUN bench.py --gpus $N --weak --nx 121 --no-cpu-baseline > gpurun_out/${TAG}_weak121_$N.json 2> gpurun_out/${TAG}_weak121_$N.log
  echo "weak121 N=$N rc $?"
  if [ -z "$SKIP_M5" ]; then
    timeout 1500 $RUN bench.py --gpus $N --workload M5 --steps 2 --warmup 1 --e2e-runs 1 --no-cpu-baseline > gpurun_out/${TAG}_scale_M5_$N.json 2> gpurun_out/${TAG}_scale_M5_$N.log
    echo "M5 N=$N rc $?"
  fi
done
for f in gpurun_out/${TAG}_scale_*.json gpurun_out/${TAG}_weak121_*.json; do
  echo "$f: $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), "M G-nnz/s", round(d["ms_per_step"],1), "ms/step setup", round(d["setup_ms"],1), "iters", d["pcg_iters"])' 2>/dev/null)"
done
