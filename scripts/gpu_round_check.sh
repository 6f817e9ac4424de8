#!/bin/bash
# One box, NMAX GPUs: the GPU suite, the multi-GPU oracle checks, bench on M3 (1..NMAX GPUs),
# and the fp32 / fp64 set-up on M4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r02c}
NMAX=${NMAX:-4}
python -m pytest tests -q -m gpu --durations=6 2>&1 | tail -12 > gpurun_out/${TAG}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/${TAG}_tests.log 2>&1
for N in 2 4; do
  [ $N -gt $NMAX ] && break
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29700 + N)) \
    scripts/dist_check.py > gpurun_out/${TAG}_dist$N.json 2> gpurun_out/${TAG}_dist$N.err
done
python bench.py > gpurun_out/${TAG}_bench_M3_1.json 2> gpurun_out/${TAG}_bench_M3_1.log
for N in 2 4; do
  [ $N -gt $NMAX ] && break
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29710 + N)) \
    bench.py --gpus $N --no-cpu-baseline > gpurun_out/${TAG}_bench_M3_$N.json 2> gpurun_out/${TAG}_bench_M3_$N.log
done
for P in fp64 fp32; do
  python bench.py --workload M4 --precision $P --steps 2 --warmup 1 --e2e-runs 1 --no-cpu-baseline \
    > gpurun_out/${TAG}_bench_M4_$P.json 2> gpurun_out/${TAG}_bench_M4_$P.log
done
cat gpurun_out/${TAG}_tests.log
grep -h '"ok"' gpurun_out/${TAG}_dist*.json | head -4
for f in gpurun_out/${TAG}_bench_*.json; do
  echo "$f: $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), "M G-nnz/s", round(d["ms_per_step"],1), "ms/step setup", round(d["setup_ms"],1), d["setup_phase_ms"], "iters", d["pcg_iters"])' 2>/dev/null)"
done
