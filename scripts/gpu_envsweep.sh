#!/bin/bash
# set-up rows-kernel time on Poisson N^3 under plan overrides (AFSAI_* env); one JSON line per variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${N:-100}
for v in "" "AFSAI_LOCKSTEP_LPR=8" "$@"; do
  echo "== $v" >> gpurun_out/envsweep.txt
  env $v timeout 300 python scripts/prof_setup.py ${KIND:-poisson} $N 2 2>&1 | python -c "import sys,json; d=json.load(sys.stdin); print(json.dumps({k:d[k] for k in ['ms_rows','rows_per_cta','table_size','nnz_G']}))" >> gpurun_out/envsweep.txt 2>&1
done
cat gpurun_out/envsweep.txt
