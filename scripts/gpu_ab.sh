#!/bin/bash
# A/B of set-up kernel variants (lib/libafsai_b200_<v>.so built with build.py --variant=<v> -D...):
# parity (bitwise vs the oracle, test_setup_parity) and rows-kernel time on M2 / M3 per variant.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
VARS=${VARS:-"base smb opt1 opt1smb"}
for v in $VARS; do
  if [ "$v" = base ]; then unset AFSAI_LIB; else export AFSAI_LIB=$PWD/paper_2010_14175_b200/lib/libafsai_b200_$v.so; fi
  echo "== $v" >> gpurun_out/ab.log
  python -m pytest tests/test_gpu_parity.py -q -x -k "setup_parity" 2>&1 | tail -1 >> gpurun_out/ab.log
  IFS=';' read -ra CL <<< "${CFGS:-poisson 100;hetero 200}"
  for cfg in "${CL[@]}"; do
    python scripts/prof_setup.py $cfg 3 | python -c "import json,sys; d=json.load(sys.stdin); print('$v', '$cfg', round(d['ms_rows'],2), d['rows_per_cta'], d['phase_share'])" >> gpurun_out/ab.log 2>&1
  done
done
unset AFSAI_LIB
cat gpurun_out/ab.log
