#!/bin/bash
# A/B of pattern-row (FE) set-up kernel variants: FE parity (bitwise vs the oracle)
# and rows-kernel time on FE N^3 per variant (lib/libafsai_b200_<v>.so, AFSAI_LIB).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
VARS=${VARS:-"base"}
SIZES=${SIZES:-"60 79"}
for v in $VARS; do
  if [ "$v" = base ]; then unset AFSAI_LIB; else export AFSAI_LIB=$PWD/paper_2010_14175_b200/lib/libafsai_b200_$v.so; fi
  echo "== $v" >> gpurun_out/abfe.log
  python -m pytest tests/test_gpu_parity.py -q -x -k "setup_parity and fe and not fp32" 2>&1 | tail -1 >> gpurun_out/abfe.log
  for n in $SIZES; do
    python scripts/prof_setup.py fe $n 2 | python -c "import json,sys; d=json.load(sys.stdin); print('$v', 'fe $n', round(d['ms_rows'],2), d['rows_per_cta'], d['phase_share'])" >> gpurun_out/abfe.log 2>&1
  done
done
unset AFSAI_LIB
cat gpurun_out/abfe.log
