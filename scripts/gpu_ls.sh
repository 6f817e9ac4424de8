#!/bin/bash
cd "$(dirname "$0")/.."
python scripts/prof_setup.py poisson 100 3 > gpurun_out/prof_p100_default.json 2>&1
python - <<'PY'
import json
d=json.load(open('gpurun_out/prof_p100_default.json'))
per_row=sum(d['phase_cycles_per_row'].values())
T=d['ms_rows']*1e-3
print('ms', d['ms_rows'], 'per-row cycles', per_row)
for f in (1.965e9, 1.8e9):
    R = 1e6*per_row/(148*f*T)
    print('implied rows in flight per SM at %.2f GHz: %.1f' % (f/1e9, R))
PY
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
