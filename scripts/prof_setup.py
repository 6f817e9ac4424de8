"""Profile helper: one warm-up + one measured afsai_setup on a Poisson cube (or FE),
prints stats / phase shares as JSON.  Used under ncu for the set-up kernel.
phase_fp64_frac: per phase with fp64 work, the counted algorithmic FMAs x 2 over
(the phase's share of the in-kernel clock64 cycles x the rows-kernel time) over the
fp64 peak (37.2 TF: 148 SM x 64 DFMA/clk x 2 x 1965 MHz) -- the share-of-time split
is an approximation (phases of different warps overlap).
usage: prof_setup.py [poisson|hetero|fe] [N] [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import afsai_inputs as ai
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

kind = sys.argv[1] if len(sys.argv) > 1 else "poisson"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 100
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if kind == "poisson":
    A, k, s, cap = ai.poisson3d(N), 20, 2, 1000
elif kind == "hetero":
    A, k, s, cap = ai.hetero_poisson3d(N), 20, 2, 1000
else:
    A, k, s, cap = ai.fe_elasticity(N), 30, 3, 100
ctx = Context()
dA = DeviceCSR.from_numpy(A)
out = {}
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F = Factor(ctx, dA, k, s, 0.0, cap)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    st = F.stats()
    F.close()
out["wall_ms"] = (t1 - t0) * 1e3
out.update({k_: st[k_] for k_ in ["ms_total", "ms_rows", "ms_assemble", "ms_transpose", "nnz_G", "table_size",
                                   "rows_per_cta", "retried_rows", "fma_border", "fma_backsub", "fma_grad",
                                   "grad_entries", "steps_total", "rows_by_reason", "max_universe"]})
ph = st["phase_cycles"]
names = ["prologue", "gradient", "select", "gather", "border", "backsub", "output"]
tot = sum(ph)
out["phase_share"] = {n: round(v / tot, 4) for n, v in zip(names, ph)}
out["phase_cycles_per_row"] = {n: v / A.n for n, v in zip(names, ph)}
PEAK = 148 * 64 * 2 * 1.965e9
fl = {"gradient": st["fma_grad"], "border": st["fma_border"], "backsub": st["fma_backsub"]}
out["phase_fp64_frac"] = {n: round(2 * f / (out["phase_share"][n] * st["ms_rows"] * 1e-3) / PEAK, 5)
                          for n, f in fl.items() if out["phase_share"][n] > 0}
out["kernel_fp64_frac"] = round(2 * sum(fl.values()) / (st["ms_rows"] * 1e-3) / PEAK, 5)
print(json.dumps(out, indent=1))
