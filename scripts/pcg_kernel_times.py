"""Per-class kernel times of one afsai_pcg (CUDA events per launch, afsai_ctx_kernel_times)
on a BASELINE.json config: average launch duration and achieved GB/s of the SpMVs against
their algorithmic bytes (12 B/nnz + 8 B/row rowptr + 8 B/row y + 8 B/row x; the fused
dot partner w of the fused dot adds 8 B/row, not counted).
usage: [AFSAI_SPMV_WIDTH=w] python scripts/pcg_kernel_times.py [M3]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import afsai_inputs as ai
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

name = sys.argv[1] if len(sys.argv) > 1 else "M3"
c = ai.CONFIGS[name]
A = c["make"]()
b, _ = ai.rhs_for(A)
ctx = Context()
dA = DeviceCSR.from_numpy(A)
F = Factor(ctx, dA, c["nsteps"], c["s"], c["eps"], c["max_row_nnz"])
bd = torch.from_numpy(b).cuda()
F.pcg(bd, tol=1e-8, max_iters=20000)
ctx.set_timing(True)
x, rep = F.pcg(bd, tol=1e-8, max_iters=20000)
kt = ctx.kernel_times()
ctx.set_timing(False)
n, nnzA = A.n, A.nnz
nG, nT = F.nnz
alg = {"spmv_A": 12 * nnzA + 32 * n, "spmv_G": 12 * nG + 32 * n, "spmv_Gt": 12 * nT + 32 * n}
out = {"workload": name, "width_env": {k: os.environ.get(k) for k in ("AFSAI_SPMV_WIDTH", "AFSAI_SPMV_WIDTH_A",
                                                                       "AFSAI_SPMV_WIDTH_G", "AFSAI_SPMV_WIDTH_GT")},
       "iters": rep["iters"],
       "ms_solve": rep["ms_solve"], "ms_per_iter": rep["ms_per_iter"], "classes": {}}
for k, (la, ms) in kt.items():
    if la:
        d = {"launches": la, "ms_per_launch": ms / la}
        if k in alg:
            d["alg_bytes"] = alg[k]
            d["GBps"] = alg[k] / (ms / la * 1e-3) / 1e9
        out["classes"][k] = d
print(json.dumps(out))
