"""Small set-up + apply + PCG cases over every kernel plan (lockstep, hits, pattern-row,
scan, the retry path), fp64 and fp32 (fp64 only with AFSAI_CASES_FP64_ONLY=1); run with the
bounds-checked library by tests/test_bounds_checked.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import afsai_inputs as ai
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

ctx = Context()
cases = [(ai.poisson2d(32, 32), 10, 1, 1 << 30), (ai.poisson3d(16), 20, 2, 1 << 30),
         (ai.poisson3d(8), 4, 5, 1 << 30), (ai.fe_elasticity(4), 30, 3, 100),
         (ai.random_sparse_spd(1500, 10, sub=4), 6, 5, 12)]
for prec in ("fp64",) if os.environ.get("AFSAI_CASES_FP64_ONLY") else ("fp64", "fp32"):
    for A, k, s, cap in cases:
        F = Factor(ctx, DeviceCSR.from_numpy(A), k, s, 0.0, cap, precision=prec)
        b, _ = ai.rhs_for(A)
        bd = torch.from_numpy(b).cuda()
        F.apply(bd)
        x, rep = F.pcg(bd, tol=1e-8, max_iters=2000)
        assert rep["converged"], (A.name, prec)
        F.close()
os.environ["AFSAI_TABLE"] = "64"   # forced overflows: the retry passes
A = ai.fe_elasticity(4)
F = Factor(ctx, DeviceCSR.from_numpy(A), 30, 3, 0.0, 100)
assert F.stats()["retried_rows"] > 0
F.close()
ctx.close()
torch.cuda.synchronize()
print("sanitize cases ok")
