"""Profile helper: afsai_setup + one afsai_pcg on a BASELINE.json config (default M3),
for ncu captures of the solve kernels (SpMVs t = G r, z = G^T t, q = A p; PCG vectors)."""
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
F = Factor(ctx, DeviceCSR.from_numpy(A), c["nsteps"], c["s"], c["eps"], c["max_row_nnz"])
x, rep = F.pcg(torch.from_numpy(b).cuda(), tol=1e-8, max_iters=20000)
print(name, "nnz(A)", A.nnz, "n", A.n, "nnz(G)", F.nnz, "iters", rep["iters"])
