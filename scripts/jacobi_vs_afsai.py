"""Paper behaviour (Fig. 8): aFSAI-PCG vs Jacobi-PCG, total time
(set-up + solve) and iterations to an 8-order residual drop, on one B200.
Jacobi is aFSAI with k_max = 0 (G = D^-1/2, SURVEY pin P11), through the same
kernels; aFSAI with the fp64 and the fp32 set-up.  usage: jacobi_vs_afsai.py [M2 M3 ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import afsai_inputs as ai
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

names = sys.argv[1:] or ["M2", "M3"]
ctx = Context()
out = {}
for name in names:
    cfg = ai.CONFIGS[name]
    A = cfg["make"]()
    dA = DeviceCSR.from_numpy(A)
    b, _ = ai.rhs_for(A)
    bd = torch.from_numpy(b).cuda()
    res = {}
    for label, k, prec in (("jacobi", 0, "fp64"), ("afsai", cfg["nsteps"], "fp64"), ("afsai_fp32", cfg["nsteps"], "fp32")):
        best = None
        for rep in range(3):  # first = warm-up
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            F = Factor(ctx, dA, k, cfg["s"], cfg["eps"], cfg["max_row_nnz"], precision=prec)
            e1.record()
            x, rep_ = F.pcg(bd, tol=1e-8, max_iters=20000)
            e2.record()
            torch.cuda.synchronize()
            r = {"setup_ms": e0.elapsed_time(e1), "solve_ms": e1.elapsed_time(e2), "iters": rep_["iters"],
                 "converged": bool(rep_["converged"]), "true_rel_res": rep_["true_rel_res"], "nnz_G": F.nnz[0]}
            r["total_ms"] = r["setup_ms"] + r["solve_ms"]
            F.close()
            if rep > 0 and (best is None or r["total_ms"] < best["total_ms"]):
                best = r
        res[label] = best
    res["speedup_total"] = res["jacobi"]["total_ms"] / res["afsai"]["total_ms"]
    res["speedup_total_fp32"] = res["jacobi"]["total_ms"] / res["afsai_fp32"]["total_ms"]
    res["iters_ratio"] = res["afsai"]["iters"] / res["jacobi"]["iters"]
    out[name] = res
    print(name, json.dumps(res), flush=True)
print(json.dumps(out))
