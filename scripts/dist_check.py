"""Multi-GPU checks under torchrun (one process per GPU, NCCL):
  - G from the N-GPU set-up is bitwise the 1-GPU G (exact halo);
  - G^T rows equal the 1-GPU G^T rows;
  - afsai_apply equals the 1-GPU apply within the SpMV rounding bound;
  - PCG iterations equal the 1-GPU count within 1.
Each rank also runs the 1-GPU path on the whole (small) matrix for reference."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import afsai_inputs as ai
from paper_2010_14175_b200 import capi
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
results = {}
cases = [("poisson3d_24", ai.poisson3d(24), 20, 2, 1000),
         ("hetero_16", ai.hetero_poisson3d(16), 20, 2, 1000),
         ("fe_7", ai.fe_elasticity(7), 30, 3, 100)]
for name, A, k, s, cap in cases:
    n = A.n
    bounds = [n * q // world for q in range(world + 1)]
    b, e = bounds[rank], bounds[rank + 1]
    # 1-GPU reference on this rank (non-NCCL context)
    h1 = capi.afsai_ctx_create(torch.cuda.current_stream().cuda_stream)
    Afull = DeviceCSR.from_numpy(A)
    Afull_c = Afull.c()
    F1 = capi.afsai_setup(h1, Afull_c, k, s, 0.0, cap)
    nnz1, nnzt1 = capi.afsai_factor_nnz(F1)
    g1 = [torch.empty(n + 1, dtype=torch.int64, device="cuda"), torch.empty(nnz1, dtype=torch.int32, device="cuda"),
          torch.empty(nnz1, dtype=torch.float64, device="cuda")]
    capi.afsai_factor_copy(F1, 0, *g1)
    t1 = [torch.empty(n + 1, dtype=torch.int64, device="cuda"), torch.empty(nnzt1, dtype=torch.int32, device="cuda"),
          torch.empty(nnzt1, dtype=torch.float64, device="cuda")]
    capi.afsai_factor_copy(F1, 1, *t1)
    bvec, _ = ai.rhs_for(A)
    rep1 = capi.afsai_pcg(h1, Afull_c, F1, torch.from_numpy(bvec).cuda(),
                          torch.empty(n, dtype=torch.float64, device="cuda"), 1e-8, 5000)
    r = torch.from_numpy(ai.rng("vectors", 21).standard_normal(n)).cuda()
    z1 = torch.empty_like(r)
    capi.afsai_apply(h1, F1, r, z1)
    # N-GPU
    ctx = Context()
    dA = DeviceCSR.from_numpy(A, row_begin=b, n_rows=e - b)
    F = Factor(ctx, dA, k, s, 0.0, cap)
    rp, ci, v = F.G()
    rp1 = g1[0][b:e + 1] - g1[0][b]
    lo1, hi1 = int(g1[0][b]), int(g1[0][e])
    ok_G = (torch.equal(rp, rp1) and torch.equal(ci, g1[1][lo1:hi1])
            and torch.equal(v.view(torch.int64), g1[2][lo1:hi1].view(torch.int64)))
    trp, tci, tv = F.Gt()
    trp1 = t1[0][b:e + 1] - t1[0][b]
    tl, th = int(t1[0][b]), int(t1[0][e])
    ok_T = (torch.equal(trp, trp1) and torch.equal(tci, t1[1][tl:th])
            and torch.equal(tv.view(torch.int64), t1[2][tl:th].view(torch.int64)))
    z = F.apply(r[b:e].contiguous())
    dz = (z - z1[b:e]).abs().max().item() / max(z1.abs().max().item(), 1e-300)
    x, rep = F.pcg(torch.from_numpy(bvec[b:e].copy()).cuda(), tol=1e-8, max_iters=5000)
    stats = F.stats()
    results[name] = {"G_bitwise": bool(ok_G), "Gt_bitwise": bool(ok_T), "apply_rel_diff": dz,
                     "iters_N": rep["iters"], "iters_1": rep1.iters, "true_rel_res": rep["true_rel_res"],
                     "halo_rows": stats["halo_rows"], "ms_total": stats["ms_total"], "ms_halo": stats["ms_halo"]}
    F.close()
    ctx.close()
    capi.afsai_factor_destroy(F1)
    capi.afsai_ctx_destroy(h1)
allr = [None] * world
dist.all_gather_object(allr, results)
if rank == 0:
    ok = all(r[c]["G_bitwise"] and r[c]["Gt_bitwise"] and abs(r[c]["iters_N"] - r[c]["iters_1"]) <= 1
             and r[c]["apply_rel_diff"] < 1e-12 and r[c]["true_rel_res"] <= 1e-7 for r in allr for c in r)
    print(json.dumps({"world": world, "ok": ok, "ranks": allr}, indent=1))
dist.destroy_process_group()
