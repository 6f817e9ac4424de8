"""Bounded-communication set-up vs the exact halo,
under torchrun (one process per GPU, NCCL).  For each workload and halo_k in
{0 (exact), 1, 2, 3}: set-up time T_p (max over ranks), set-up halo bytes received
(sum over ranks), nnz(G), PCG iterations to 1e-8 and solve time.  rank 0 prints
one JSON document.

usage: torchrun --nproc-per-node N scripts/measure_halo_k.py [M4] [thin]
  M4   : FE elasticity 79^3 nodes (1.48M rows), aFSAI 30x3 cap 100
  thinP: 3D Poisson 100 x 100 x (P N) (stripes of P planes per GPU, default 8), aFSAI 20x2
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import afsai_inputs as ai
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = Context()
names = [a for a in sys.argv[1:]] or ["M4", "thin"]
out = {"world": world, "workloads": {}}
for name in names:
    if name.startswith("thin"):
        pl = int(name[4:] or 8)   # planes per GPU stripe
        A = ai.poisson3d(100, 100, pl * world)
        k, s, eps, cap = 20, 2, 0.0, 1000
        desc = f"3D 7-point Poisson 100x100x{pl * world}: {pl} planes per GPU stripe, exact halo 20 planes"
    else:
        c = ai.CONFIGS[name]
        A = c["make"]()
        k, s, eps, cap = c["nsteps"], c["s"], c["eps"], c["max_row_nnz"]
        desc = c["desc"]
    n = A.n
    b, e = rank * n // world, (rank + 1) * n // world
    dA = DeviceCSR.from_numpy(A, row_begin=b, n_rows=e - b)
    bvec, _ = ai.rhs_for(A)
    bd = torch.from_numpy(np.ascontiguousarray(bvec[b:e])).cuda()
    rows = {}
    for hk in (0, 1, 2, 3):
        tp = []
        for rep_ in range(3):   # warm-up + 2 timed
            dist.barrier()
            F = Factor(ctx, dA, k, s, eps, cap, halo_k=hk)
            st = F.stats()
            if rep_ > 0:
                tp.append(st["ms_total"])
            if rep_ < 2:
                F.close()
        x, rep = F.pcg(bd, tol=1e-8, max_iters=20000)
        loc = torch.tensor([float(np.median(tp)), st["halo_bytes"], st["nnz_G"], rep["ms_solve"]],
                           dtype=torch.float64, device="cuda")
        mx, sm = loc.clone(), loc.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        masks = [None] * world
        dist.all_gather_object(masks, [q for q in range(world) if (st["halo_mask"] >> q) & 1] if hk else "exact")
        rows["exact" if hk == 0 else f"k={hk}"] = {
            "T_p_ms_max": float(mx[0]), "halo_bytes_total": int(sm[1]), "nnz_G": int(sm[2]),
            "pcg_iters": rep["iters"], "pcg_converged": bool(rep["converged"]), "T_s_ms_max": float(mx[3]),
            "true_rel_res": rep["true_rel_res"], "stripes_used_per_rank": masks}
        F.close()
    out["workloads"][name] = {"desc": desc, "n": n, "nnz_A": A.nnz, "params": [k, s, eps, cap], "by_halo": rows}
    if rank == 0:
        print(json.dumps({name: out["workloads"][name]}), file=sys.stderr, flush=True)
ctx.close()
if rank == 0:
    print(json.dumps(out, indent=1))
dist.destroy_process_group()
