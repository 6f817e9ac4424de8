"""Multi-GPU parity under torchrun (one process per GPU, NCCL), against the CPU ORACLE:
  - the local rows of G from the N-GPU set-up are bitwise the oracle's rows
    (exact halo; row independence P:370-372);
  - the local rows of G^T are bitwise the oracle transpose's rows (C10);
  - afsai_apply matches oracle.apply within the SpMV rounding bound;
  - PCG iterations within 1 of the oracle PCG (BASELINE.json north_star);
  - error agreement: a matrix that is not SPD in the LAST rank's rows only makes
    every rank return an error (no rank is left waiting in a collective).
Prints one JSON document on rank 0 with "ok"."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import afsai_inputs as ai
import oracle
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
ctx = Context()
u = 2.0 ** -53
for name, A, k, s, cap in cases:
    n = A.n
    bounds = [n * q // world for q in range(world + 1)]
    b, e = bounds[rank], bounds[rank + 1]
    # oracle: this rank's rows of G, the full G / G^T for apply and PCG
    Gref, Tref, _ = oracle.setup_full(A, k, s, 0.0, cap)
    bvec, _ = ai.rhs_for(A)
    pr = oracle.pcg(A, Gref, Tref, bvec, tol=1e-8, max_iters=5000)
    rv = ai.rng("vectors", 21).standard_normal(n)
    zref = oracle.apply(Gref, Tref, rv)
    # N-GPU
    dA = DeviceCSR.from_numpy(A, row_begin=b, n_rows=e - b)
    F = Factor(ctx, dA, k, s, 0.0, cap)
    rp, ci, v = (t.cpu().numpy() for t in F.G())
    a0, a1 = Gref.rowptr[b], Gref.rowptr[e]
    ok_G = (np.array_equal(rp, Gref.rowptr[b:e + 1] - a0) and np.array_equal(ci, Gref.col[a0:a1])
            and np.array_equal(v.view(np.int64), Gref.val[a0:a1].view(np.int64)))
    trp, tci, tv = (t.cpu().numpy() for t in F.Gt())
    t0, t1 = Tref.rowptr[b], Tref.rowptr[e]
    ok_T = (np.array_equal(trp, Tref.rowptr[b:e + 1] - t0) and np.array_equal(tci, Tref.col[t0:t1])
            and np.array_equal(tv.view(np.int64), Tref.val[t0:t1].view(np.int64)))
    z = F.apply(torch.from_numpy(rv[b:e].copy()).cuda()).cpu().numpy()
    bound = 2 * 64 * u * (abs(Tref.to_scipy()) @ (abs(Gref.to_scipy()) @ np.abs(rv)))[b:e] + 1e-300
    ok_apply = bool(np.all(np.abs(z - zref[b:e]) <= bound))
    x, rep = F.pcg(torch.from_numpy(bvec[b:e].copy()).cuda(), tol=1e-8, max_iters=5000)
    stats = F.stats()
    results[name] = {"G_bitwise_vs_oracle": bool(ok_G), "Gt_bitwise_vs_oracle": bool(ok_T),
                     "apply_within_bound_vs_oracle": ok_apply,
                     "iters_N": rep["iters"], "iters_oracle": pr.iters, "true_rel_res": rep["true_rel_res"],
                     "halo_rows": stats["halo_rows"], "ms_total": stats["ms_total"], "ms_halo": stats["ms_halo"]}
    F.close()
# bounded-communication set-up: halo_k = 1, 2 against the oracle on A[I_p, I_p]
for name, A, k, s, cap in [("poisson3d_24", ai.poisson3d(24), 20, 2, 1000), ("fe_7", ai.fe_elasticity(7), 30, 3, 100)]:
    n = A.n
    bounds = [n * q // world for q in range(world + 1)]
    b, e = bounds[rank], bounds[rank + 1]
    bvec, _ = ai.rhs_for(A)
    for hk in (1, 2):
        ref, used = oracle.setup_bounded(A, bounds, rank, hk, k, s, 0.0, cap)
        F = Factor(ctx, DeviceCSR.from_numpy(A, row_begin=b, n_rows=e - b), k, s, 0.0, cap, halo_k=hk)
        rp, ci, v = (t.cpu().numpy() for t in F.G())
        ok = True
        for t in range(e - b):
            c0, v0 = ref.row(t)
            if not (np.array_equal(ci[rp[t]:rp[t + 1]], c0) and
                    np.array_equal(v[rp[t]:rp[t + 1]].view(np.int64), v0.view(np.int64))):
                ok = False
                break
        x, rep = F.pcg(torch.from_numpy(bvec[b:e].copy()).cuda(), tol=1e-8, max_iters=5000)
        st = F.stats()
        mask = [q for q in range(world) if (st["halo_mask"] >> q) & 1]
        results[f"{name}_halo_k{hk}"] = {"G_bitwise_vs_oracle": bool(ok), "stripes": mask, "oracle_stripes": used,
                                         "iters_N": rep["iters"], "converged": bool(rep["converged"]),
                                         "halo_rows": st["halo_rows"], "halo_bytes": st["halo_bytes"]}
        F.close()
# fp32 set-up on N GPUs against the fp32 oracle
for name, A, k, s, cap in [("hetero_16", ai.hetero_poisson3d(16), 20, 2, 1000), ("fe_7", ai.fe_elasticity(7), 30, 3, 100)]:
    n = A.n
    bounds = [n * q // world for q in range(world + 1)]
    b, e = bounds[rank], bounds[rank + 1]
    Gr = oracle.setup(A, k, s, 0.0, cap, precision="fp32").to_csr(n)
    F = Factor(ctx, DeviceCSR.from_numpy(A, row_begin=b, n_rows=e - b), k, s, 0.0, cap, precision="fp32")
    rp, ci, v = (t.cpu().numpy() for t in F.G())
    a0, a1 = Gr.rowptr[b], Gr.rowptr[e]
    ok = (np.array_equal(rp, Gr.rowptr[b:e + 1] - a0) and np.array_equal(ci, Gr.col[a0:a1])
          and np.array_equal(v.view(np.int64), Gr.val[a0:a1].view(np.int64)))
    bvec, _ = ai.rhs_for(A)
    x, rep = F.pcg(torch.from_numpy(bvec[b:e].copy()).cuda(), tol=1e-8, max_iters=5000)
    results[f"{name}_fp32"] = {"G_bitwise_vs_oracle": bool(ok), "converged": bool(rep["converged"]),
                               "iters_N": rep["iters"], "stripes": [], "oracle_stripes": []}
    F.close()
# error agreement: row n-1 has a tiny diagonal (psi < 0 at step 1 on the last rank only)
B = ai.poisson3d(12)
val = B.val.copy()
last = B.n - 1
val[B.rowptr[last]:B.rowptr[last + 1]][B.col[B.rowptr[last]:B.rowptr[last + 1]] == last] = 0.01
B = ai.CSR(B.n, B.rowptr, B.col, val)
try:
    oracle.setup(B, 20, 2)
    oracle_code = 0
except oracle.OracleError as ex:
    oracle_code = ex.code
bounds = [B.n * q // world for q in range(world + 1)]
b, e = bounds[rank], bounds[rank + 1]
try:
    Factor(ctx, DeviceCSR.from_numpy(B, row_begin=b, n_rows=e - b), 20, 2, 0.0, 1000).close()
    code = 0
except capi.AfsaiError as ex:
    code = ex.code
results["error_agreement"] = {"code": code, "oracle_code": oracle_code,
                              "ok": code != 0 and (rank != world - 1 or code == capi.AFSAI_ENOTSPD)}
ctx.close()
allr = [None] * world
dist.all_gather_object(allr, results)
if rank == 0:
    ok = all(r[c]["G_bitwise_vs_oracle"] and r[c]["Gt_bitwise_vs_oracle"] and r[c]["apply_within_bound_vs_oracle"]
             and abs(r[c]["iters_N"] - r[c]["iters_oracle"]) <= 1 and r[c]["true_rel_res"] <= 1e-7
             for r in allr for c in r if c != "error_agreement" and "_halo_k" not in c and "_fp32" not in c)
    ok = ok and all(r[c]["G_bitwise_vs_oracle"] and r[c]["converged"] and r[c]["stripes"] == r[c]["oracle_stripes"]
                    for r in allr for c in r if "_halo_k" in c or "_fp32" in c)
    ok = ok and all(r["error_agreement"]["ok"] for r in allr) and allr[0]["error_agreement"]["oracle_code"] == 2
    print(json.dumps({"world": world, "ok": ok, "ranks": allr}, indent=1))
dist.destroy_process_group()
