"""Set-up / apply / PCG measurement of one BASELINE config on N GPUs (torchrun,
one process per GPU, NCCL) or on 1 GPU (plain python).  SURVEY §8(d) protocol:
T_p = max over ranks of the device-timed set-up (halo exchange included),
median of `reps` after one warm-up; G-nnz/s = global nnz(G) / T_p; apply GB/s
from 50 applies (max over ranks); PCG iterations and T_s.  Each rank builds
only its own rows (FE slabs via afsai_inputs.fe_elasticity_rows, in chunks).
usage: [torchrun --nproc-per-node N] measure_dist.py CONFIG [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import afsai_inputs as ai
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = ai.CONFIGS[name]
k, s, eps, cap = cfg["nsteps"], cfg["s"], cfg["eps"], cfg["max_row_nnz"]
FE_N = {"M4": 79, "M5": 159}
t0 = time.time()
if name in FE_N:
    N = FE_N[name]
    n = 3 * N ** 3
    lo, hi = n * rank // world, n * (rank + 1) // world
    parts, step = [], 1_500_000
    for a in range(lo, hi, step):
        parts.append(ai.fe_elasticity_rows(N, a, min(hi, a + step)))
    rp = np.zeros(hi - lo + 1, dtype=np.int64)
    off, pos = 0, 0
    for P in parts:
        rp[pos + 1: pos + P.n + 1] = P.rowptr[1:] + off
        off += P.nnz
        pos += P.n
    col = np.concatenate([P.col for P in parts])
    val = np.concatenate([P.val for P in parts])
    del parts
    dA = DeviceCSR(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(), n, lo)
    A_full = None
else:
    A_full = cfg["make"]()
    n = A_full.n
    lo, hi = n * rank // world, n * (rank + 1) // world
    dA = DeviceCSR.from_numpy(A_full, row_begin=lo, n_rows=hi - lo)
gen_s = time.time() - t0
ctx = Context()


def allmax(x):
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allsum(x):
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()


tp, st, F = [], None, None
for r in range(reps + 1):
    if F is not None:
        F.close()
    barrier()
    F = Factor(ctx, dA, k, s, eps, cap)
    st = F.stats()
    if r > 0:
        tp.append(allmax(st["ms_total"]))
Tp = float(np.median(tp))
nG_local = F.nnz[0]
nG = allsum(nG_local)
flop = allsum(2.0 * (st["fma_border"] + st["fma_backsub"] + st["fma_grad"]))
rows_ms = allmax(st["ms_rows"])
# apply: bytes of the two sparse products, summed over ranks
r_ = torch.rand(hi - lo, dtype=torch.float64, device="cuda")
z_ = torch.empty_like(r_)
for _ in range(3):
    F.apply(r_, z_)
barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    F.apply(r_, z_)
e1.record()
torch.cuda.synchronize()
ams = allmax(e0.elapsed_time(e1) / 50)
abytes = allsum(2 * (12 * nG_local + 8 * (hi - lo + 1)) + 32 * (hi - lo))
# PCG on b = A x* (x* seeded); each rank holds its slice of b
if A_full is not None:
    b_full, _ = ai.rhs_for(A_full)
    b_loc = torch.from_numpy(b_full[lo:hi]).cuda()
else:
    # FE: b = A x* with x* ~ U(-1,1) from the seeded generator, computed from the local rows
    # (input preparation with torch on the device: the host would need ~20 GB for M5)
    xs = torch.from_numpy(ai.rng("rhs").uniform(-1.0, 1.0, n)).cuda()
    cnt = dA.rowptr[1:] - dA.rowptr[:-1]
    rows = torch.repeat_interleave(torch.arange(hi - lo, device="cuda"), cnt)
    b_loc = torch.zeros(hi - lo, dtype=torch.float64, device="cuda")
    b_loc.index_add_(0, rows, dA.val * xs[dA.col.long()])
    del rows, xs
barrier()
x, rep = F.pcg(b_loc, tol=1e-8, max_iters=20000)
Ts = allmax(rep["ms_solve"])
fp64_peak = torch.cuda.get_device_properties(local).multi_processor_count * 64 * 2 * 1965e6
out = {"config": name, "n_gpus": world, "n": n, "nnz_G": nG, "gen_s_rank0": gen_s,
       "T_p_ms": Tp, "T_p_runs_ms": tp, "G_nnz_per_s": nG / (Tp * 1e-3),
       "rows_kernel_ms_max": rows_ms, "halo_ms_rank0": st["ms_halo"], "transpose_ms_rank0": st["ms_transpose"],
       "setup_fp64_frac": flop / (rows_ms * 1e-3) / (fp64_peak * world),
       "apply_ms": ams, "apply_GBs": abytes / (ams * 1e-3) / 1e9,
       "pcg_iters": rep["iters"], "pcg_converged": bool(rep["converged"]), "T_s_ms": Ts,
       "T_s_per_iter_ms": Ts / max(1, rep["iters"]), "true_rel_res": rep["true_rel_res"],
       "table": st["table_size"], "rows_per_cta": st["rows_per_cta"], "retried_rows": st["retried_rows"]}
if rank == 0:
    print(json.dumps(out), flush=True)
F.close()
ctx.close()
if world > 1:
    dist.destroy_process_group()
