"""Measure the BASELINE.json configs on one GPU (SURVEY §8(d) protocol):
T_p (median of reps after one warm-up), G-nnz/s, set-up fp64 fraction, apply
GB/s (mean of 50 applies), PCG iterations and T_s; the oracle timed on the same
host (full for small configs, a seeded row sample otherwise, extrapolated and
labelled so).  Writes one JSON document to stdout."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import afsai_inputs as ai
import oracle
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

names = sys.argv[1:] or ["M1", "M2", "M3", "M4"]
cores = os.cpu_count() or 1
ctx = Context()
fp64_peak = torch.cuda.get_device_properties(0).multi_processor_count * 64 * 2 * 1965e6
hbm_peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9 if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6.45e12
out = {"cores": cores, "fp64_peak_tflops": fp64_peak / 1e12, "hbm_peak_gbs": hbm_peak / 1e9, "configs": {}}
for name in names:
    cfg = ai.CONFIGS[name]
    t0 = time.time()
    A = cfg["make"]()
    gen_s = time.time() - t0
    k, s, eps, cap = cfg["nsteps"], cfg["s"], cfg["eps"], cfg["max_row_nnz"]
    dA = DeviceCSR.from_numpy(A)
    reps = 3 if A.n <= 2_000_000 and name not in ("M4",) else 2
    tp, st = [], None
    for r in range(reps + 1):  # one warm-up (pool growth, module load), then reps
        torch.cuda.synchronize()
        F = Factor(ctx, dA, k, s, eps, cap)
        st = F.stats()
        if r > 0:
            tp.append(st["ms_total"])
        if r < reps:
            F.close()
    Tp = float(np.median(tp))
    flop = 2.0 * (st["fma_border"] + st["fma_backsub"] + st["fma_grad"])
    # apply
    r = torch.rand(A.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    for _ in range(3):
        F.apply(r, z)
    ctx.set_timing(True)
    for _ in range(50):
        F.apply(r, z)
    kt = ctx.kernel_times()
    ctx.set_timing(False)
    nG, nT = F.nnz
    n = A.n
    abytes = 2 * (12 * nG + 8 * (n + 1) + 16 * n)
    ams = (kt["spmv_G"][1] + kt["spmv_Gt"][1]) / 50
    # PCG
    b, _ = ai.rhs_for(A)
    x, rep = F.pcg(torch.from_numpy(b).cuda(), tol=1e-8, max_iters=20000)
    res = {"n": n, "nnz_A": A.nnz, "nnz_G": nG, "params": [k, s, eps, cap], "gen_s": gen_s,
           "T_p_ms": Tp, "G_nnz_per_s": nG / (Tp * 1e-3),
           "setup_rows_kernel_ms": st["ms_rows"], "setup_flop": flop,
           "setup_fp64_tflops": flop / (st["ms_rows"] * 1e-3) / 1e12,
           "setup_fp64_frac": flop / (st["ms_rows"] * 1e-3) / fp64_peak,
           "setup_hbm_bytes": 12 * A.nnz + 8 * (n + 1) + 2 * (12 * nG + 8 * (n + 1)),
           "apply_ms": ams, "apply_GBs": abytes / (ams * 1e-3) / 1e9, "apply_hbm_frac": abytes / (ams * 1e-3) / hbm_peak,
           "pcg_iters": rep["iters"], "pcg_converged": bool(rep["converged"]), "T_s_ms": rep["ms_solve"],
           "T_s_per_iter_ms": rep["ms_per_iter"], "pcg_true_rel_res": rep["true_rel_res"],
           "stop_reasons": st["rows_by_reason"], "kernel_plan": {"table": st["table_size"],
                                                                  "rows_per_cta": st["rows_per_cta"],
                                                                  "retried_rows": st["retried_rows"]}}
    F.close()
    # oracle on the same host
    if n <= 1_100_000 and name != "M4":
        t0 = time.time()
        G, Gt, _ = oracle.setup_full(A, k, s, eps, cap, threads=cores)
        t1 = time.time()
        pr = oracle.pcg(A, G, Gt, b, tol=1e-8, max_iters=20000)
        t2 = time.time()
        res["oracle"] = {"T_p_s": t1 - t0, "pcg_s": t2 - t1, "pcg_iters": pr.iters, "cores": cores, "kind": "full"}
    else:
        rows = ai.sample_rows(n, 4000 if name != "M4" else 400, sub=7)
        t0 = time.time()
        oracle.setup(A, k, s, eps, cap, rows=rows, threads=cores, trace=False)
        dt = time.time() - t0
        res["oracle"] = {"T_p_s": dt * n / len(rows), "cores": cores,
                         "kind": f"extrapolated from a seeded sample of {len(rows)} rows ({dt:.1f} s)"}
    out["configs"][name] = res
    print(json.dumps({name: res}), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
