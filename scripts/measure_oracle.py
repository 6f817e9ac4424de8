"""Oracle (CPU) set-up timing on all host cores for the BASELINE configs, on a
seeded row sample sized for a few seconds each (rows are independent, so a
sample's per-row rate extrapolates exactly in work; the extrapolation is
labelled).  M5's rows have M4's structure; its sample comes from a row slab.
Test / measurement infrastructure: the only place besides tests/ and bench.py's
baseline leg that runs oracle/.  usage: measure_oracle.py [CONFIG ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import afsai_inputs as ai
import oracle

names = sys.argv[1:] or ["M1", "M2", "M3", "M4", "M5"]
cores = os.cpu_count() or 1
SAMPLE = {"M3": 200_000, "M4": 16_000, "M5": 16_000}
res = {"cores": cores}
for name in names:
    cfg = ai.CONFIGS[name]
    k, s, eps, cap = cfg["nsteps"], cfg["s"], cfg["eps"], cfg["max_row_nnz"]
    if name == "M5":
        # a slab of whole node planes around the middle of the 159^3 mesh, enough for
        # the exact halo of its interior rows; timed rows are the slab's middle third
        N = 159
        n = 3 * N ** 3
        plane = 3 * N * N
        lo = (n // 2 // plane) * plane - 12 * plane
        A = ai.fe_elasticity_rows(N, lo, lo + 24 * plane)
        # re-index to a standalone square matrix over [lo, lo + 24 planes): columns
        # outside are dropped (rows far from the cut are unaffected: exact halo)
        keep = (A.col >= lo) & (A.col < lo + 24 * plane)
        rows = np.repeat(np.arange(A.n), np.diff(A.rowptr))
        cnt = np.bincount(rows[keep], minlength=A.n)
        rp = np.zeros(A.n + 1, dtype=np.int64)
        np.cumsum(cnt, out=rp[1:])
        B = ai.CSR(A.n, rp, (A.col[keep] - lo).astype(np.int32), A.val[keep], "M5 slab")
        mid = np.arange(8 * plane, 16 * plane)
        g = ai.rng("sample_rows", 9)
        sample = np.sort(g.choice(mid, size=SAMPLE["M5"], replace=False)).astype(np.int64)
        t0 = time.time()
        oracle.setup(B, k, s, eps, cap, rows=sample, threads=cores, trace=False)
        dt = time.time() - t0
        res[name] = {"T_p_s": dt * n / len(sample), "sample_rows": len(sample), "sample_s": dt, "cores": cores,
                     "kind": f"extrapolated from {len(sample)} interior rows of a 24-plane slab"}
        print(json.dumps({name: res[name]}), file=sys.stderr, flush=True)
        continue
    A = cfg["make"]()
    if name in SAMPLE:
        sample = ai.sample_rows(A.n, SAMPLE[name], sub=11)
        t0 = time.time()
        oracle.setup(A, k, s, eps, cap, rows=sample, threads=cores, trace=False)
        dt = time.time() - t0
        res[name] = {"T_p_s": dt * A.n / len(sample), "sample_rows": len(sample), "sample_s": dt, "cores": cores,
                     "kind": f"extrapolated from a seeded sample of {len(sample)} rows"}
    else:
        t0 = time.time()
        G, Gt, _ = oracle.setup_full(A, k, s, eps, cap, threads=cores)
        t1 = time.time()
        b, _ = ai.rhs_for(A)
        pr = oracle.pcg(A, G, Gt, b, tol=1e-8, max_iters=20000)
        t2 = time.time()
        # per-core rate: one thread on a sample
        smp = ai.sample_rows(A.n, min(A.n, 20000), sub=12)
        t3 = time.time()
        oracle.setup(A, k, s, eps, cap, rows=smp, threads=1, trace=False)
        t4 = time.time()
        res[name] = {"T_p_s": t1 - t0, "pcg_s": t2 - t1, "pcg_iters": pr.iters, "cores": cores, "kind": "full",
                     "one_core_rows_per_s": len(smp) / (t4 - t3)}
    print(json.dumps({name: res[name]}), file=sys.stderr, flush=True)
print(json.dumps(res, indent=1))
