"""Oracle-only golden values for the full-size GPU tests (tests/golden/pcg_iters.json).

For each named BASELINE.json config this runs ONLY the CPU oracle (oracle/,
DESIGN.md §3.1 contract) on the seeded input of afsai_inputs: the full aFSAI
set-up, its transpose, and the oracle PCG (x0 = 0, ||r||/||b|| <= 1e-8,
P:1091-1092; R12) on b = A x*.  Nothing here touches the CUDA path.
The GPU test asserts its PCG iteration count within +-1 of the stored count
(BASELINE.json north_star) and nnz(G) equal.

usage: python scripts/oracle_goldens.py M3 M4 [--out tests/golden/pcg_iters.json]
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import afsai_inputs as ai  # noqa: E402
import oracle  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = os.path.join(ROOT, "tests", "golden", "pcg_iters.json")
    for a in sys.argv[1:]:
        if a.startswith("--out="):
            out = a.split("=", 1)[1]
    doc = json.load(open(out)) if os.path.exists(out) else {}
    cores = os.cpu_count() or 1
    for name in args or ["M3", "M4"]:
        cfg = ai.CONFIGS[name]
        t0 = time.time()
        A = cfg["make"]()
        k, s, eps, cap = cfg["nsteps"], cfg["s"], cfg["eps"], cfg["max_row_nnz"]
        t1 = time.time()
        G, Gt, res = oracle.setup_full(A, k, s, eps, cap, threads=cores)
        t2 = time.time()
        b, _ = ai.rhs_for(A)
        pr = oracle.pcg(A, G, Gt, b, tol=1e-8, max_iters=20000)
        t3 = time.time()
        h = hashlib.sha256()
        h.update(G.rowptr.tobytes())
        h.update(G.col.tobytes())
        h.update(G.val.tobytes())
        doc[name] = {"desc": cfg["desc"], "n": int(A.n), "nnz_A": int(A.nnz), "params": [k, s, eps, cap],
                     "nnz_G": int(G.nnz), "G_sha256": h.hexdigest(), "pcg_tol": 1e-8,
                     "pcg_iters": int(pr.iters), "pcg_relres": float(pr.relres), "pcg_converged": bool(pr.converged),
                     "stop_reasons": np.bincount(res.reason, minlength=4).tolist(),
                     "how": f"oracle.setup_full + oracle.pcg, {cores} threads; gen {t1 - t0:.0f} s, "
                            f"set-up {t2 - t1:.0f} s, PCG {t3 - t2:.0f} s",
                     "source": "scripts/oracle_goldens.py (calls only oracle/ and afsai_inputs/)"}
        print(json.dumps({name: doc[name]}), flush=True)
        del A, G, Gt, res
        with open(out, "w") as f:
            json.dump(doc, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
