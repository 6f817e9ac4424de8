"""Parity at BASELINE.json's full sizes, in bench.py's launch configuration
(whole-matrix afsai_setup on one GPU), against the CPU oracle:

- M2 (configs[1]): EVERY row of G bitwise against the oracle's full set-up, and
  the PCG iteration count within 1 of the oracle's PCG.
- M3 (configs[2]), M4 (configs[3]): a seeded row sample plus EVERY row the set-up
  recomputed in a retry pass (its on-chip tables overflowed), bitwise; PCG
  iterations within 1 of the oracle count stored in tests/golden/pcg_iters.json
  (written by scripts/oracle_goldens.py, which runs only oracle/).
- M5 (configs[4], ~1B nnz): 2000 seeded rows, the 256 rows on each side of every
  partition boundary of the 2-, 4- and 8-GPU splits, and every retried row,
  bitwise.  Row independence makes a row's result a function of A
  alone, so sampled rows of the whole-matrix run are the rows a multi-GPU run
  computes.
Marked slow (minutes each)."""
import json
import os

import numpy as np
import pytest
import torch

import afsai_inputs as ai
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pcg_iters.json")


@pytest.fixture(scope="module")
def ctx():
    from paper_2010_14175_b200.api import Context
    c = Context()
    yield c
    c.close()


def check_rows(rp, ci, v, ref, rows):
    bad = []
    for t, i in enumerate(rows):
        c0, v0 = ref.row(t)
        a, b = rp[i], rp[i + 1]
        if not (np.array_equal(ci[a:b], c0) and np.array_equal(v[a:b].view(np.int64), v0.view(np.int64))):
            bad.append(int(i))
    return bad


def sampled_parity(ctx, A, cfg, nsample, sub, extra_rows=()):
    from paper_2010_14175_b200.api import DeviceCSR, Factor
    k, s, cap = cfg["nsteps"], cfg["s"], cfg["max_row_nnz"]
    dA = DeviceCSR.from_numpy(A)
    F = Factor(ctx, dA, k, s, 0.0, cap)
    rp, ci, v = (t.cpu().numpy() for t in F.G())
    retried = F.retried_rows()
    rows = np.unique(np.concatenate([ai.sample_rows(A.n, nsample, sub=sub), retried,
                                     np.asarray(extra_rows, dtype=np.int64)])).astype(np.int64)
    ref = oracle.setup(A, k, s, 0.0, cap, rows=rows, trace=False)
    bad = check_rows(rp, ci, v, ref, rows)
    assert not bad, f"{len(bad)} of {len(rows)} checked rows differ (retried: {len(retried)}): {bad[:10]}"
    st = F.stats()
    assert sum(st["rows_by_reason"]) == A.n
    assert st["retried_rows"] >= len(retried)
    return F, dA, retried, len(rows)


def golden(name):
    doc = json.load(open(GOLDEN))
    if name not in doc:
        pytest.fail(f"no oracle golden for {name}: run scripts/oracle_goldens.py {name}")
    return doc[name]


def pcg_vs_golden(F, A, name):
    g = golden(name)
    assert F.nnz[0] == g["nnz_G"], (F.nnz[0], g["nnz_G"])
    b, _ = ai.rhs_for(A)
    x, rep = F.pcg(torch.from_numpy(b).cuda(), tol=1e-8, max_iters=20000)
    assert rep["converged"] and rep["true_rel_res"] <= 10 * 1e-8
    assert abs(rep["iters"] - g["pcg_iters"]) <= 1, (rep["iters"], g["pcg_iters"])


def test_M2_full_size(ctx):
    """Every one of the 10^6 rows bitwise, plus PCG iterations against the oracle PCG."""
    from paper_2010_14175_b200.api import DeviceCSR, Factor
    cfg = ai.CONFIGS["M2"]
    A = cfg["make"]()
    k, s, cap = cfg["nsteps"], cfg["s"], cfg["max_row_nnz"]
    F = Factor(ctx, DeviceCSR.from_numpy(A), k, s, 0.0, cap)
    rp, ci, v = (t.cpu().numpy() for t in F.G())
    G, Gt, res = oracle.setup_full(A, k, s, 0.0, cap)
    assert np.array_equal(rp, G.rowptr)
    assert np.array_equal(ci, G.col)
    assert np.array_equal(v.view(np.int64), G.val.view(np.int64))
    st, rs = F.trace()
    assert np.array_equal(st.cpu().numpy(), res.steps) and np.array_equal(rs.cpu().numpy(), res.reason)
    b, _ = ai.rhs_for(A)
    x, rep = F.pcg(torch.from_numpy(b).cuda(), tol=1e-8)
    assert rep["converged"] and rep["true_rel_res"] <= 10 * 1e-8
    pr = oracle.pcg(A, G, Gt, b, tol=1e-8)
    assert abs(rep["iters"] - pr.iters) <= 1, (rep["iters"], pr.iters)
    F.close()


def test_M3_full_size(ctx):
    """M3 (8M rows, anisotropic coefficients): the overflow-reason table sizing and
    every row its retry passes recomputed; PCG iterations against the oracle golden."""
    cfg = ai.CONFIGS["M3"]
    A = cfg["make"]()
    F, dA, retried, nchk = sampled_parity(ctx, A, cfg, 400, 3)
    assert F.stats()["table_size"] >= 256
    assert len(retried) > 0, "M3 is expected to exercise the retry path"
    pcg_vs_golden(F, A, "M3")
    F.close()


def test_M3_full_size_fp32(ctx):
    """The single-precision set-up at full size: seeded rows and every retried
    row bitwise against the fp32 oracle; PCG iterations within 1.2x of the fp64 golden."""
    from paper_2010_14175_b200.api import DeviceCSR, Factor
    cfg = ai.CONFIGS["M3"]
    A = cfg["make"]()
    k, s, cap = cfg["nsteps"], cfg["s"], cfg["max_row_nnz"]
    F = Factor(ctx, DeviceCSR.from_numpy(A), k, s, 0.0, cap, precision="fp32")
    rp, ci, v = (t.cpu().numpy() for t in F.G())
    rows = np.unique(np.concatenate([ai.sample_rows(A.n, 400, sub=11), F.retried_rows()])).astype(np.int64)
    ref = oracle.setup(A, k, s, 0.0, cap, rows=rows, trace=False, precision="fp32")
    bad = check_rows(rp, ci, v, ref, rows)
    assert not bad, f"{len(bad)} of {len(rows)} rows differ: {bad[:10]}"
    b, _ = ai.rhs_for(A)
    x, rep = F.pcg(torch.from_numpy(b).cuda(), tol=1e-8, max_iters=20000)
    assert rep["converged"] and rep["iters"] <= int(np.ceil(1.2 * golden("M3")["pcg_iters"]))
    F.close()


def test_M4_full_size(ctx):
    cfg = ai.CONFIGS["M4"]
    A = cfg["make"]()
    F, dA, retried, nchk = sampled_parity(ctx, A, cfg, 300, 2)
    pcg_vs_golden(F, A, "M4")
    F.close()


def test_M5_full_size(ctx):
    """The largest config (12.06M rows, 0.96B nnz): 2000 seeded rows, both sides of
    every 2/4/8-GPU partition boundary, and every retried row."""
    cfg = ai.CONFIGS["M5"]
    A = cfg["make"]()
    n = A.n
    bnd = sorted({n * q // w for w in (2, 4, 8) for q in range(1, w)})
    extra = np.concatenate([np.arange(max(0, b - 256), min(n, b + 256)) for b in bnd])
    F, dA, retried, nchk = sampled_parity(ctx, A, cfg, 2000, 9, extra)
    assert nchk >= 2000 + len(extra) // 2
    F.close()
