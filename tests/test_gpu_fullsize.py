"""Parity at BASELINE.json's full sizes, in bench.py's launch configuration
(DESIGN.md §3.2): the GPU set-up of the whole matrix, checked on a seeded row
sample (plus the first and last rows) against the oracle row by row; on M2 (the
bench workload) also PCG iterations against the oracle's PCG and the explicit
residual.  Marked slow (minutes)."""
import numpy as np
import pytest
import torch

import afsai_inputs as ai
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def ctx():
    from paper_2010_14175_b200.api import Context
    c = Context()
    yield c
    c.close()


def sampled_parity(ctx, A, k, s, cap, nsample, sub):
    from paper_2010_14175_b200.api import DeviceCSR, Factor
    dA = DeviceCSR.from_numpy(A)
    F = Factor(ctx, dA, k, s, 0.0, cap)
    rp, ci, v = (t.cpu().numpy() for t in F.G())
    rows = ai.sample_rows(A.n, nsample, sub=sub)
    ref = oracle.setup(A, k, s, 0.0, cap, rows=rows)
    bad = []
    for t, i in enumerate(rows):
        c0, v0 = ref.row(t)
        a, b = rp[i], rp[i + 1]
        if not (np.array_equal(ci[a:b], c0) and np.array_equal(v[a:b].view(np.int64), v0.view(np.int64))):
            bad.append(int(i))
    assert not bad, f"{len(bad)} of {len(rows)} sampled rows differ: {bad[:10]}"
    st = F.stats()
    assert sum(st["rows_by_reason"]) == A.n
    return F, dA


def test_M2_full_size(ctx):
    cfg = ai.CONFIGS["M2"]
    A = cfg["make"]()
    F, dA = sampled_parity(ctx, A, cfg["nsteps"], cfg["s"], cfg["max_row_nnz"], 400, 1)
    b, _ = ai.rhs_for(A)
    x, rep = F.pcg(torch.from_numpy(b).cuda(), tol=1e-8)
    assert rep["converged"] and rep["true_rel_res"] <= 10 * 1e-8
    G, Gt, _ = oracle.setup_full(A, cfg["nsteps"], cfg["s"], 0.0, cfg["max_row_nnz"])
    pr = oracle.pcg(A, G, Gt, b, tol=1e-8)
    assert abs(rep["iters"] - pr.iters) <= 1, (rep["iters"], pr.iters)
    F.close()


def test_M4_full_size_sampled(ctx):
    cfg = ai.CONFIGS["M4"]
    A = cfg["make"]()
    F, dA = sampled_parity(ctx, A, cfg["nsteps"], cfg["s"], cfg["max_row_nnz"], 150, 2)
    F.close()


def test_M3_full_size_sampled(ctx):
    """M3 (8M rows, anisotropic coefficients): exercises the overflow-reason table
    sizing (256 table slots, 84 active slots) and its retries at full size."""
    cfg = ai.CONFIGS["M3"]
    A = cfg["make"]()
    F, dA = sampled_parity(ctx, A, cfg["nsteps"], cfg["s"], cfg["max_row_nnz"], 400, 3)
    st = F.stats()
    assert st["table_size"] >= 256
    F.close()
