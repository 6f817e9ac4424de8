"""GPU vs oracle parity through the C ABI.

Set-up: patterns identical and G within 1e-10 row-relative (BASELINE.json
north_star); under the arithmetic contract C1-C12 we also expect, and assert,
bitwise equality.  Trace (steps, stop reasons) equal.  G^T bitwise.  Apply
within the SpMV rounding bound.  PCG iterations within +-1.
"""
import numpy as np
import pytest
import torch

import afsai_inputs as ai
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.fail("no GPU")
    from paper_2010_14175_b200.api import Context
    c = Context()
    yield c
    c.close()


def gpu_setup(ctx, A, nsteps, s, eps=0.0, cap=1 << 30, precision="fp64"):
    from paper_2010_14175_b200.api import DeviceCSR, Factor
    F = Factor(ctx, DeviceCSR.from_numpy(A), nsteps, s, eps, cap, precision=precision)
    return F


def host_csr(F, which=0):
    rp, ci, v = F.G() if which == 0 else F.Gt()
    return ai.CSR(rp.numel() - 1, rp.cpu().numpy(), ci.cpu().numpy(), v.cpu().numpy())


def compare_rows(Gg, ref, rows, label):
    """Per-row parity: pattern identical (else flagged iff the oracle margin < 1e-12),
    values row-relative <= 1e-10, plus a count of non-bitwise rows."""
    failed, flagged, nonbit = [], [], 0
    for t, i in enumerate(rows):
        c0, v0 = ref.row(t)
        a, b = Gg.rowptr[i], Gg.rowptr[i + 1]
        c1, v1 = Gg.col[a:b], Gg.val[a:b]
        if len(c0) != len(c1) or not np.array_equal(c0, c1):
            mg = ref.margin[t, : max(1, ref.steps[t])]
            if np.nanmin(mg) < 1e-12:
                flagged.append(int(i))
            else:
                failed.append(int(i))
            continue
        rel = np.max(np.abs(v1 - v0)) / np.max(np.abs(v0))
        if rel > 1e-10:
            failed.append(int(i))
        if not np.array_equal(v0.view(np.int64), v1.view(np.int64)):
            nonbit += 1
    assert not failed, f"{label}: {len(failed)} rows fail parity, first {failed[:10]}"
    return flagged, nonbit


CASES = [
    ("M1_poisson2d_32", lambda: ai.poisson2d(32, 32), 10, 1, 0.0, 1 << 30),
    ("poisson3d_12_20x2", lambda: ai.poisson3d(12), 20, 2, 0.0, 1 << 30),
    ("hetero_10_20x2", lambda: ai.hetero_poisson3d(10), 20, 2, 0.0, 1 << 30),
    ("fe_5_30x3_cap100", lambda: ai.fe_elasticity(5), 30, 3, 0.0, 100),
    ("rsparse_cap12_s5", lambda: ai.random_sparse_spd(3000, 10, sub=4), 6, 5, 0.0, 12),
    ("rsparse_banded_s8", lambda: ai.random_sparse_spd(2000, 6, sub=5, bandwidth=40), 8, 8, 0.0, 1 << 30),
    ("poisson3d_8_eps095", lambda: ai.poisson3d(8), 20, 2, 0.95, 1 << 30),
    ("poisson2d_kmax0", lambda: ai.poisson2d(9, 7), 0, 1, 0.0, 1 << 30),
    ("tridiag_64_k7", lambda: ai.tridiag(64), 7, 1, 0.0, 1 << 30),
    ("dense50_full", lambda: ai.from_dense(ai.random_spd_dense(50, sub=50)), 50, 1, 0.0, 1 << 30),
    ("dense90_s16", lambda: ai.from_dense(ai.random_spd_dense(90, sub=90)), 8, 16, 0.0, 1 << 30),
    ("dense130_cap129", lambda: ai.from_dense(ai.random_spd_dense(130, sub=130)), 200, 1, 0.0, 129),
    ("single_row", lambda: ai.diagonal([3.0]), 5, 2, 0.0, 1 << 30),
    # pattern-row kernel instances (long rows, s <= 4) and the hit-list table probe
    ("fe_4_12x1", lambda: ai.fe_elasticity(4), 12, 1, 0.0, 100),
    ("fe_4_10x2_cap15", lambda: ai.fe_elasticity(4), 10, 2, 0.0, 15),
    ("rsparse_s4", lambda: ai.random_sparse_spd(3000, 10, sub=6), 8, 4, 0.0, 1 << 30),
    ("hetero_32_probe", lambda: ai.hetero_poisson3d(32), 20, 2, 0.0, 1 << 30),
    # s > 4 on a stencil: the hit-list kernel that is not in lockstep
    ("poisson3d_8_s5", lambda: ai.poisson3d(8), 4, 5, 0.0, 1 << 30),
    # hub column: G^T row 0 is ~n long (the long-row transpose sort, > 1024 entries)
    ("arrow_3000_12x3", lambda: ai.arrow_spd(3000), 12, 3, 0.0, 1 << 30),
]


# the kernel plan each case must exercise (afsai_setup_stats_t.plan)
PLAN = {"M1_poisson2d_32": 0, "poisson3d_12_20x2": 0, "hetero_10_20x2": 0, "fe_5_30x3_cap100": 1,
        "rsparse_cap12_s5": 3, "poisson3d_8_s5": 2, "fe_4_12x1": 1}


@pytest.mark.parametrize("name,make,k,s,eps,cap", CASES, ids=[c[0] for c in CASES])
def test_setup_parity(ctx, name, make, k, s, eps, cap):
    A = make()
    F = gpu_setup(ctx, A, k, s, eps, cap)
    G = host_csr(F)
    ref = oracle.setup(A, k, s, eps, cap)
    rows = np.arange(A.n)
    flagged, nonbit = compare_rows(G, ref, rows, name)
    assert not flagged, f"{name}: flagged rows under the contract: {flagged[:10]}"
    assert nonbit == 0, f"{name}: {nonbit} rows not bitwise equal"
    Gr = ref.to_csr(A.n)
    assert np.array_equal(G.rowptr, Gr.rowptr)
    st, rs = F.trace()
    assert np.array_equal(st.cpu().numpy(), ref.steps)
    assert np.array_equal(rs.cpu().numpy(), ref.reason)
    stats = F.stats()
    if name in PLAN:
        assert stats["plan"] == PLAN[name], (name, stats["plan"])
    assert stats["nnz_G"] == Gr.nnz
    assert sum(stats["rows_by_reason"]) == A.n
    # transpose: exact, rows ascending (C10)
    T = host_csr(F, 1)
    Tr = oracle.transpose(Gr)
    assert np.array_equal(T.rowptr, Tr.rowptr) and np.array_equal(T.col, Tr.col)
    assert np.array_equal(T.val.view(np.int64), Tr.val.view(np.int64))
    if name.startswith("arrow"):
        assert np.diff(T.rowptr).max() > 2048, "the long-row transpose path was not exercised"
    F.close()


@pytest.mark.parametrize("name,make,k,s,eps,cap", CASES, ids=[c[0] for c in CASES])
def test_setup_parity_fp32(ctx, name, make, k, s, eps, cap):
    """The single-precision set-up (afsai::sp kernels) against the fp32
    oracle: bitwise G (= double(G_s)), identical trace, G^T bitwise."""
    A = make()
    F = gpu_setup(ctx, A, k, s, eps, cap, precision="fp32")
    G = host_csr(F)
    ref = oracle.setup(A, k, s, eps, cap, precision="fp32")
    Gr = ref.to_csr(A.n)
    assert np.array_equal(G.rowptr, Gr.rowptr) and np.array_equal(G.col, Gr.col)
    assert np.array_equal(G.val.view(np.int64), Gr.val.view(np.int64)), name
    st, rs = F.trace()
    assert np.array_equal(st.cpu().numpy(), ref.steps) and np.array_equal(rs.cpu().numpy(), ref.reason)
    assert F.stats()["value_bytes"] == 4
    T = host_csr(F, 1)
    Tr = oracle.transpose(Gr)
    assert np.array_equal(T.col, Tr.col) and np.array_equal(T.val.view(np.int64), Tr.val.view(np.int64))
    F.close()


@pytest.mark.parametrize("env", [{"AFSAI_TABLE": "64"}, {"AFSAI_PROW": "0"}, {"AFSAI_HITS": "0"}],
                         ids=["retry_from_64", "scan_kernel_fe", "scan_kernel_stencil"])
def test_setup_parity_fp32_plans(ctx, env, monkeypatch):
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    for A, k, s, cap in [(ai.fe_elasticity(4), 30, 3, 100), (ai.hetero_poisson3d(12), 20, 2, 1 << 30)]:
        F = gpu_setup(ctx, A, k, s, 0.0, cap, precision="fp32")
        G = host_csr(F)
        Gr = oracle.setup(A, k, s, 0.0, cap, precision="fp32").to_csr(A.n)
        assert np.array_equal(G.col, Gr.col) and np.array_equal(G.val.view(np.int64), Gr.val.view(np.int64))
        F.close()


@pytest.mark.parametrize("make,k,s,cap", [(lambda: ai.poisson3d(16), 20, 2, 1 << 30),
                                          (lambda: ai.hetero_poisson3d(12), 20, 2, 1 << 30),
                                          (lambda: ai.fe_elasticity(6), 30, 3, 100)])
def test_pcg_fp32_setup(ctx, make, k, s, cap):
    """PCG with the fp32-set-up G needs <= 1.2x the iterations of the fp64 G,
    and its count is within 1 of the oracle PCG on the fp32 oracle's G."""
    A = make()
    b, _ = ai.rhs_for(A)
    bd = torch.from_numpy(b).cuda()
    F64 = gpu_setup(ctx, A, k, s, 0.0, cap)
    F32 = gpu_setup(ctx, A, k, s, 0.0, cap, precision="fp32")
    _, r64 = F64.pcg(bd, tol=1e-8, max_iters=5000)
    _, r32 = F32.pcg(bd, tol=1e-8, max_iters=5000)
    assert r64["converged"] and r32["converged"]
    assert r32["iters"] <= int(np.ceil(1.2 * r64["iters"])), (r32["iters"], r64["iters"])
    G, Gt, _ = oracle.setup_full(A, k, s, 0.0, cap, precision="fp32")
    pr = oracle.pcg(A, G, Gt, b, tol=1e-8, max_iters=5000)
    assert abs(r32["iters"] - pr.iters) <= 1
    F64.close()
    F32.close()


@pytest.mark.parametrize("env", [{"AFSAI_TABLE": "64"}, {"AFSAI_PROW": "0"}, {"AFSAI_NOPROBE": "1"},
                                 {"AFSAI_TRANSPOSE": "radix"}],
                         ids=["prow_retry_from_64", "scan_kernel", "hits_no_probe", "radix_transpose"])
def test_setup_parity_plans(ctx, env, monkeypatch):
    """The other kernel plans (forced small tables and retries, the general scan
    kernel on FE rows, the hit-list kernel without the table probe) give the
    same bits as the oracle."""
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    cases = [(ai.fe_elasticity(4), 30, 3, 100)]
    if "AFSAI_TRANSPOSE" in env:   # G^T by the stable radix sort, checked bitwise against oracle.transpose
        cases = [(ai.fe_elasticity(4), 30, 3, 100), (ai.arrow_spd(3000), 12, 3, 1 << 30),
                 (ai.hetero_poisson3d(24), 20, 2, 1 << 30)]
    if "AFSAI_NOPROBE" in env:
        cases = [(ai.hetero_poisson3d(32), 20, 2, 1 << 30)]
    for A, k, s, cap in cases:
        F = gpu_setup(ctx, A, k, s, 0.0, cap)
        G = host_csr(F)
        ref = oracle.setup(A, k, s, 0.0, cap)
        flagged, nonbit = compare_rows(G, ref, np.arange(A.n), str(env))
        assert not flagged and nonbit == 0
        T, Tr = host_csr(F, 1), oracle.transpose(ref.to_csr(A.n))
        assert np.array_equal(T.rowptr, Tr.rowptr) and np.array_equal(T.col, Tr.col)
        assert np.array_equal(T.val.view(np.int64), Tr.val.view(np.int64))
        if "AFSAI_TABLE" in env:
            assert F.stats()["retried_rows"] > 0
        F.close()


def apply_tolerance(G, Gt, r):
    """|dz| <= gamma * G^T(|G||r|) (+ same for the inner product), u = 2^-53, gamma ~ 64u:
    the standard SpMV rounding bound with a factor covering row lengths <= ~60."""
    u = 2.0 ** -53
    Ga, Gta = abs(G.to_scipy()), abs(Gt.to_scipy())
    inner = Ga @ np.abs(r)
    return 2 * 64 * u * (Gta @ inner) + 1e-300


@pytest.mark.parametrize("make,k,s", [(lambda: ai.poisson3d(16), 20, 2), (lambda: ai.fe_elasticity(5), 30, 3)])
def test_apply_parity(ctx, make, k, s):
    A = make()
    F = gpu_setup(ctx, A, k, s, 0.0, 100)
    G, Gt = host_csr(F), host_csr(F, 1)
    r = ai.rng("vectors", 11).standard_normal(A.n)
    z_ref = oracle.apply(G, Gt, r)
    z = F.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    tol = apply_tolerance(G, Gt, r)
    assert np.all(np.abs(z - z_ref) <= tol), np.max(np.abs(z - z_ref) / tol)
    # host buffers through the same C call (staged inside the library)
    zh = torch.empty(A.n, dtype=torch.float64)
    F.apply(torch.from_numpy(r), zh)
    assert np.array_equal(zh.numpy(), z)
    # preconditioner symmetry (u, M v) = (M u, v)
    v = ai.rng("vectors", 12).standard_normal(A.n)
    Mv = F.apply(torch.from_numpy(v).cuda()).cpu().numpy()
    assert abs(r @ Mv - z @ v) <= 1e-12 * abs(r @ Mv)
    F.close()


@pytest.mark.parametrize("make,k,s,cap", [
    (lambda: ai.poisson3d(16), 20, 2, 1 << 30),
    (lambda: ai.poisson3d(16), 0, 1, 1 << 30),        # Jacobi (kmax = 0, P11)
    (lambda: ai.hetero_poisson3d(12), 20, 2, 1 << 30),
    (lambda: ai.fe_elasticity(6), 30, 3, 100),
])
def test_pcg_parity(ctx, make, k, s, cap):
    A = make()
    b, xs = ai.rhs_for(A)
    F = gpu_setup(ctx, A, k, s, 0.0, cap)
    x, rep = F.pcg(torch.from_numpy(b).cuda(), tol=1e-8, max_iters=5000)
    G, Gt, _ = oracle.setup_full(A, k, s, 0.0, cap)
    pr = oracle.pcg(A, G, Gt, b, tol=1e-8, max_iters=5000)
    assert rep["converged"] and pr.converged
    assert abs(rep["iters"] - pr.iters) <= 1, (rep["iters"], pr.iters)
    assert rep["true_rel_res"] <= 10 * 1e-8
    xg = x.cpu().numpy()
    assert np.linalg.norm(xg - pr.x) <= 1e-6 * np.linalg.norm(pr.x)
    F.close()


@pytest.mark.parametrize("make,k,s,cap", [(lambda: ai.poisson3d(16), 20, 2, 1 << 30),
                                          (lambda: ai.hetero_poisson3d(12), 20, 2, 1 << 30),
                                          (lambda: ai.fe_elasticity(6), 30, 3, 100)])
def test_pcg_single_pass_apply(ctx, make, k, s, cap, monkeypatch):
    """AFSAI_APPLY=single: M^-1 r in one pass over G with fp64 reductions (non-deterministic
    summation order): PCG iterations within 1 of the oracle, solution to 1e-6."""
    monkeypatch.setenv("AFSAI_APPLY", "single")
    A = make()
    b, xs = ai.rhs_for(A)
    F = gpu_setup(ctx, A, k, s, 0.0, cap)
    x, rep = F.pcg(torch.from_numpy(b).cuda(), tol=1e-8, max_iters=5000)
    G, Gt, _ = oracle.setup_full(A, k, s, 0.0, cap)
    pr = oracle.pcg(A, G, Gt, b, tol=1e-8, max_iters=5000)
    assert rep["converged"] and abs(rep["iters"] - pr.iters) <= 1, (rep["iters"], pr.iters)
    assert rep["true_rel_res"] <= 10 * 1e-8
    assert np.linalg.norm(x.cpu().numpy() - pr.x) <= 1e-6 * np.linalg.norm(pr.x)
    F.close()


def test_pcg_identity_and_host_buffers(ctx):
    I = ai.diagonal(np.ones(100))
    b = ai.rng("vectors", 13).standard_normal(100)
    F = gpu_setup(ctx, I, 3, 1)
    xh = torch.empty(100, dtype=torch.float64)
    x, rep = F.pcg(torch.from_numpy(b), tol=1e-8, x=xh)   # host b and x
    assert rep["iters"] == 1 and np.allclose(xh.numpy(), b, rtol=0, atol=1e-15)
    F.close()


def test_errors(ctx):
    from paper_2010_14175_b200 import capi
    # not SPD: [[1,2],[2,1]] -> ENOTSPD at row 1, step 1 (same as the oracle)
    A = ai.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(capi.AfsaiError) as e:
        gpu_setup(ctx, A, 3, 1)
    assert e.value.code == capi.AFSAI_ENOTSPD and (e.value.row, e.value.step) == (1, 1)
    # invalid: unsorted columns
    B = ai.poisson2d(4, 4)
    col = B.col.copy()
    col[1], col[2] = col[2], col[1]
    with pytest.raises(capi.AfsaiError) as e:
        gpu_setup(ctx, ai.CSR(B.n, B.rowptr, col, B.val), 2, 1)
    assert e.value.code == capi.AFSAI_EINVAL
    # not bitwise symmetric (contract C1): one off-diagonal value moved by one ulp
    val = B.val.copy()
    e01 = B.rowptr[0] + 1   # entry (0, 1); (1, 0) keeps the old bits
    val[e01] = np.nextafter(val[e01], 0.0)
    with pytest.raises(capi.AfsaiError) as e:
        gpu_setup(ctx, ai.CSR(B.n, B.rowptr, B.col, val), 2, 1)
    assert e.value.code == capi.AFSAI_EINVAL and "symmetric" in str(e.value)
    # invalid params
    with pytest.raises(capi.AfsaiError) as e:
        gpu_setup(ctx, B, 2, 0)
    assert e.value.code == capi.AFSAI_EINVAL
    with pytest.raises(capi.AfsaiError) as e:
        gpu_setup(ctx, B, 200, 2)   # mmax 400 > 128
    assert e.value.code == capi.AFSAI_ELIMIT
    # the context still works after errors
    F = gpu_setup(ctx, B, 2, 1)
    F.close()


def test_host_csr_input(ctx):
    """afsai_setup with HOST arrays (staged by the library) gives the same G."""
    from paper_2010_14175_b200.api import DeviceCSR, Factor
    A = ai.poisson3d(10)
    Fh = Factor(ctx, DeviceCSR.from_numpy(A, device="cpu"), 20, 2)
    Fd = Factor(ctx, DeviceCSR.from_numpy(A), 20, 2)
    for a, b in zip(Fh.G(), Fd.G()):
        assert torch.equal(a, b)


def test_determinism_repeat(ctx):
    A = ai.hetero_poisson3d(12)
    G1 = [t.cpu() for t in gpu_setup(ctx, A, 20, 2).G()]
    G2 = [t.cpu() for t in gpu_setup(ctx, A, 20, 2).G()]
    for a, b in zip(G1, G2):
        assert torch.equal(a, b)


@pytest.mark.parametrize("make,k,s,cap", [(lambda: ai.hetero_poisson3d(12), 8, 2, 1 << 30),
                                          (lambda: ai.fe_elasticity(6), 10, 3, 100),
                                          (lambda: ai.poisson3d(14), 20, 2, 1 << 30)])
@pytest.mark.parametrize("env", [{}, {"AFSAI_PROW": "0", "AFSAI_HITS": "0"}], ids=["default", "scan_kernel"])
def test_block_setup_partition_emulation(ctx, make, k, s, cap, env, monkeypatch):
    """Rows of a block computed from a halo-extended copy of A (rows [b - k*beta, e)
    only) are bitwise the oracle's rows of the whole matrix (pin P12 on the GPU:
    the multi-GPU set-up's building block).  Also with the general
    scan kernel, whose last-step universe reaches one hop past the halo."""
    from paper_2010_14175_b200 import capi
    from paper_2010_14175_b200.api import DeviceCSR
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    A = make()
    G = oracle.setup(A, k, s, 0.0, cap, trace=False).to_csr(A.n)   # the reference is the oracle
    beta = A.bandwidth()
    n = A.n
    for b, e in [(0, n // 3), (n // 3, 2 * n // 3), (2 * n // 3, n)]:
        lo = max(0, b - k * beta)
        X = DeviceCSR.from_numpy(A, row_begin=lo, n_rows=e - lo)
        h = capi.afsai_setup_block(ctx.h, X.c(), b, e - b, k, s, 0.0, min(cap, 2**31 - 1))
        nnz, _ = capi.afsai_factor_nnz(h)
        rp = torch.empty(e - b + 1, dtype=torch.int64, device="cuda")
        ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
        v = torch.empty(nnz, dtype=torch.float64, device="cuda")
        capi.afsai_factor_copy(h, 0, rp, ci, v)
        # a block factor has no G^T: apply must refuse it (no illegal-address fault)
        rr = torch.zeros(e - b, dtype=torch.float64, device="cuda")
        with pytest.raises(capi.AfsaiError) as ex:
            capi.afsai_apply(ctx.h, h, rr, torch.empty_like(rr))
        assert ex.value.code == capi.AFSAI_EINVAL
        capi.afsai_factor_destroy(h)
        a0, a1 = G.rowptr[b], G.rowptr[e]
        assert np.array_equal(rp.cpu().numpy(), G.rowptr[b:e + 1] - a0)
        assert np.array_equal(ci.cpu().numpy(), G.col[a0:a1])
        assert np.array_equal(v.cpu().numpy().view(np.int64), G.val[a0:a1].view(np.int64))
