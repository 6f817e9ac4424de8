"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY.md §8(c) "What pins each part", P1-P13).  No GPU; nothing here calls
the CUDA path.  Each pin is chosen so a plausible slip in the oracle (dropped
term, wrong sign, transposed operand, wrong index, missing sqrt) fails it.
"""
import json
import math
import os

import numpy as np
import pytest

import afsai_inputs as ai
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def dense_G(A, nsteps, s, eps=0.0, cap=1 << 30):
    G, Gt, res = oracle.setup_full(A, nsteps, s, eps, cap)
    return G.to_dense(), G, Gt, res


def kaporin(B):
    """Eq. 10: (tr(B)/n) / det(B)^(1/n), via a Cholesky log-determinant."""
    n = B.shape[0]
    L = np.linalg.cholesky(B)
    logdet = 2.0 * np.sum(np.log(np.diag(L)))
    return (np.trace(B) / n) / math.exp(logdet / n)


# ------------------------------------------------------------------ P1
@pytest.mark.parametrize("n,s", [(30, 1), (30, 30), (50, 3)])
def test_P1_full_pattern_is_inverse_cholesky(n, s):
    """kmax*s >= n on a dense SPD: the pattern fills the lower triangle and
    G = L^-1 with A = L L^T (LAPACK), G^T G = A^-1."""
    Ad = ai.random_spd_dense(n, sub=n)
    Gd, G, Gt, res = dense_G(ai.from_dense(Ad), nsteps=n, s=s)
    Linv = np.linalg.inv(np.linalg.cholesky(Ad))
    assert np.max(np.abs(Gd - Linv)) <= 1e-12 * np.max(np.abs(Linv))
    Ainv = np.linalg.inv(Ad)
    assert np.max(np.abs(Gd.T @ Gd - Ainv)) <= 1e-12 * np.max(np.abs(Ainv))
    assert np.linalg.norm(Gd @ Ad @ Gd.T - np.eye(n)) <= 1e-10
    assert np.all(res.nnz == np.arange(1, n + 1))


# ------------------------------------------------------------------ P2
def test_P2_tridiagonal_closed_forms():
    """tri(-1,2,-1): full-pattern g[i,j] = (j+1)/(i+1), psi_i = (i+2)/(i+1); with s = 1,
    kmax = k, rows i >= k get P = {i-1..i-k}, g[i,i-q] = (k+1-q)/(k+1), psi = (k+2)/(k+1);
    rows i < k reach the full pattern and stop with no candidates."""
    n, k = 64, 7
    A = ai.tridiag(n)
    res = oracle.setup(A, k, 1)
    for i in range(n):
        c, v = res.row(i)
        psi = res.psi[i, res.steps[i]]
        d = 1.0 / math.sqrt(psi)
        if i >= k:
            assert list(c) == list(range(i - k, i + 1))
            assert res.reason[i] == 0 and res.steps[i] == k
            expect_psi = (k + 2) / (k + 1)
            expect_g = {i - q: (k + 1 - q) / (k + 1) for q in range(1, k + 1)}
        else:
            assert list(c) == list(range(0, i + 1))
            assert res.reason[i] == (2 if i < k else 0)
            expect_psi = (i + 2) / (i + 1)
            expect_g = {j: (j + 1) / (i + 1) for j in range(i)}
        assert abs(psi - expect_psi) <= 1e-15 * 4
        assert abs(v[-1] - 1.0 / math.sqrt(expect_psi)) <= 1e-15 * 4
        for j, gj in expect_g.items():
            got = v[list(c).index(j)] / d
            assert abs(got - gj) <= 1e-14, (i, j, got, gj)
    # insertion order: P grows leftwards, one per step (psi strictly decreasing)
    assert np.all(np.diff(res.psi[k + 3, : k + 1]) < 0)


# ------------------------------------------------------------------ P3 (SPEC worked examples)
def test_P3_spec_2x2_example():
    g = GOLD["setup_2x2"]
    A = ai.from_dense(np.array(g["A"]))
    res = oracle.setup(A, g["nsteps"], g["s"])
    c0, v0 = res.row(0)
    c1, v1 = res.row(1)
    assert list(c0) == [0] and v0[0] == g["row0_d"]
    assert list(c1) == [0, 1]
    assert res.psi[1, 1] == g["row1_psi"]
    # 1/sqrt(2) as two correctly rounded operations (C9): within 1 ulp
    assert abs(v1[1] - g["row1_d"]) <= 2.0 ** -53
    assert v1[0] == g["row1_gt"] * v1[1]          # g~ * d, exact for g~ = -0.5


def test_P3_spec_gradient_examples():
    g = GOLD["gradient_tridiag_row2"]
    A = ai.tridiag(g["n"], g["diag"], g["off"])
    j, acc = oracle.gradient(A, g["row"], [], [])
    assert {str(int(a)): 2 * b for a, b in zip(j, acc)} == g["grad"]
    g = GOLD["gradient_identity_guess"]
    A = ai.from_dense(np.array(g["A"]))
    j, acc = oracle.gradient(A, g["row"], [], [])
    assert {str(int(a)): 2 * b for a, b in zip(j, acc)} == g["grad"]


def test_P3_spec_diagonal_scale():
    g = GOLD["diag_scale"]
    A = ai.diagonal(g["d"])
    res = oracle.setup(A, 5, 2)
    assert [res.row(i)[1][0] for i in range(2)] == g["G_diag"]
    assert list(res.reason) == [2, 2]  # diagonal A: no candidates


def test_P3_kaporin_examples():
    g = GOLD["kaporin"]
    assert abs(kaporin(np.diag([1.0, 4.0])) - g["diag_1_4"]) < 1e-15
    assert kaporin(np.eye(7)) == g["identity"]


def test_P3_notspd():
    g = GOLD["notspd_2x2"]
    with pytest.raises(oracle.OracleError) as e:
        oracle.setup(ai.from_dense(np.array(g["A"])), 3, 1)
    assert e.value.code == oracle.ENOTSPD
    assert (e.value.row, e.value.step) == (g["row"], g["step"])


# ------------------------------------------------------------------ P4
def test_P4_stencil_interior_rows():
    """Interior-row rationals derived by hand; with exact ties at
    step 1 the lowest column wins (R5)."""
    nx = 12
    A = ai.poisson2d(nx, nx)
    i = 5 * nx + 5
    r = oracle.setup(A, 3, 1, rows=[i])
    c, v = r.row(0)
    assert list(c - i) == [-nx - 1, -nx, -1, 0]
    d = v[-1]
    np.testing.assert_allclose(v[:3] / d, [1 / 7, 2 / 7, 2 / 7], rtol=0, atol=1e-15)
    assert abs(r.psi[0, 3] - 24 / 7) <= 2e-15 * 4
    nx = 8
    A = ai.poisson3d(nx)
    i = 4 * nx * nx + 4 * nx + 4
    r = oracle.setup(A, 3, 1, rows=[i])
    c, v = r.row(0)
    assert list(c - i) == [-nx * nx, -nx, -1, 0]
    np.testing.assert_allclose(v[:3] / v[-1], [1 / 6] * 3, rtol=0, atol=1e-15)
    assert abs(r.psi[0, 3] - 11 / 2) <= 1e-15 * 6
    r = oracle.setup(A, 2, 2, rows=[i])
    c, v = r.row(0)
    assert list(c - i) == [-nx * nx - nx, -nx * nx, -nx, -1, 0]
    np.testing.assert_allclose(v[:4] / v[-1], [1 / 17, 3 / 17, 3 / 17, 1 / 6], rtol=0, atol=1e-15)
    assert abs(r.psi[0, 2] - 559 / 102) <= 1e-15 * 6


# ------------------------------------------------------------------ P5, P6, P7
CASES = [
    ("poisson2d", lambda: ai.poisson2d(20, 20), 10, 1, 1 << 30),
    ("poisson3d", lambda: ai.poisson3d(9), 20, 2, 1 << 30),
    ("hetero", lambda: ai.hetero_poisson3d(8), 20, 2, 1 << 30),
    ("fe", lambda: ai.fe_elasticity(5), 30, 3, 100),
    ("rsparse", lambda: ai.random_sparse_spd(600, 8, sub=1), 8, 3, 20),
]


@pytest.mark.parametrize("name,make,k,s,cap", CASES, ids=[c[0] for c in CASES])
def test_P5_P6_P7_invariants(name, make, k, s, cap):
    A = make()
    Ad = A.to_dense()
    Gd, G, Gt, res = dense_G(A, k, s, cap=cap)
    # P5: psi non-increasing, bitwise (RN(psi - y^2) <= psi)
    for t in range(A.n):
        p = res.psi[t, : res.steps[t] + 1]
        assert np.all(np.diff(p) <= 0.0)
    # P6: unit diagonal of G A G^T (Eq. 8)
    GAGt = Gd @ Ad @ Gd.T
    assert np.max(np.abs(np.diag(GAGt) - 1.0)) <= 1e-12
    # P7: local optimality (Eq. 7): (G A)[i, j] = 0 for j in P-bar_i, row-relative
    GA = Gd @ Ad
    for i in range(A.n):
        c, _ = res.row(i)
        off = c[c != i]
        if len(off):
            scale = np.max(np.abs(Ad[i])) * np.max(np.abs(Gd[i]))
            assert np.max(np.abs(GA[i, off])) <= 1e-12 * scale * len(c)
    # cap respected, pattern strictly lower
    assert np.all(res.nnz <= cap)
    assert np.all(np.triu(Gd, 1) == 0.0)


# ------------------------------------------------------------------ P8
@pytest.mark.parametrize("sub", range(5))
def test_P8_gradient_finite_differences(sub):
    """Eq. 15 against central differences of psi(g) = g~^T A g~ (g~_i = 1), step 1e-6."""
    n = 40
    Ad = ai.random_spd_dense(n, sub=100 + sub)
    Ad[np.abs(Ad) < 0.05] = 0.0          # some structure
    A = ai.from_dense(Ad)
    i = n - 3
    rng = ai.rng("vectors", sub)
    P = rng.choice(i, size=6, replace=False)
    gt = rng.standard_normal(6)
    j, acc = oracle.gradient(A, i, P, gt)

    def psi(extra_j=None, h=0.0):
        g = np.zeros(n)
        g[i] = 1.0
        g[P] = gt
        if extra_j is not None:
            g[extra_j] += h
        return g @ Ad @ g

    h = 1e-6
    assert len(j) > 0
    for jj, a in zip(j, acc):
        fd = (psi(jj, h) - psi(jj, -h)) / (2 * h)
        assert abs(2 * a - fd) <= 1e-5 * max(1.0, abs(fd)), (jj, 2 * a, fd)
    # universe: exactly the j < i, j not in P, with some a_jr != 0 for r in P U {i}
    rows = list(P) + [i]
    expect = sorted(set(int(c) for r in rows for c in np.nonzero(Ad[r])[0] if c < i) - set(int(p) for p in P))
    assert list(j) == expect


# ------------------------------------------------------------------ P9
@pytest.mark.parametrize("name,make,k,s,cap", CASES[:4], ids=[c[0] for c in CASES[:4]])
def test_P9_brute_force_selection(name, make, k, s, cap):
    """Step-(k+1) selection = top-room of the dense |A g~| over j < i, j not in P
    (sort-based brute force).  Exact when the oracle's margin >= 1e-12; otherwise
    the chosen set must still be a valid top-room within 1e-12*max."""
    A = make()
    Ad = A.to_dense()
    kk = max(1, k // 2)
    r0 = oracle.setup(A, kk, s, max_row_nnz=cap)
    r1 = oracle.setup(A, kk + 1, s, max_row_nnz=cap)
    checked = 0
    for i in range(0, A.n, max(1, A.n // 150)):
        if r0.steps[i] != kk or r1.steps[i] != kk + 1:
            continue
        c0, v0 = r0.row(i)
        c1, _ = r1.row(i)
        d = v0[list(c0).index(i)]
        g = np.zeros(A.n)
        g[c0] = v0 / d                   # g~ with unit diagonal
        grad = Ad @ g
        new = sorted(set(c1) - set(c0))
        room = min(s, cap - 1 - (len(c0) - 1))
        cand = [j for j in range(i) if j not in set(c0) and grad[j] != 0.0
                and np.any(Ad[j, list(c0)] != 0.0)]
        order = sorted(cand, key=lambda j: (-abs(grad[j]), j))
        top = order[:room]
        margin = r1.margin[i, kk]
        if margin >= 1e-12:
            assert new == sorted(top), (i, new, top)
        else:
            mx = abs(grad[order[0]])
            thresh = abs(grad[top[-1]])
            assert all(abs(grad[j]) >= thresh - 1e-12 * mx for j in new)
        checked += 1
    assert checked > 5


# ------------------------------------------------------------------ P10
def test_P10_kaporin():
    n = 30
    Ad = ai.random_spd_dense(n, sub=7)
    A = ai.from_dense(Ad)
    D = np.diag(1.0 / np.sqrt(np.diag(Ad)))
    kj = kaporin(D @ Ad @ D)
    prev = np.inf
    for k in range(0, 7):
        Gd, G, Gt, res = dense_G(A, k, 2)
        B = Gd @ Ad @ Gd.T
        kap = kaporin(B)
        # Eq. 14: kappa = (prod psi_i / det A)^(1/n) with tr(GAG^T)/n = 1
        psis = np.array([res.psi[i, res.steps[i]] for i in range(n)])
        sign, logdet = np.linalg.slogdet(Ad)
        kap14 = math.exp((np.sum(np.log(psis)) - logdet) / n)
        assert abs(kap - kap14) <= 1e-12 * kap
        assert kap >= 1.0 - 1e-14
        assert kap <= prev + 1e-12           # non-increasing with kmax
        assert kap <= kj + 1e-10             # dominance over Jacobi
        if k == 0:
            assert abs(kap - kj) <= 1e-13
        prev = kap


# ------------------------------------------------------------------ P11
def test_P11_special_cases():
    A = ai.poisson2d(16, 16)
    d = np.array([A.val[A.rowptr[i]:A.rowptr[i + 1]][A.col[A.rowptr[i]:A.rowptr[i + 1]] == i][0] for i in range(A.n)])
    for k, cap in [(0, 100), (5, 1)]:
        res = oracle.setup(A, k, 2, max_row_nnz=cap)
        assert np.all(res.nnz == 1)
        assert np.array_equal(res.val[:, 0], 1.0 / np.sqrt(d))
        assert np.all(res.reason == (0 if k == 0 else 1))
    # diagonal A: G^T G r = A^-1 r
    dd = ai.rng("vectors", 9).uniform(0.5, 3.0, 50)
    Ad = ai.diagonal(dd)
    G, Gt, _ = oracle.setup_full(Ad, 4, 2)
    r = ai.rng("vectors", 10).standard_normal(50)
    np.testing.assert_allclose(oracle.apply(G, Gt, r), r / dd, rtol=2e-16 * 4)
    # row 0: G00 = a00^-1/2
    A = ai.random_sparse_spd(100, sub=3)
    res = oracle.setup(A, 5, 2, rows=[0])
    assert res.row(0)[1][0] == 1.0 / math.sqrt(A.val[A.rowptr[0] + list(A.col[A.rowptr[0]:A.rowptr[1]]).index(0)])


def test_tolerance_stop_path():
    """Eq. 16 with eps = 0.95 on Poisson 8^3: every row stops with 'tolerance' as soon as
    psi_k/psi_0 <= 0.95, never later (the survey's T1 case)."""
    A = ai.poisson3d(8)
    res = oracle.setup(A, 20, 2, eps=0.95)
    for i in range(A.n):
        st = res.steps[i]
        ratios = res.psi[i, 1: st + 1] / res.psi[i, 0]
        if res.reason[i] == 3:
            assert ratios[-1] <= 0.95 and np.all(ratios[:-1] > 0.95)
        else:
            assert np.all(ratios > 0.95)
    assert np.sum(res.reason == 3) > A.n // 2


# ------------------------------------------------------------------ P12
def test_P12_row_independence_and_halo():
    """Rows are independent: a row subset computed alone, from a copy of A in
    which every row outside [b - kmax*beta, e) is EMPTY, equals the full run bitwise
    (the exact-halo rule of DESIGN.md §6)."""
    A = ai.hetero_poisson3d(10)
    k, s = 6, 2
    full = oracle.setup(A, k, s)
    beta = A.bandwidth()
    b, e = 500, 800
    lo = max(0, b - k * beta)
    keep = np.zeros(A.n, dtype=bool)
    keep[lo:e] = True
    cnt = np.where(keep, np.diff(A.rowptr), 0)
    rp = np.zeros(A.n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rp[1:])
    m = np.repeat(keep, np.diff(A.rowptr))
    Ah = ai.CSR(A.n, rp, A.col[m], A.val[m])
    part = oracle.setup(Ah, k, s, rows=np.arange(b, e))
    assert np.array_equal(part.nnz, full.nnz[b:e])
    assert np.array_equal(part.col, full.col[b:e])
    assert np.array_equal(part.val.view(np.int64), full.val[b:e].view(np.int64))


# ------------------------------------------------------------------ transpose / apply
def test_transpose_and_apply_against_scipy_dense():
    A = ai.poisson3d(7)
    G, Gt, _ = oracle.setup_full(A, 8, 2)
    S = G.to_scipy()
    T = S.T.tocsr()
    T.sort_indices()
    assert np.array_equal(Gt.rowptr, T.indptr) and np.array_equal(Gt.col, T.indices)
    assert np.array_equal(Gt.val, T.data)
    r = ai.rng("vectors", 3).standard_normal(A.n)
    z = oracle.apply(G, Gt, r)
    Gd = G.to_dense()
    np.testing.assert_allclose(z, Gd.T @ (Gd @ r), rtol=1e-13, atol=1e-13 * np.max(np.abs(z)))


# ------------------------------------------------------------------ P13
def test_P13_pcg():
    g = GOLD["pcg_identity"]
    I = ai.diagonal(np.ones(20))
    b = ai.rng("vectors", 4).standard_normal(20)
    G, Gt, _ = oracle.setup_full(I, 3, 1)
    r = oracle.pcg(I, G, Gt, b)
    assert r.iters == g["iters"] and np.array_equal(r.x, b)
    g = GOLD["cg_diag3"]
    D = ai.diagonal(g["d"])
    r = oracle.pcg(D, None, None, np.array(g["b"]), tol=1e-12)
    assert r.iters <= g["max_iters"]
    np.testing.assert_allclose(r.x, g["x"], rtol=1e-12)
    # aFSAI beats Jacobi, solution matches a direct solve
    A = ai.poisson3d(16)
    b, xs = ai.rhs_for(A)
    G0, Gt0, _ = oracle.setup_full(A, 0, 1)
    Gf, Gtf, _ = oracle.setup_full(A, 20, 2)
    rj = oracle.pcg(A, G0, Gt0, b)
    rf = oracle.pcg(A, Gf, Gtf, b)
    assert rj.converged and rf.converged
    assert rf.iters <= 0.5 * rj.iters
    import scipy.sparse.linalg as spla
    xd = spla.spsolve(A.to_scipy().tocsc(), b)
    for r in (rj, rf):
        assert np.linalg.norm(r.x - xd) <= 1e-6 * np.linalg.norm(xd)
        assert np.linalg.norm(b - A.to_scipy() @ r.x) <= 10 * 1e-8 * np.linalg.norm(b)
    # the recurrence residual history is what it says
    assert rf.history[-1] <= 1e-8 < rf.history[-2]


def test_generators_are_bitwise_symmetric_spd():
    for A in [ai.poisson2d(6, 5), ai.poisson3d(4), ai.hetero_poisson3d(5), ai.fe_elasticity(3),
              ai.random_sparse_spd(80, sub=2)]:
        S = A.to_scipy()
        T = S.T.tocsr()
        T.sort_indices()
        assert np.array_equal(S.indptr, T.indptr) and np.array_equal(S.indices, T.indices)
        assert np.array_equal(S.data.view(np.int64), T.data.view(np.int64))
        assert np.linalg.eigvalsh(A.to_dense()).min() > 0
    A = ai.poisson3d(5)
    assert A.nnz == 7 * 125 - 6 * 25 and A.n == 125
    A = ai.fe_elasticity(4)
    assert A.n == 3 * 64


def test_fe_row_slabs_are_rows_of_the_full_matrix():
    """fe_elasticity_rows (multi-GPU slabs without the whole matrix) returns exactly
    the full generator's rows, bitwise, also for slabs that split a node's 3 rows."""
    N = 6
    A = ai.fe_elasticity(N)
    n = A.n
    for lo, hi in [(0, n), (0, 7), (5, n), (n // 3 + 1, 2 * n // 3 - 1), (n - 4, n)]:
        S = ai.fe_elasticity_rows(N, lo, hi)
        a, b = A.rowptr[lo], A.rowptr[hi]
        assert S.n == hi - lo and S.n_cols == n
        assert np.array_equal(S.rowptr, A.rowptr[lo:hi + 1] - a)
        assert np.array_equal(S.col, A.col[a:b])
        assert np.array_equal(S.val.view(np.int64), A.val[a:b].view(np.int64))


# ------------------------------------------------------------------ bounded communication
def test_bounded_setup_large_k_equals_full():
    """k >= n_p: every lower stripe is gathered, so each stripe's rows equal the
    whole-matrix set-up (row independence)."""
    A = ai.poisson3d(10)
    bounds = [0, 250, 500, 750, 1000]
    G = oracle.setup(A, 20, 2)
    for p in range(4):
        res, used = oracle.setup_bounded(A, bounds, p, 4, 20, 2)
        assert used == list(range(p + 1))
        for t, i in enumerate(range(bounds[p], bounds[p + 1])):
            c0, v0 = G.row(i)
            c1, v1 = res.row(t)
            assert np.array_equal(c0, c1) and np.array_equal(v0.view(np.int64), v1.view(np.int64))


def test_bounded_setup_k1_truncates():
    """Stripes of 2 planes and k = 1 on a 7-point grid: A-hat is tridiagonal, stripe p
    sees only p-1 and p; patterns stay inside I_p, rows near the lower boundary of
    I_p lose entries, and the local optimality (Eq. 7) holds on A[I_p, I_p]."""
    nx = 10
    A = ai.poisson3d(nx)
    bounds = [q * 2 * nx * nx for q in range(6)]
    H = oracle.comm_matrix(A, bounds)
    assert np.array_equal(H, np.eye(5, dtype=bool) | np.eye(5, k=1, dtype=bool) | np.eye(5, k=-1, dtype=bool))
    full = oracle.setup(A, 20, 2)
    res, used = oracle.setup_bounded(A, bounds, 3, 1, 20, 2)
    assert used == [2, 3]
    lo = bounds[2]
    differ = 0
    for t, i in enumerate(range(bounds[3], bounds[4])):
        c, v = res.row(t)
        assert c.min() >= lo
        c0, _ = full.row(i)
        differ += not np.array_equal(c, c0)
    assert differ > 0
    # rows near the top of the stripe reach at most 20 hops ~ 2 planes: some may still match
    assert res.reason.max() <= 2
