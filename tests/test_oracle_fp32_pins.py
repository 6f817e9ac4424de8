"""Pins of the SINGLE-PRECISION set-up oracle (§4.3: the
set-up may run in fp32 on A_s = single(A); G = double(G_s)), against what the
mathematics fixes at fp32 accuracy.  No GPU.  u32 = 2^-24.

- P1/32 full pattern: G = L^-1 (LAPACK on the fp64 A) within fp32 rounding.
- P2/32 tridiagonal closed forms within fp32 rounding.
- P4/32 stencil interior rationals within fp32 rounding (same patterns as fp64).
- P5/32 psi monotone, bitwise (RN(psi - y^2) <= psi in any precision).
- P6/32 unit diagonal of G A_s G^T within fp32 rounding.
- P-consistency: with selection margins far above fp32 rounding the fp32 oracle
  picks the fp64 oracle's pattern and its values agree to fp32 accuracy.
- exactness: every value of G is a float widened to double (G = double(G_s)).
- P13/32 PCG with the fp32-set-up G converges within 1.2x the fp64 iterations
  (the paper: fp32 set-up is "safe").
"""
import math

import numpy as np
import pytest

import afsai_inputs as ai
import oracle

U32 = 2.0 ** -24


def is_float_widened(v):
    return np.array_equal(v.astype(np.float32).astype(np.float64), v)


@pytest.mark.parametrize("n,s", [(30, 1), (40, 4)])
def test_P1_fp32_full_pattern(n, s):
    Ad = ai.random_spd_dense(n, sub=n)
    G, Gt, res = oracle.setup_full(ai.from_dense(Ad), n, s, precision="fp32")
    Gd = G.to_dense()
    Linv = np.linalg.inv(np.linalg.cholesky(Ad))
    # forward error of a Cholesky-based inverse ~ n * kappa * u
    assert np.max(np.abs(Gd - Linv)) <= 200 * n * U32 * np.max(np.abs(Linv))
    assert np.all(res.nnz == np.arange(1, n + 1))
    assert is_float_widened(G.val)


def test_P2_fp32_tridiagonal_closed_forms():
    n, k = 64, 7
    res = oracle.setup(ai.tridiag(n), k, 1, precision="fp32")
    for i in range(k, n):
        c, v = res.row(i)
        assert list(c) == list(range(i - k, i + 1))
        psi = res.psi[i, k]
        assert abs(psi - (k + 2) / (k + 1)) <= 8 * U32 * 2
        d = 1.0 / math.sqrt((k + 2) / (k + 1))
        for q in range(1, k + 1):
            got = v[list(c).index(i - q)]
            assert abs(got - d * (k + 1 - q) / (k + 1)) <= 16 * U32, (i, q, got)


def test_P4_fp32_stencil_rationals():
    """3D 7-point, s = 1, k = 3: interior P - i = [-nx^2, -nx, -1], g~ = 1/6 each,
    psi = 11/2 (the fp64 pin P4), within fp32 rounding."""
    nx = 7
    A = ai.poisson3d(nx)
    i = 3 * nx * nx + 3 * nx + 3
    res = oracle.setup(A, 3, 1, rows=np.array([i]), precision="fp32")
    c, v = res.row(0)
    assert sorted(int(x) - i for x in c) == sorted([-nx * nx, -nx, -1, 0])
    psi = res.psi[0, 3]
    assert abs(psi - 5.5) <= 8 * 5.5 * U32
    d = v[list(c).index(i)]
    for j in c:
        if j != i:
            assert abs(v[list(c).index(j)] / d - 1.0 / 6.0) <= 16 * U32


@pytest.mark.parametrize("make,k,s,cap", [(lambda: ai.poisson3d(8), 20, 2, 1 << 30),
                                          (lambda: ai.fe_elasticity(4), 30, 3, 100)])
def test_P5_fp32_psi_monotone_bitwise(make, k, s, cap):
    res = oracle.setup(make(), k, s, 0.0, cap, precision="fp32")
    for t in range(len(res.rows)):
        p = res.psi[t, : res.steps[t] + 1]
        assert np.all(np.diff(p) <= 0)


def test_P6_fp32_unit_diagonal():
    A = ai.hetero_poisson3d(8)
    G, _, _ = oracle.setup_full(A, 20, 2, precision="fp32")
    As = A.to_scipy().astype(np.float32).astype(np.float64)
    Gs = G.to_scipy()
    dg = (Gs @ As @ Gs.T).diagonal()
    assert np.max(np.abs(dg - 1.0)) <= 2e-5


def test_fp32_agrees_with_fp64_when_margins_are_large():
    """Dense random SPD: no exact ties; rows whose fp64 selection margins all exceed
    1e-3 must pick the same pattern in fp32, with values within fp32 accuracy."""
    Ad = ai.random_spd_dense(60, sub=61)
    A = ai.from_dense(Ad)
    r64 = oracle.setup(A, 6, 2)
    r32 = oracle.setup(A, 6, 2, precision="fp32")
    checked = 0
    for t in range(A.n):
        mg = r64.margin[t, : r64.steps[t]]
        if mg.size and np.nanmin(mg) < 1e-3:
            continue
        c64, v64 = r64.row(t)
        c32, v32 = r32.row(t)
        assert np.array_equal(c64, c32), t
        assert np.max(np.abs(v32 - v64)) <= 1e-4 * np.max(np.abs(v64)), t
        checked += 1
    assert checked >= 20


def test_fp32_pcg_within_1p2x_of_fp64():
    """PCG iterations with the fp32-set-up G <= 1.2x those with the fp64 G."""
    for A, k, s, cap in [(ai.poisson3d(16), 20, 2, 1 << 30), (ai.hetero_poisson3d(12), 20, 2, 1 << 30),
                         (ai.fe_elasticity(6), 30, 3, 100)]:
        b, _ = ai.rhs_for(A)
        G, Gt, _ = oracle.setup_full(A, k, s, 0.0, cap)
        G32, Gt32, _ = oracle.setup_full(A, k, s, 0.0, cap, precision="fp32")
        p64 = oracle.pcg(A, G, Gt, b, tol=1e-8)
        p32 = oracle.pcg(A, G32, Gt32, b, tol=1e-8)
        assert p64.converged and p32.converged
        assert p32.iters <= math.ceil(1.2 * p64.iters), (p32.iters, p64.iters)


def test_fp32_notspd_detected():
    with pytest.raises(oracle.OracleError) as e:
        oracle.setup(ai.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]])), 3, 1, precision="fp32")
    assert e.value.code == oracle.ENOTSPD and (e.value.row, e.value.step) == (1, 1)
