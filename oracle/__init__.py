"""ORACLE for the aFSAI hot path — TEST INFRASTRUCTURE ONLY.

Plain fp64 CPU implementation (oracle/afsai_oracle.c, loaded with ctypes) of
what the B200 path computes: the adaptive FSAI set-up (PAPER.md P:289-398,
Eqs. 5-16), the exact transpose, z = G^T(G r) (Eq. 1) and PCG.
See the C file's header for the arithmetic contract and DESIGN.md §3 for every
reading of the paper it encodes.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with
paper_2010_14175_b200/ and never imports it.

Parity status: every function here is pinned by tests/test_oracle_pins.py
(closed forms, dense LAPACK/numpy identities, brute force, finite differences,
SPEC worked examples under tests/golden/).  None is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "afsai_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB32 = os.path.join(_HERE, "liboracle_f32.so")   # the same source with -DOR_FP32

OK, EINVAL, ENOTSPD, ENOMEM, ENOTCONV = 0, 1, 2, 3, 6
STOP_NAMES = {0: "kmax", 1: "cap", 2: "no_candidates", 3: "tolerance"}


class OracleError(RuntimeError):
    def __init__(self, code, row=-1, step=-1):
        super().__init__(f"oracle error {code} (row {row}, step {step})")
        self.code, self.row, self.step = code, row, step


def build(force: bool = False) -> str:
    """Compile liboracle.so and liboracle_f32.so (plain gcc, -ffp-contract=off, libm fma)."""
    for lib, extra in ((_LIB, []), (_LIB32, ["-DOR_FP32"])):
        if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(_SRC):
            cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                   "-pthread"] + extra + ["-o", lib, _SRC, "-lm"]
            subprocess.check_call(cmd)
    return _LIB


_lib = None
_lib32 = None


def _load32():
    """The single-precision set-up oracle (A_s = single(A), float arithmetic, G = double(G_s))."""
    global _lib32
    if _lib32 is None:
        build()
        lib = ctypes.CDLL(_LIB32)
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        lib.oracle_setup_rows.argtypes = [i64, P, P, P, i32, i32, f64, i32, P, i64, i32,
                                          P, P, P, P, P, P, P, P, P, i32]
        lib.oracle_setup_rows.restype = ctypes.c_int
        _lib32 = lib
    return _lib32


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        lib.oracle_setup_rows.argtypes = [i64, P, P, P, i32, i32, f64, i32, P, i64, i32,
                                          P, P, P, P, P, P, P, P, P, i32]
        lib.oracle_setup_rows.restype = ctypes.c_int
        lib.oracle_transpose.argtypes = [i64, P, P, P, P, P, P]
        lib.oracle_transpose.restype = ctypes.c_int
        lib.oracle_apply.argtypes = [i64, P, P, P, P, P, P, P, P, P]
        lib.oracle_apply.restype = ctypes.c_int
        lib.oracle_pcg.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P, f64, i32, P, P, P]
        lib.oracle_pcg.restype = ctypes.c_int
        lib.oracle_gradient.argtypes = [i64, P, P, P, i64, i32, P, P, P, P, i64]
        lib.oracle_gradient.restype = ctypes.c_int64
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _csr_arrays(A):
    rp = np.ascontiguousarray(A.rowptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col, dtype=np.int32)
    v = np.ascontiguousarray(A.val, dtype=np.float64)
    return rp, ci, v


@dataclass
class SetupResult:
    rows: np.ndarray        # int64: global row index of each output row
    nnz: np.ndarray         # int32 per row (incl. diagonal)
    col: np.ndarray         # int32 [nrows, stride]
    val: np.ndarray         # float64 [nrows, stride]
    steps: np.ndarray       # int32 per row
    reason: np.ndarray      # int32 per row (STOP_NAMES)
    psi: np.ndarray | None  # float64 [nrows, nsteps+1] (NaN beyond steps)
    margin: np.ndarray | None  # float64 [nrows, nsteps]

    def row(self, t: int):
        k = int(self.nnz[t])
        return self.col[t, :k].copy(), self.val[t, :k].copy()

    def to_csr(self, n: int):
        """Assemble the CSR of G (requires rows == arange(n))."""
        from afsai_inputs import CSR
        assert len(self.rows) == n and np.all(self.rows == np.arange(n))
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(self.nnz, out=rp[1:])
        mask = np.arange(self.col.shape[1])[None, :] < self.nnz[:, None]
        return CSR(n, rp, self.col[mask].astype(np.int32), self.val[mask].astype(np.float64), "G")


def mmax_of(n, nsteps, s, max_row_nnz):
    return int(min(nsteps * s, max_row_nnz - 1, n))


def setup(A, nsteps: int, s: int, eps: float = 0.0, max_row_nnz: int = 1 << 30,
          rows=None, threads: int | None = None, trace: bool = True, precision: str = "fp64") -> SetupResult:
    """aFSAI set-up of rows `rows` (default: all) of the full symmetric CSR A.
    precision="fp32": the single-precision set-up of P:953-965 -- A's values rounded
    to float (A_s = single(A)), the whole set-up in float, G = double(G_s)."""
    rp, ci, v = _csr_arrays(A)
    if precision == "fp32":
        lib = _load32()
        v = v.astype(np.float32)   # A_s = single(A), round to nearest even
    elif precision == "fp64":
        lib = _load()
    else:
        raise ValueError(precision)
    n = A.n
    rows = np.arange(n, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    nr = len(rows)
    stride = mmax_of(n, nsteps, s, max_row_nnz) + 1
    out_nnz = np.zeros(nr, dtype=np.int32)
    out_col = np.zeros((nr, stride), dtype=np.int32)
    out_val = np.zeros((nr, stride), dtype=np.float64)
    steps = np.zeros(nr, dtype=np.int32)
    reason = np.zeros(nr, dtype=np.int32)
    psi = np.full((nr, nsteps + 1), np.nan) if trace else None
    margin = np.full((nr, max(nsteps, 1)), np.nan) if trace else None
    err_row = np.zeros(1, dtype=np.int64)
    err_step = np.zeros(1, dtype=np.int32)
    if threads is None:
        threads = os.cpu_count() or 1
    rc = lib.oracle_setup_rows(n, _p(rp), _p(ci), _p(v), nsteps, s, float(eps), int(min(max_row_nnz, 2**31 - 1)),
                               _p(rows), nr, stride, _p(out_nnz), _p(out_col), _p(out_val),
                               _p(steps), _p(reason), _p(psi), _p(margin),
                               _p(err_row), _p(err_step), int(threads))
    if rc != OK:
        raise OracleError(rc, int(err_row[0]), int(err_step[0]))
    return SetupResult(rows, out_nnz, out_col, out_val, steps, reason, psi, margin)


def gradient(A, i: int, P, gt):
    """Eq. 15 accumulator (d psi/d gt_j = 2*acc_j) over row i's candidate universe for
    pattern P (insertion order) and off-diagonal values gt.  Returns (j, acc), j ascending."""
    lib = _load()
    rp, ci, v = _csr_arrays(A)
    P = np.ascontiguousarray(P, dtype=np.int32)
    gt = np.ascontiguousarray(gt, dtype=np.float64)
    cap = int(A.n)
    oj = np.zeros(cap, dtype=np.int32)
    oa = np.zeros(cap)
    cnt = lib.oracle_gradient(A.n, _p(rp), _p(ci), _p(v), int(i), len(P), _p(P), _p(gt), _p(oj), _p(oa), cap)
    if cnt < 0:
        raise OracleError(ENOMEM)
    return oj[:cnt].copy(), oa[:cnt].copy()


def transpose(G):
    from afsai_inputs import CSR
    lib = _load()
    rp, ci, v = _csr_arrays(G)
    n = G.n
    trp = np.zeros(n + 1, dtype=np.int64)
    tci = np.zeros(G.nnz, dtype=np.int32)
    tv = np.zeros(G.nnz, dtype=np.float64)
    rc = lib.oracle_transpose(n, _p(rp), _p(ci), _p(v), _p(trp), _p(tci), _p(tv))
    if rc != OK:
        raise OracleError(rc)
    return CSR(n, trp, tci, tv, "Gt")


def apply(G, Gt, r: np.ndarray) -> np.ndarray:
    lib = _load()
    g = _csr_arrays(G)
    t = _csr_arrays(Gt)
    r = np.ascontiguousarray(r, dtype=np.float64)
    z = np.zeros(G.n)
    tmp = np.zeros(G.n)
    lib.oracle_apply(G.n, *map(_p, g), *map(_p, t), _p(r), _p(z), _p(tmp))
    return z


@dataclass
class PcgResult:
    x: np.ndarray
    iters: int
    relres: float
    converged: bool
    history: np.ndarray


def pcg(A, G, Gt, b: np.ndarray, tol: float = 1e-8, max_iters: int = 10000) -> PcgResult:
    """PCG with M^-1 = G^T G (G = None: unpreconditioned CG)."""
    lib = _load()
    a = _csr_arrays(A)
    if G is not None:
        g, t = _csr_arrays(G), _csr_arrays(Gt)
    else:
        g = t = (None, None, None)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(A.n)
    it = np.zeros(1, dtype=np.int32)
    rel = np.zeros(1)
    hist = np.full(max_iters + 1, np.nan)
    rc = lib.oracle_pcg(A.n, *map(_p, a), *map(_p, g), *map(_p, t), _p(b), _p(x), float(tol), int(max_iters),
                        _p(it), _p(rel), _p(hist))
    if rc not in (OK, ENOTCONV):
        raise OracleError(rc)
    return PcgResult(x, int(it[0]), float(rel[0]), rc == OK, hist[: int(it[0]) + 1])


def setup_full(A, nsteps, s, eps=0.0, max_row_nnz=1 << 30, threads=None, precision="fp64"):
    """Convenience: (G, Gt, SetupResult) for all rows."""
    res = setup(A, nsteps, s, eps, max_row_nnz, threads=threads, precision=precision)
    G = res.to_csr(A.n)
    return G, transpose(G), res


# ------------------------------------------------------------------ bounded communication
def comm_matrix(A, bounds):
    """A-hat: n_p x n_p boolean, A-hat[p, q] = 1 iff the block of A
    with rows in stripe p and columns in stripe q holds a nonzero.  Stripe q = rows
    [bounds[q], bounds[q+1])."""
    bounds = np.asarray(bounds, dtype=np.int64)
    npr = len(bounds) - 1
    rows = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.rowptr))
    po = np.searchsorted(bounds, rows, side="right") - 1
    qo = np.searchsorted(bounds, A.col.astype(np.int64), side="right") - 1
    H = np.zeros((npr, npr), dtype=bool)
    H[po, qo] = True
    return H


def stripes_used(Ahat, p, k):
    """The stripes q <= p with (A-hat^k)[p, q] != 0: G-hat <= lower(A-hat^k),
    by k boolean matrix products."""
    R = np.eye(Ahat.shape[0], dtype=bool)
    for _ in range(k):
        R = (R.astype(np.int64) @ Ahat.astype(np.int64)) > 0
    return [q for q in range(p + 1) if R[p, q]]


def setup_bounded(A, bounds, p, k, nsteps, s, eps=0.0, max_row_nnz=1 << 30, precision="fp64"):
    """The rows of stripe p of the bounded-communication set-up: aFSAI on
    the principal submatrix A[I_p, I_p], I_p = the union of the stripes q <= p with
    (A-hat^k)[p, q] != 0; every entry of A outside I_p x I_p is zero.  (Rows outside
    I_p keep only their diagonal: they are never read.)"""
    from afsai_inputs import CSR
    bounds = np.asarray(bounds, dtype=np.int64)
    used = stripes_used(comm_matrix(A, bounds), p, k)
    inI = np.zeros(A.n, dtype=bool)
    for q in used:
        inI[bounds[q]:bounds[q + 1]] = True
    rows = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.rowptr))
    keep = (inI[rows] & inI[A.col]) | (rows == A.col)
    cnt = np.bincount(rows[keep], minlength=A.n)
    rp = np.zeros(A.n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rp[1:])
    T = CSR(A.n, rp, A.col[keep].astype(np.int32), A.val[keep].astype(np.float64), "A_Ip")
    res = setup(T, nsteps, s, eps, max_row_nnz, rows=np.arange(bounds[p], bounds[p + 1]), precision=precision)
    return res, used
