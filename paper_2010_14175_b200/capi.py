"""Thin ctypes binding of include/afsai.h (argument marshalling only).

Every function here forwards to libafsai_b200.so under the same name; all
computation happens in the library's CUDA kernels.  There is no fallback: if
the shared library is missing or fails to load, importing this module raises.
Tensors may live on the GPU or on the host (the library stages host arrays).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libafsai_b200.so")
if os.environ.get("AFSAI_DEBUG_LIB") == "1":  # bounds-checked build (build.py --debug)
    LIB_PATH = os.path.join(HERE, "lib", "libafsai_b200_dbg.so")
if os.environ.get("AFSAI_LIB"):  # A/B experiments against another build of the library
    LIB_PATH = os.environ["AFSAI_LIB"]

AFSAI_OK, AFSAI_EINVAL, AFSAI_ENOTSPD, AFSAI_ECUDA, AFSAI_ENCCL, AFSAI_ENOMEM, AFSAI_ENOTCONV, AFSAI_ELIMIT = range(8)
STOP_NAMES = {0: "kmax", 1: "cap", 2: "no_candidates", 3: "tolerance"}

# every symbol declared in include/afsai.h
EXPORTS = [
    "afsai_version", "afsai_strerror", "afsai_ctx_create", "afsai_nccl_unique_id", "afsai_ctx_create_nccl",
    "afsai_ctx_rank", "afsai_ctx_destroy", "afsai_setup", "afsai_apply", "afsai_pcg", "afsai_factor_nnz",
    "afsai_factor_copy", "afsai_factor_trace", "afsai_factor_stats", "afsai_factor_retried", "afsai_factor_destroy",
    "afsai_ctx_launches", "afsai_probe_dfma_peak", "afsai_ctx_set_timing", "afsai_ctx_kernel_times",
    "afsai_setup_block", "afsai_plan_ranges", "afsai_bounded_stripes",
]
KERNEL_CLASSES = ["setup_rows", "assemble", "transpose", "spmv_G", "spmv_Gt", "spmv_A", "vector", "comm"]


class afsai_csr_t(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_begin", ctypes.c_int64), ("rowptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("val", ctypes.c_void_p)]


class afsai_params_t(ctypes.Structure):
    _fields_ = [("nsteps", ctypes.c_int32), ("s", ctypes.c_int32), ("eps", ctypes.c_double),
                ("max_row_nnz", ctypes.c_int32), ("precision", ctypes.c_int32), ("halo_k", ctypes.c_int32)]


class afsai_status_t(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("row", ctypes.c_int64), ("step", ctypes.c_int32),
                ("msg", ctypes.c_char * 160)]


class afsai_setup_stats_t(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("nnz_G", ctypes.c_int64), ("nnz_Gt", ctypes.c_int64),
                ("rows_by_reason", ctypes.c_int64 * 4), ("steps_total", ctypes.c_int64),
                ("fma_border", ctypes.c_int64), ("fma_backsub", ctypes.c_int64), ("fma_grad", ctypes.c_int64),
                ("grad_entries", ctypes.c_int64), ("ms_total", ctypes.c_double), ("ms_rows", ctypes.c_double),
                ("ms_assemble", ctypes.c_double), ("ms_transpose", ctypes.c_double), ("ms_halo", ctypes.c_double),
                ("table_size", ctypes.c_int32), ("rows_per_cta", ctypes.c_int32), ("retried_rows", ctypes.c_int32),
                ("halo_rows", ctypes.c_int32), ("phase_cycles", ctypes.c_int64 * 7),
                ("max_universe", ctypes.c_int64), ("plan", ctypes.c_int32), ("lanes_per_row", ctypes.c_int32),
                ("value_bytes", ctypes.c_int32), ("reserved", ctypes.c_int32), ("halo_bytes", ctypes.c_int64),
                ("halo_mask", ctypes.c_int64)]
    PLANS = {0: "lockstep", 1: "prow", 2: "hits", 3: "scan"}

    PHASES = ["prologue", "gradient", "select", "gather", "border", "backsub", "output"]

    def to_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if name in ("rows_by_reason", "phase_cycles") else v
        return d


class afsai_pcg_report_t(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32), ("rel_res", ctypes.c_double),
                ("true_rel_res", ctypes.c_double), ("ms_solve", ctypes.c_double), ("ms_per_iter", ctypes.c_double)]

    def to_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


def load_library(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"libafsai_b200.so not built ({path}); run __graft_entry__.build()")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    P, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "afsai_version": ([], ctypes.c_char_p),
        "afsai_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "afsai_ctx_create": ([P, P], ctypes.c_int),
        "afsai_nccl_unique_id": ([P], ctypes.c_int),
        "afsai_ctx_create_nccl": ([P, P, P, i32, i32], ctypes.c_int),
        "afsai_ctx_rank": ([P, P, P], ctypes.c_int),
        "afsai_ctx_destroy": ([P], None),
        "afsai_setup": ([P, ctypes.POINTER(afsai_csr_t), ctypes.POINTER(afsai_params_t), P,
                         ctypes.POINTER(afsai_status_t)], ctypes.c_int),
        "afsai_apply": ([P, P, P, P], ctypes.c_int),
        "afsai_pcg": ([P, ctypes.POINTER(afsai_csr_t), P, P, P, f64, i32, ctypes.POINTER(afsai_pcg_report_t),
                       ctypes.POINTER(afsai_status_t)], ctypes.c_int),
        "afsai_factor_nnz": ([P, P, P], ctypes.c_int),
        "afsai_factor_copy": ([P, i32, P, P, P], ctypes.c_int),
        "afsai_factor_trace": ([P, P, P], ctypes.c_int),
        "afsai_factor_stats": ([P, ctypes.POINTER(afsai_setup_stats_t)], ctypes.c_int),
        "afsai_factor_retried": ([P, P, i64, P], ctypes.c_int),
        "afsai_factor_destroy": ([P], None),
        "afsai_ctx_launches": ([P], i64),
        "afsai_probe_dfma_peak": ([P, P, P], ctypes.c_int),
        "afsai_ctx_set_timing": ([P, i32], ctypes.c_int),
        "afsai_ctx_kernel_times": ([P, P, P], ctypes.c_int),
        "afsai_setup_block": ([P, ctypes.POINTER(afsai_csr_t), i64, i64, ctypes.POINTER(afsai_params_t), P,
                               ctypes.POINTER(afsai_status_t)], ctypes.c_int),
        "afsai_plan_ranges": ([i32, i32, P, P, P, P, i32], ctypes.c_int),
        "afsai_bounded_stripes": ([i32, i32, P, i32, P], ctypes.c_int),
    }
    for name in EXPORTS:
        fn = getattr(lib, name)  # AttributeError if the symbol is missing
        fn.argtypes, fn.restype = sig[name]
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


class AfsaiError(RuntimeError):
    def __init__(self, code, status: afsai_status_t | None = None, where: str = ""):
        msg = lib().afsai_strerror(code).decode()
        self.code = code
        self.row = status.row if status is not None else -1
        self.step = status.step if status is not None else -1
        detail = status.msg.decode(errors="replace") if status is not None else ""
        super().__init__(f"{where}: {msg} (code {code}) {detail} row={self.row} step={self.step}")


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return t.ctypes.data_as(ctypes.c_void_p)  # numpy


def make_csr(rowptr, col, val, n_cols: int, row_begin: int = 0) -> afsai_csr_t:
    n_rows = (rowptr.numel() if hasattr(rowptr, "numel") else len(rowptr)) - 1
    nnz = int(col.numel() if hasattr(col, "numel") else len(col))
    c = afsai_csr_t(n_rows, n_cols, nnz, row_begin, None, None, None)
    c.rowptr = _ptr(rowptr).value if n_rows >= 0 else None
    c.col = _ptr(col).value
    c.val = _ptr(val).value
    c._keep = (rowptr, col, val)  # the struct keeps its arrays alive
    return c


# ----------------------------------------------------------------- same-name wrappers
def afsai_ctx_create(stream_ptr: int = 0):
    h = ctypes.c_void_p()
    rc = lib().afsai_ctx_create(ctypes.byref(h), ctypes.c_void_p(stream_ptr))
    if rc:
        raise AfsaiError(rc, where="afsai_ctx_create")
    return h


def afsai_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().afsai_nccl_unique_id(buf)
    if rc:
        raise AfsaiError(rc, where="afsai_nccl_unique_id")
    return buf.raw


def afsai_ctx_create_nccl(stream_ptr: int, uid: bytes, rank: int, nranks: int):
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    rc = lib().afsai_ctx_create_nccl(ctypes.byref(h), ctypes.c_void_p(stream_ptr), buf, rank, nranks)
    if rc:
        raise AfsaiError(rc, where="afsai_ctx_create_nccl")
    return h


def afsai_ctx_destroy(ctx):
    lib().afsai_ctx_destroy(ctx)


def afsai_ctx_launches(ctx) -> int:
    return int(lib().afsai_ctx_launches(ctx))


AFSAI_PREC_FP64, AFSAI_PREC_FP32 = 0, 1
PRECISIONS = {"fp64": AFSAI_PREC_FP64, "fp32": AFSAI_PREC_FP32}


def afsai_setup(ctx, A: afsai_csr_t, nsteps: int, s: int, eps: float, max_row_nnz: int, precision: int = 0,
                halo_k: int = 0):
    p = afsai_params_t(nsteps, s, eps, max_row_nnz, precision, halo_k)
    f = ctypes.c_void_p()
    st = afsai_status_t()
    rc = lib().afsai_setup(ctx, ctypes.byref(A), ctypes.byref(p), ctypes.byref(f), ctypes.byref(st))
    if rc:
        raise AfsaiError(rc, st, "afsai_setup")
    return f


def afsai_apply(ctx, F, r, z):
    rc = lib().afsai_apply(ctx, F, _ptr(r), _ptr(z))
    if rc:
        raise AfsaiError(rc, where="afsai_apply")


def afsai_pcg(ctx, A: afsai_csr_t, F, b, x, tol: float = 1e-8, max_iters: int = 10000, raise_notconv=False):
    rep = afsai_pcg_report_t()
    st = afsai_status_t()
    rc = lib().afsai_pcg(ctx, ctypes.byref(A), F, _ptr(b), _ptr(x), float(tol), int(max_iters),
                         ctypes.byref(rep), ctypes.byref(st))
    if rc and (rc != AFSAI_ENOTCONV or raise_notconv):
        raise AfsaiError(rc, st, "afsai_pcg")
    return rep


def afsai_factor_nnz(F):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    rc = lib().afsai_factor_nnz(F, ctypes.byref(a), ctypes.byref(b))
    if rc:
        raise AfsaiError(rc, where="afsai_factor_nnz")
    return a.value, b.value


def afsai_factor_copy(F, which: int, rowptr, col, val):
    rc = lib().afsai_factor_copy(F, which, _ptr(rowptr), _ptr(col), _ptr(val))
    if rc:
        raise AfsaiError(rc, where="afsai_factor_copy")


def afsai_factor_trace(F, steps, reason):
    rc = lib().afsai_factor_trace(F, _ptr(steps), _ptr(reason))
    if rc:
        raise AfsaiError(rc, where="afsai_factor_trace")


def afsai_factor_stats(F) -> afsai_setup_stats_t:
    s = afsai_setup_stats_t()
    rc = lib().afsai_factor_stats(F, ctypes.byref(s))
    if rc:
        raise AfsaiError(rc, where="afsai_factor_stats")
    return s


def afsai_factor_retried(F, rows=None) -> int:
    """Number of retried rows; with a (host or device) int64 tensor `rows`, also copies them."""
    cnt = ctypes.c_int64()
    mx = rows.numel() if rows is not None else 0
    rc = lib().afsai_factor_retried(F, _ptr(rows) if rows is not None else None, mx, ctypes.byref(cnt))
    if rc:
        raise AfsaiError(rc, where="afsai_factor_retried")
    return int(cnt.value)


def afsai_factor_destroy(F):
    lib().afsai_factor_destroy(F)


def afsai_probe_dfma_peak(ctx):
    fl, ms = ctypes.c_double(), ctypes.c_double()
    rc = lib().afsai_probe_dfma_peak(ctx, ctypes.byref(fl), ctypes.byref(ms))
    if rc:
        raise AfsaiError(rc, where="afsai_probe_dfma_peak")
    return fl.value, ms.value


def afsai_ctx_set_timing(ctx, enable: bool):
    rc = lib().afsai_ctx_set_timing(ctx, 1 if enable else 0)
    if rc:
        raise AfsaiError(rc, where="afsai_ctx_set_timing")


def afsai_ctx_kernel_times(ctx) -> dict:
    """{class: (launches, total_ms)} since the last afsai_ctx_set_timing."""
    n = len(KERNEL_CLASSES)
    la = (ctypes.c_int64 * n)()
    ms = (ctypes.c_double * n)()
    rc = lib().afsai_ctx_kernel_times(ctx, la, ms)
    if rc:
        raise AfsaiError(rc, where="afsai_ctx_kernel_times")
    return {k: (int(la[i]), float(ms[i])) for i, k in enumerate(KERNEL_CLASSES)}


def afsai_setup_block(ctx, A_ext: afsai_csr_t, row_lo: int, n_rows: int, nsteps: int, s: int, eps: float,
                      max_row_nnz: int, precision: int = 0):
    p = afsai_params_t(nsteps, s, eps, max_row_nnz, precision)
    f = ctypes.c_void_p()
    st = afsai_status_t()
    rc = lib().afsai_setup_block(ctx, ctypes.byref(A_ext), int(row_lo), int(n_rows), ctypes.byref(p),
                                 ctypes.byref(f), ctypes.byref(st))
    if rc:
        raise AfsaiError(rc, st, "afsai_setup_block")
    return f


def afsai_plan_ranges(me: int, nranks: int, bounds, lo, hi):
    """Host-only halo plan: list of (kind 'send'|'recv', peer, begin, count)."""
    import numpy as np
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    l = np.ascontiguousarray(lo, dtype=np.int64)
    h = np.ascontiguousarray(hi, dtype=np.int64)
    cap = 4 * nranks + 4
    out = np.zeros(4 * cap, dtype=np.int64)
    k = lib().afsai_plan_ranges(me, nranks, _ptr(b), _ptr(l), _ptr(h), _ptr(out), cap)
    if k < 0:
        raise AfsaiError(AFSAI_EINVAL, where="afsai_plan_ranges")
    return [("send" if out[4 * t] == 0 else "recv", int(out[4 * t + 1]), int(out[4 * t + 2]), int(out[4 * t + 3]))
            for t in range(k)]


def afsai_bounded_stripes(me: int, ahat_rows, k: int) -> list:
    """Host-only: the stripes q <= me with (A-hat^k)_me,q != 0 (ahat_rows: one int bit mask per rank)."""
    import numpy as np
    rows = np.ascontiguousarray(np.asarray(ahat_rows, dtype=np.uint64))
    mask = ctypes.c_uint64()
    rc = lib().afsai_bounded_stripes(int(me), len(rows), rows.ctypes.data_as(ctypes.c_void_p), int(k),
                                     ctypes.byref(mask))
    if rc:
        raise AfsaiError(rc, where="afsai_bounded_stripes")
    return [q for q in range(len(rows)) if (mask.value >> q) & 1]
