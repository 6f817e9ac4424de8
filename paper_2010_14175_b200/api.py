"""Torch conveniences over the C ABI: device CSR tensors, a context bound to a
torch CUDA stream (and optionally a torch.distributed group for NCCL), and a
Factor object.  PyTorch provides memory, streams and process groups only;
every step of the path runs in libafsai_b200.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import capi


@dataclass
class DeviceCSR:
    """Row block [row_begin, row_begin + n_rows) of an n_cols x n_cols CSR matrix."""
    rowptr: torch.Tensor  # int64
    col: torch.Tensor     # int32
    val: torch.Tensor     # float64
    n_cols: int
    row_begin: int = 0

    @property
    def n_rows(self):
        return self.rowptr.numel() - 1

    @property
    def nnz(self):
        return self.col.numel()

    def c(self) -> capi.afsai_csr_t:
        return capi.make_csr(self.rowptr, self.col, self.val, self.n_cols, self.row_begin)

    @staticmethod
    def from_numpy(A, device="cuda", row_begin=0, n_rows=None, pin=False):
        """From an afsai_inputs.CSR (or any object with rowptr/col/val/n)."""
        import numpy as np
        n = A.n
        if n_rows is None:
            n_rows = n - row_begin
        rp = np.asarray(A.rowptr[row_begin: row_begin + n_rows + 1], dtype=np.int64)
        lo, hi = int(rp[0]), int(rp[-1])
        rowptr = torch.from_numpy(rp - lo)
        col = torch.from_numpy(np.ascontiguousarray(A.col[lo:hi], dtype=np.int32))
        val = torch.from_numpy(np.ascontiguousarray(A.val[lo:hi], dtype=np.float64))
        if device == "cpu":
            if pin:
                rowptr, col, val = rowptr.pin_memory(), col.pin_memory(), val.pin_memory()
            return DeviceCSR(rowptr, col, val, n, row_begin)
        return DeviceCSR(rowptr.to(device), col.to(device), val.to(device), n, row_begin)


class Context:
    def __init__(self, stream: torch.cuda.Stream | None = None, group=None):
        self.stream = stream or torch.cuda.current_stream()
        self.rank, self.world = 0, 1
        if group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()):
            import torch.distributed as dist
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if self.world > 1:
            import torch.distributed as dist
            uid = [capi.afsai_nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(uid, src=0, group=group)
            self.h = capi.afsai_ctx_create_nccl(self.stream.cuda_stream, uid[0], self.rank, self.world)
        else:
            self.h = capi.afsai_ctx_create(self.stream.cuda_stream)

    def launches(self) -> int:
        return capi.afsai_ctx_launches(self.h)

    def set_timing(self, enable: bool = True):
        capi.afsai_ctx_set_timing(self.h, enable)

    def kernel_times(self) -> dict:
        return capi.afsai_ctx_kernel_times(self.h)

    def dfma_peak(self):
        return capi.afsai_probe_dfma_peak(self.h)

    def close(self):
        if self.h:
            capi.afsai_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Factor:
    """G (and G^T) of one afsai_setup call."""

    def __init__(self, ctx: Context, A: DeviceCSR, nsteps: int, s: int, eps: float = 0.0,
                 max_row_nnz: int = 1 << 30, precision: str = "fp64", halo_k: int = 0):
        """precision="fp32": the single-precision set-up; G is fp64 either way.
        halo_k (multi-GPU): 0 = exact set-up halo; 1..3 = bounded communication A-hat^k."""
        self.ctx = ctx
        self.A = A
        self.h = capi.afsai_setup(ctx.h, A.c(), nsteps, s, eps, min(max_row_nnz, 2**31 - 1),
                                  capi.PRECISIONS[precision], halo_k)

    @property
    def nnz(self):
        return capi.afsai_factor_nnz(self.h)

    def _copy(self, which: int, device="cuda"):
        nnzG, nnzT = self.nnz
        nnz = nnzT if which else nnzG
        n = self.A.n_rows
        rp = torch.empty(n + 1, dtype=torch.int64, device=device)
        ci = torch.empty(nnz, dtype=torch.int32, device=device)
        v = torch.empty(nnz, dtype=torch.float64, device=device)
        capi.afsai_factor_copy(self.h, which, rp, ci, v)
        return rp, ci, v

    def G(self, device="cuda"):
        return self._copy(0, device)

    def Gt(self, device="cuda"):
        return self._copy(1, device)

    def trace(self, device="cuda"):
        n = self.A.n_rows
        st = torch.empty(n, dtype=torch.int32, device=device)
        rs = torch.empty(n, dtype=torch.int32, device=device)
        capi.afsai_factor_trace(self.h, st, rs)
        return st, rs

    def retried_rows(self):
        """Global rows the set-up recomputed with larger on-chip tables (sorted, int64 numpy)."""
        import numpy as np
        k = capi.afsai_factor_retried(self.h)
        rows = torch.empty(max(k, 1), dtype=torch.int64)
        if k:
            capi.afsai_factor_retried(self.h, rows)
        return np.sort(rows[:k].numpy())

    def stats(self) -> dict:
        return capi.afsai_factor_stats(self.h).to_dict()

    def apply(self, r: torch.Tensor, z: torch.Tensor | None = None) -> torch.Tensor:
        if z is None:
            z = torch.empty_like(r)
        capi.afsai_apply(self.ctx.h, self.h, r, z)
        return z

    def pcg(self, b: torch.Tensor, tol=1e-8, max_iters=10000, x: torch.Tensor | None = None):
        if x is None:
            x = torch.empty_like(b)
        rep = capi.afsai_pcg(self.ctx.h, self.A.c(), self.h, b, x, tol, max_iters)
        return x, rep.to_dict()

    def close(self):
        if self.h:
            capi.afsai_factor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
