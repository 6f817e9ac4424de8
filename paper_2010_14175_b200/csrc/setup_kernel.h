// Launch interface of the per-row set-up kernels (setup_scan.cu, setup_hits.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace afsai {

struct SetupKArgs {
    // A: global rows [a_lo, a_hi); entries of row r: [rowptr[r-a_lo]-base, rowptr[r-a_lo+1]-base)
    const int64_t *rowptr;
    const int32_t *col;
    const double *val;    // fp64 set-up (afsai::dp kernels)
    const float *val32;   // fp32 set-up (afsai::sp kernels): A_s = single(A), same layout
    int64_t base, a_lo, a_hi;
    int64_t nnz;  // entries of A_ext (bounds checks of the debug build)
    // rows to compute: rows ? rows[t] : row_lo + t, for t < nrows
    const int64_t *rows;
    int64_t row_lo, nrows;
    // params (C1-C12)
    int32_t nsteps, s, cap, mmax;
    double eps;
    int32_t H, log2H;   // per-row hash table slots (power of two)
    int32_t cact;       // hit-list kernel: active candidate slots per row
    int32_t lcap;       // pattern-row kernel: list entries per row
    int16_t *lu_global; // pattern-row kernel: per-warp lu lists (lcap each) in global memory
    int32_t warp_smem;  // bytes of shared memory per row (group)
    // outputs, index = global row - out_base
    int64_t out_base;
    int32_t stride;     // slots per row in the fixed-stride scratch (mmax + 1)
    int32_t *scol;
    double *sval;
    int32_t *nnz_row, *steps, *reason;
    unsigned long long *err;       // packed (row << 24) | (step << 4) | code, atomicMin
    int64_t *retry_rows;           // rows whose on-chip tables overflowed
    int32_t *retry_count;
    unsigned long long *work;      // row queue counter
    unsigned long long *counters;  // [0] steps [1] fma_border [2] fma_backsub [3] fma_grad
                                   // [4] grad_entries [5..8] rows by stop reason
                                   // [9..15] phase cycles [16] max universe
};

using SetupKernFn = void (*)(SetupKArgs);

// The kernel factories exist twice: afsai::dp (fp64 set-up) and afsai::sp (fp32
// set-up); the same sources compiled with and without
// -DAFSAI_SETUP_FP32 (setup_common.cuh).
#define AFSAI_SETUP_FACTORIES                                                                        \
    /* general kernel: candidates' rows of A re-read every step (any row length) */                  \
    SetupKernFn scan_kernel_for(int lpr, int mmax, int s);                                             \
    int64_t scan_row_bytes(int H, int mmax, int s);                                                    \
    /* hit-list kernel: rows of A with at most hc + 1 entries (stencils) */                          \
    SetupKernFn hits_kernel_for(int lpr, int mmax, int s, int hc);                                     \
    int64_t hits_row_bytes(int H, int mmax, int s, int cact, int hc);                                  \
    /* hit-list kernel, 32/lpr rows per warp in lockstep (rows <= lpr entries, s <= 4,                 \
       mmax <= 6*lpr) */                                                                               \
    SetupKernFn lockstep_kernel_for(int lpr, int mmax, int s, int hc);                                 \
    int64_t lockstep_row_bytes(int H, int mmax, int s, int cact, int hc);                              \
    /* pattern-row kernel (long rows, s <= 4, mmax <= 128, rows <= 128 entries): 32 lanes per row */   \
    SetupKernFn prow_kernel_for(int mmax, int s, int64_t max_row_len);                                 \
    int64_t prow_row_bytes(int H, int mmax, int s, int lcap);
namespace dp {
AFSAI_SETUP_FACTORIES
}  // namespace dp
namespace sp {
AFSAI_SETUP_FACTORIES
}  // namespace sp
#undef AFSAI_SETUP_FACTORIES

}  // namespace afsai
