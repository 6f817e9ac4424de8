// Launch interface of the per-row set-up kernel (setup_kernel.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace afsai {

struct SetupKArgs {
    // A: global rows [a_lo, a_hi); entries of row r: [rowptr[r-a_lo]-base, rowptr[r-a_lo+1]-base)
    const int64_t *rowptr;
    const int32_t *col;
    const double *val;
    int64_t base, a_lo, a_hi;
    // rows to compute: rows ? rows[t] : row_lo + t, for t < nrows
    const int64_t *rows;
    int64_t row_lo, nrows;
    // params (C1-C12)
    int32_t nsteps, s, cap, mmax;
    double eps;
    int32_t H, log2H;   // per-row hash table slots (power of two)
    int32_t warp_smem;  // bytes of shared memory per warp (setup_warp_bytes)
    // outputs, index = global row - out_base
    int64_t out_base;
    int32_t stride;     // slots per row in the fixed-stride scratch (mmax + 1)
    int32_t *scol;
    double *sval;
    int32_t *nnz_row, *steps, *reason;
    unsigned long long *err;       // packed (row << 24) | (step << 4) | code, atomicMin
    int64_t *retry_rows;           // rows whose table overflowed
    int32_t *retry_count;
    unsigned long long *work;      // row queue counter
    unsigned long long *counters;  // [0] steps [1] fma_border [2] fma_backsub [3] fma_grad
                                   // [4] grad_entries [5..8] rows by stop reason
};

int64_t setup_warp_bytes(int H, int mmax, int s);
cudaError_t launch_setup_rows(const SetupKArgs &a, int warps_per_cta, int grid, cudaStream_t st);
int setup_occupancy(int mmax, int s, int warps_per_cta, size_t smem);

}  // namespace afsai
