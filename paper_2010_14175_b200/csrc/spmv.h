// Launch interface of spmv.cu
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace afsai {

// PCG scalars, resident in device memory for the whole solve (no per-iteration
// host round trip)
struct PcgState {
    double rz, pq, rr, alpha, beta, bnorm2, rel, true_rr;
    int32_t iters, done;  // done: 0 running, 1 converged, 2 max_iters
    double sum[4];        // multi-GPU: local dot products, all-reduced in place
};

struct SpmvArgs {
    int64_t n;               // rows
    const int64_t *rowptr;   // n + 1, absolute offsets into col/val
    const int32_t *col;
    const double *val;
    const double *x;         // x[col - x_off]
    int64_t x_off;
    double *y;               // n
    const double *w;         // fused dot partner (mode 1, 2, 3)
    double *partials;        // gridDim.x doubles
    unsigned *counter;       // last-block counter (zero at rest)
    PcgState *st;            // optional: skip when st->done; scalar updates
    int sum_idx;             // mode 4: local dot stored in st->sum[sum_idx]
};

// which: 0 = A, 1 = G, 2 = G^T (per-operand override of the miniwarp width)
int spmv_group_width(double avg_nnz, int which);
// mode 0: y = M x; 1: + dot(y, w) -> alpha; 2: + dot(y, w) -> beta, rz; 3: + dot(y, w) -> rz
void launch_spmv(const SpmvArgs &a, int mode, int width, int grid, cudaStream_t st);
void launch_pcg_init(int64_t n, const double *b, double *x, double *r, double *partials, unsigned *counter,
                     PcgState *st, int grid, cudaStream_t s);
void launch_pcg_axpy(int64_t n, double *x, double *r, const double *p, const double *q, double *partials,
                     unsigned *counter, PcgState *st, double tol, int32_t max_iters, int grid, cudaStream_t s);
void launch_pcg_update_p(int64_t n, double *p, const double *z, const PcgState *st, int first, int grid,
                         cudaStream_t s);
void launch_residual(int64_t n, const double *b, const double *ax, double *partials, unsigned *counter, double *out,
                     int grid, cudaStream_t s);
void launch_dfma_probe(double *out, int iters, int grid, cudaStream_t s);
// single-pass apply z += G^T (G r) (z zero on entry; fp64 reductions, non-deterministic order)
void launch_apply_single_pass(int64_t n, const int64_t *rowptr, const int32_t *col, const double *val,
                              const double *r, double *z, const PcgState *st, int width, int grid, cudaStream_t s);
// rz = r.z and beta = rz / rz_old (first: rz only)
void launch_pcg_rz(int64_t n, const double *r, const double *z, double *partials, unsigned *counter, PcgState *st,
                   int first, int grid, cudaStream_t s);
// multi-GPU PCG pieces (scalars from all-reduced st->sum[])
void launch_pcg_init_dist(int64_t n, const double *b, double *x, double *r, double *partials, unsigned *counter,
                          PcgState *st, int grid, cudaStream_t s);      // sum[1] = local b.b
void launch_pcg_start_dist(PcgState *st, cudaStream_t s);               // bnorm2 = sum[1], rz = sum[2]
void launch_pcg_axpy_dist(int64_t n, double *x, double *r, const double *p, const double *q, double *partials,
                          unsigned *counter, PcgState *st, int grid, cudaStream_t s);  // sum[1] = local r.r
void launch_pcg_check_dist(PcgState *st, double tol, int32_t max_iters, cudaStream_t s);
void launch_pcg_update_p_dist(int64_t n, double *p, const double *z, PcgState *st, int first, int grid,
                              cudaStream_t s);
void launch_pcg_rz_dist(PcgState *st, cudaStream_t s);                  // rz = sum[2]

}  // namespace afsai
