/*
 * afsai.h -- C ABI of libafsai_b200.so: the B200-native adaptive FSAI hot path.
 *
 * What the library computes (PAPER.md = P:n, SPEC.md = S:n):
 *   afsai_setup  the adaptive factored sparse approximate inverse G of an SPD A,
 *                G^T G ~ A^-1 (Eq. 1), grown row by row with the
 *                Kaporin gradient (Eqs. 13-16), each row scaled so
 *                diag(G A G^T) = I (Eqs. 8-9, with the square root,
 *                DESIGN.md R1); also builds G^T.
 *   afsai_apply  z = G^T (G r) (Eq. 1).
 *   afsai_pcg    PCG preconditioned with G^T G, x0 = 0, stop at
 *                ||r||_2/||b||_2 <= tol (R12).
 * The arithmetic of afsai_setup follows the contract C1-C12 of DESIGN.md §3.1,
 * so its G is bitwise reproducible and equal to the CPU oracle's.
 *
 * Conventions
 *   - Every call returns an afsai error code (AFSAI_OK = 0).  On failure the
 *     optional afsai_status_t* is filled (code, offending row/step, message).
 *   - Pointers to arrays may be DEVICE or HOST memory unless stated otherwise;
 *     the library detects which (cudaPointerGetAttributes) and stages host
 *     arrays through device memory inside the call.  Device arrays must be on
 *     the context's device.
 *   - All device work is ordered on the context's CUDA stream.
 *   - Inputs are caller-owned, read-only during the call and never freed by the
 *     library.  Factors are library-owned until afsai_factor_destroy.
 *   - Index widths: row pointers int64, column indices int32 (n < 2^31),
 *     values fp64.
 *   - Multi-GPU: one process per GPU.  A context created with
 *     afsai_ctx_create_nccl owns an NCCL communicator; A_local then holds only
 *     the contiguous rows [row_begin, row_begin + n_rows) of the global A, with
 *     GLOBAL column indices.  The library exchanges the set-up halo and the
 *     PCG halos itself.
 */
#ifndef AFSAI_H
#define AFSAI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes */
#define AFSAI_OK 0
#define AFSAI_EINVAL 1      /* bad argument: null, sizes, unsorted/duplicate columns, missing or <= 0
                               diagonal, non-finite value, params out of range                    */
#define AFSAI_ENOTSPD 2     /* Cholesky pivot !(t > 1e-30) or psi !(> 0): A is not SPD;
                               status.row / status.step identify the first (lowest) failing row     */
#define AFSAI_ECUDA 3       /* a CUDA runtime error                                                */
#define AFSAI_ENCCL 4       /* an NCCL error                                                       */
#define AFSAI_ENOMEM 5      /* device allocation failed                                            */
#define AFSAI_ENOTCONV 6    /* afsai_pcg only, non-fatal: max_iters reached; report filled */
#define AFSAI_ELIMIT 7      /* an implementation limit (e.g. max pattern size > AFSAI_MAX_MMAX)    */

#define AFSAI_MAX_MMAX 128  /* largest off-diagonal pattern per row: min(nsteps*s, max_row_nnz-1) */
#define AFSAI_MAX_S 16      /* largest s (entries added per step)                                  */

/* stop reasons (per row, C3/C8) */
#define AFSAI_STOP_KMAX 0
#define AFSAI_STOP_CAP 1
#define AFSAI_STOP_NOCAND 2
#define AFSAI_STOP_TOL 3

/* A CSR matrix (or a contiguous row block of one).  Columns strictly increasing
 * within each row and GLOBAL; rowptr[0] may be nonzero (offsets are relative to
 * rowptr[0]); the diagonal must be stored.  For afsai_setup A must be SPD and
 * bitwise symmetric (C1); the symmetry check (pairs within the rows
 * held here) runs by default, AFSAI_VALIDATE=0 skips it. */
typedef struct {
    int64_t n_rows;        /* rows held here                                         */
    int64_t n_cols;        /* global n                                               */
    int64_t nnz;           /* rowptr[n_rows] - rowptr[0]                             */
    int64_t row_begin;     /* global index of local row 0 (0 on one GPU)             */
    const int64_t *rowptr; /* n_rows + 1                                             */
    const int32_t *col;    /* nnz                                                    */
    const double *val;     /* nnz                                                    */
} afsai_csr_t;

/* aFSAI control parameters (BASELINE.json) */
typedef struct {
    int32_t nsteps;        /* k_max >= 0: maximum adaptive steps per row             */
    int32_t s;             /* 1 <= s <= AFSAI_MAX_S: entries added per step          */
    double eps;            /* 0 <= eps < 1: stop a row when psi_k/psi_0 <= eps (Eq.16)*/
    int32_t max_row_nnz;   /* >= 1: cap on nnz of a row of G, diagonal included (R8)  */
    int32_t precision;     /* set-up arithmetic: AFSAI_PREC_FP64 (0, default) or
                              AFSAI_PREC_FP32 (§4.3: A_s = single(A),
                              the set-up in fp32, G = double(G_s); apply/PCG stay fp64) */
    int32_t halo_k;        /* multi-GPU set-up halo: 0 (default) = the exact halo, G bitwise the
                              1-GPU G; 1..3 = the paper's bounded communication:
                              rank p sets up on A[I_p, I_p], I_p = the row stripes q <= p with
                              (A-hat^k)_pq != 0 (A-hat: the block pattern of A over ranks),
                              entries outside are zero -- G changes with k.  Ignored on 1 GPU. */
} afsai_params_t;
#define AFSAI_PREC_FP64 0
#define AFSAI_PREC_FP32 1

typedef struct {
    int32_t code;          /* AFSAI_* */
    int64_t row;           /* global row of an ENOTSPD / EINVAL, else -1             */
    int32_t step;          /* adaptive step of an ENOTSPD, else -1                   */
    char msg[160];
} afsai_status_t;

/* Set-up statistics (device-timed with CUDA events on the context stream). */
typedef struct {
    int64_t n_rows;              /* local rows                                       */
    int64_t nnz_G;               /* local nnz of G (= nnz of local rows of G^T on 1 GPU) */
    int64_t nnz_Gt;              /* local nnz of G^T                                 */
    int64_t rows_by_reason[4];   /* AFSAI_STOP_* histogram                           */
    int64_t steps_total;         /* sum over rows of adaptive steps taken            */
    int64_t fma_border;          /* algorithmic FMAs: bordering + forward solve + psi */
    int64_t fma_backsub;         /* algorithmic FMAs: back-substitution               */
    int64_t fma_grad;            /* algorithmic FMAs: gradient (pattern entries hit)  */
    int64_t grad_entries;        /* A entries scanned by the gradient                 */
    double ms_total;             /* whole afsai_setup (first kernel .. G^T ready)     */
    double ms_rows;              /* the per-row set-up kernel                         */
    double ms_assemble;          /* count/scan/fill of G                              */
    double ms_transpose;         /* G^T                                               */
    double ms_halo;              /* multi-GPU set-up halo exchange (0 on one GPU)     */
    int32_t table_size;          /* per-row hash table slots used by the kernel       */
    int32_t rows_per_cta;        /* rows (warps) resident per CTA                     */
    int32_t retried_rows;        /* rows recomputed with a larger table               */
    int32_t halo_rows;           /* rows of A received from other ranks              */
    int64_t phase_cycles[7];     /* SM cycles summed over warps in the set-up kernel:
                                    prologue, gradient, select, gather, border, backsub, output */
    int64_t max_universe;        /* largest candidate+pattern set of a row (table keys) */
    int32_t plan;                /* kernel plan of the main pass: AFSAI_PLAN_*        */
    int32_t lanes_per_row;       /* lanes of a warp working on one row               */
    int32_t value_bytes;         /* 8: fp64 set-up; 4: fp32 set-up (AFSAI_PREC_FP32)   */
    int32_t reserved;
    int64_t halo_bytes;          /* multi-GPU: bytes of A rows received for the set-up halo */
    int64_t halo_mask;           /* multi-GPU: bit q = the set-up used rank q's stripe      */
} afsai_setup_stats_t;
#define AFSAI_PLAN_LOCKSTEP 0    /* hit lists, several rows per warp in lockstep (stencils) */
#define AFSAI_PLAN_PROW 1        /* pattern-row folds (long rows, FE)                        */
#define AFSAI_PLAN_HITS 2        /* hit lists, one row per lane group                        */
#define AFSAI_PLAN_SCAN 3        /* general: candidate rows re-read every step               */

typedef struct {
    int32_t iters;               /* PCG iterations performed                          */
    int32_t converged;           /* 1 if ||r||/||b|| <= tol was reached               */
    double rel_res;              /* recurrence ||r_k||/||b||                          */
    double true_rel_res;         /* ||b - A x||/||b|| recomputed at the end           */
    double ms_solve;             /* device time of the whole solve                    */
    double ms_per_iter;
} afsai_pcg_report_t;

typedef struct afsai_ctx_s *afsai_ctx_t;       /* opaque: device, stream, optional NCCL comm */
typedef struct afsai_factor_s *afsai_factor_t; /* opaque, library-owned: G, G^T, halo plans  */

/* ---- version / errors */
const char *afsai_version(void);
const char *afsai_strerror(int code);

/* ---- contexts.  `stream` is a cudaStream_t (NULL = the legacy default stream).
 * The device is the current CUDA device of the calling thread. */
int afsai_ctx_create(afsai_ctx_t *ctx, void *stream);
/* NCCL: rank 0 calls afsai_nccl_unique_id, the caller broadcasts the 128 bytes
 * (e.g. over torch.distributed), then every rank calls afsai_ctx_create_nccl. */
int afsai_nccl_unique_id(char id[128]);
int afsai_ctx_create_nccl(afsai_ctx_t *ctx, void *stream, const char id[128], int32_t rank, int32_t nranks);
int afsai_ctx_rank(afsai_ctx_t ctx, int32_t *rank, int32_t *nranks);
void afsai_ctx_destroy(afsai_ctx_t ctx);

/* ---- the hot path */

/* Adaptive FSAI set-up of the rows of A_local.  On success *out is
 * a new factor holding the local rows of G and of G^T.  Synchronises the
 * context stream once (nnz and status).  status may be NULL. */
int afsai_setup(afsai_ctx_t ctx, const afsai_csr_t *A_local, const afsai_params_t *params,
                afsai_factor_t *out, afsai_status_t *status);

/* z = G^T (G r) on the local rows (Eq. 1).  r, z: n_rows doubles, must not
 * alias.  Fully asynchronous on device buffers; synchronous when r or z is
 * host memory.  Multi-GPU: collective over the context's communicator. */
int afsai_apply(afsai_ctx_t ctx, afsai_factor_t F, const double *r, double *z);

/* PCG on A_local x = b with M^-1 = G^T G; x0 = 0 (x is output only).
 * Returns AFSAI_OK if converged, AFSAI_ENOTCONV (report filled) otherwise.
 * A_local must be the same matrix the factor was built from.  rep may be NULL.
 * Multi-GPU: collective; b and x hold the local rows. */
int afsai_pcg(afsai_ctx_t ctx, const afsai_csr_t *A_local, afsai_factor_t F, const double *b, double *x,
              double tol, int32_t max_iters, afsai_pcg_report_t *rep, afsai_status_t *status);

/* Set-up of the row block [row_lo, row_lo + n_rows) from A_ext, a CSR holding
 * the rows [A_ext.row_begin, A_ext.row_begin + A_ext.n_rows) of the global A
 * (global columns).  A_ext must contain every row the block's patterns can
 * reach: with beta the bandwidth of A, the rows [row_lo - nsteps*beta, row_lo)
 * below the block suffice.  The factor holds the block's rows of
 * G (no G^T); they are bitwise equal to the same rows of a whole-matrix
 * afsai_setup (row independence).  One GPU, no NCCL: the
 * building block of the multi-GPU set-up, exposed for partition emulation. */
int afsai_setup_block(afsai_ctx_t ctx, const afsai_csr_t *A_ext, int64_t row_lo, int64_t n_rows,
                      const afsai_params_t *params, afsai_factor_t *out, afsai_status_t *status);

/* Host-only halo planner (no GPU): ranks own [bounds[q], bounds[q+1]) and rank q
 * needs the extended range [lo[q], hi[q]).  Writes rank `me`'s transfers as
 * 4-tuples (kind 0 = send / 1 = recv, peer, global begin, count) into out and
 * returns their number (-1 if max_out is too small). */
int afsai_plan_ranges(int32_t me, int32_t nranks, const int64_t *bounds, const int64_t *lo, const int64_t *hi,
                      int64_t *out, int32_t max_out);

/* Host-only (no GPU): the stripes rank `me` gathers in the bounded-communication
 * set-up (params.halo_k = k): ahat_rows[q] is row q of the
 * communication matrix A-hat as a bit mask (bit r set iff a row of stripe q has a
 * column in stripe r); *mask gets bit q for every q <= me with (A-hat^k)_me,q != 0.
 * nranks <= 64; returns AFSAI_EINVAL on bad arguments. */
int afsai_bounded_stripes(int32_t me, int32_t nranks, const uint64_t *ahat_rows, int32_t k, uint64_t *mask);

/* ---- factor access */
int afsai_factor_nnz(afsai_factor_t F, int64_t *nnz_G, int64_t *nnz_Gt);
/* Copy the local rows of G (which == 0) or G^T (which == 1) into caller buffers
 * (host or device): rowptr n_rows+1 (starting at 0), col/val nnz. */
int afsai_factor_copy(afsai_factor_t F, int32_t which, int64_t *rowptr, int32_t *col, double *val);
/* Per-row trace: steps taken and stop reason (int32 n_rows each; host or device). */
int afsai_factor_trace(afsai_factor_t F, int32_t *steps, int32_t *reason);
int afsai_factor_stats(afsai_factor_t F, afsai_setup_stats_t *stats);
/* Rows whose on-chip candidate tables overflowed in the first pass of the set-up
 * kernel and were recomputed by a retry pass with larger tables:
 * *count = their number (always set); the first min(count, max_rows) global row
 * indices (unordered) are copied into rows (host or device; may be NULL). */
int afsai_factor_retried(afsai_factor_t F, int64_t *rows, int64_t max_rows, int64_t *count);
void afsai_factor_destroy(afsai_factor_t F);

/* ---- instrumentation for bench/tests: number of kernels this library has
 * launched since the context was created, and a DFMA-throughput probe that
 * measures the fp64 FMA peak of the device (flop/s) used as the set-up
 * roofline denominator. */
int64_t afsai_ctx_launches(afsai_ctx_t ctx);
int afsai_probe_dfma_peak(afsai_ctx_t ctx, double *flops_per_s, double *ms);

/* Optional per-kernel-class timing (CUDA events around every launch of the
 * class, on the context stream).  Classes: */
#define AFSAI_K_SETUP_ROWS 0   /* the per-row set-up kernel                    */
#define AFSAI_K_ASSEMBLE 1     /* validation, scans, fill of G                  */
#define AFSAI_K_TRANSPOSE 2    /* G^T count/scatter/sort                        */
#define AFSAI_K_SPMV_G 3       /* t = G r                                       */
#define AFSAI_K_SPMV_GT 4      /* z = G^T t (+ fused dot)                       */
#define AFSAI_K_SPMV_A 5       /* q = A p (+ fused dot)                         */
#define AFSAI_K_VECTOR 6       /* PCG vector kernels (axpy, p update, init)     */
#define AFSAI_K_COMM 7         /* NCCL halo exchanges / all-reduces             */
#define AFSAI_K_NCLASSES 8
/* enable (1) / disable (0) and reset the accumulators */
int afsai_ctx_set_timing(afsai_ctx_t ctx, int32_t enable);
/* launches[k] and total device milliseconds ms[k] per class since the reset;
 * synchronises the context stream. */
int afsai_ctx_kernel_times(afsai_ctx_t ctx, int64_t launches[AFSAI_K_NCLASSES], double ms[AFSAI_K_NCLASSES]);

#ifdef __cplusplus
}
#endif
#endif /* AFSAI_H */
