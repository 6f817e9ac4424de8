/*
 * afsai_oracle.c -- plain, slow, fp64 CPU ORACLE for the aFSAI hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2010_14175_b200/csrc); neither includes the other.
 *
 * What it computes (PAPER.md = P:n, SPEC.md = S:n, DESIGN.md §3 "readings"):
 *   - adaptive FSAI set-up, per row i, independently (Eqs. 5-16):
 *       identity initial guess, Kaporin-gradient candidates
 *       (Eq. 15), top-s enlargement, the local SPD
 *       system of Eq. 7 solved by Cholesky, psi of Eq. 13 /
 *       the Eq. 9 denominator, exit test Eq. 16, final scaling
 *       Eqs. 8-9 with the square root (R1).
 *   - the exact transpose of G, rows ascending.
 *   - z = G^T (G r) (Eq. 1) as two plain CSR products.
 *   - PCG with x0 = 0, stop at ||r||/||r0|| <= tol.
 *
 * The oracle REFACTORS the local Cholesky factor from scratch at every step
 * (the plain reading of "solving (7)" each step); the GPU extends
 * it incrementally.  The arithmetic contract (C1-C12) fixes the
 * order of every floating-point operation so the two agree bitwise:
 *   gradient  acc_j = +0; for (r, v) in row j of A, ascending r, r in P-bar U {i}:
 *             acc_j = fma(v, gt_r, acc_j)  with gt_i = 1          (Eq. 15)
 *   select    top-room by (|acc| desc, j asc), append ascending j
 *   Cholesky  row q:  L[q][c] = (a_qc - sum_{k<c} L[q][k] L[c][k]) * inv[c]
 *             pivot t = a_qq - sum_k L[q][k]^2, inv[q] = 1/sqrt(t)
 *             y[q] = (-a_qi - sum_k L[q][k] y[k]) * inv[q]
 *             each sum folded left-to-right with fma(-a, b, t)
 *   psi       psi = a_ii; for q: psi = fma(-y[q], y[q], psi)      (Eq. 9 denominator)
 *   back-sub  g[q] = (y[q] - sum_{k>q, descending} L[k][q] g[k]) * inv[q]
 *   exit      psi / psi0 <= eps                                   (Eq. 16)
 *   scale     d = 1/sqrt(psi); G row = (g * d, d)                 (Eqs. 8-9)
 * Build with -ffp-contract=off (no implicit contraction), fma() from libm.
 *
 * Precision.  The set-up (setup_row / oracle_setup_rows / oracle_gradient) is
 * written over `real`: double by default; compiled with -DOR_FP32 (liboracle_f32.so)
 * it is the single-precision set-up of PAPER.md §4.3: A_s = single(A)
 * is the input (the caller rounds A's values to float), every operation above runs
 * in float (fmaf, sqrtf, float division), and the output G = double(G_s) is the
 * exact widening of the float values.  Comparisons against the double constants
 * 1e-30 and eps are made in double (the float operand widened exactly), as on the
 * GPU.  Transpose, apply and PCG exist only in the fp64 build (G is fp64 either way).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENOTSPD 2
#define OR_ENOMEM 3

#define OR_STOP_KMAX 0
#define OR_STOP_CAP 1
#define OR_STOP_NOCAND 2
#define OR_STOP_TOL 3

#ifdef OR_FP32
typedef float real;
#define R_FMA fmaf
#define R_SQRT sqrtf
#define R_ABS fabsf
#else
typedef double real;
#define R_FMA fma
#define R_SQRT sqrt
#define R_ABS fabs
#endif

#define MARK_NONE (-1)
#define MARK_CAND (-2)
#define MARK_SELF (-3)

typedef struct {
    int64_t n;
    const int64_t *rowptr;
    const int32_t *col;
    const real *val;
} or_csr;

typedef struct {
    int32_t j;
    real acc;
} or_cand;

/* total order of P:383-387 + DESIGN.md R5: |acc| descending, then column ascending */
static int cand_cmp(const void *a, const void *b) {
    const or_cand *x = (const or_cand *)a, *y = (const or_cand *)b;
    real ax = R_ABS(x->acc), ay = R_ABS(y->acc);
    if (ax > ay) return -1;
    if (ax < ay) return 1;
    return (x->j < y->j) ? -1 : (x->j > y->j);
}

static int int_cmp(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x < y) ? -1 : (x > y);
}

typedef struct {
    int32_t c;
    real v;
} or_entry;

static int entry_cmp(const void *a, const void *b) {
    const or_entry *x = (const or_entry *)a, *y = (const or_entry *)b;
    return (x->c < y->c) ? -1 : (x->c > y->c);
}

/* value of A(r, c) by scanning row r (plain linear search), +0.0 if absent */
static real a_entry(const or_csr *A, int64_t r, int64_t c) {
    for (int64_t e = A->rowptr[r]; e < A->rowptr[r + 1]; ++e)
        if (A->col[e] == c) return A->val[e];
    return +0.0;
}

typedef struct {
    /* problem */
    or_csr A;
    int32_t nsteps, s, cap;
    double eps;
    const int64_t *rows;
    int64_t nrows;
    int32_t stride, mmax;
    /* outputs */
    int32_t *out_nnz, *out_col;
    double *out_val;
    int32_t *out_steps, *out_reason;
    double *out_psi, *out_margin;
    /* shared state */
    int64_t next;
    pthread_mutex_t lock;
    int status;
    int64_t err_row;
    int32_t err_step;
} or_job;

typedef struct {
    int32_t *mark;   /* n: MARK_* or pattern position */
    int32_t *P;      /* mmax, insertion order */
    int32_t *cand_j; /* candidate list */
    or_cand *cand;
    int64_t cand_cap;
    real *L;         /* mmax*mmax dense row-major (only lower used) */
    real *inv, *y, *g, *arow;
    or_entry *ent;
} or_ws;

/* one row of the set-up; returns OR_OK or OR_ENOTSPD (step in *bad_step) */
static int setup_row(or_job *J, or_ws *W, int64_t idx, int32_t *bad_step) {
    const or_csr *A = &J->A;
    const int64_t i = J->rows[idx];
    const int32_t mmax = J->mmax;
    int32_t *mark = W->mark;
    int32_t m = 0;
    int64_t ncand = 0;
    double *psi_tr = J->out_psi ? J->out_psi + idx * (int64_t)(J->nsteps + 1) : NULL;
    double *mg_tr = J->out_margin ? J->out_margin + idx * (int64_t)J->nsteps : NULL;

    const real a_ii = a_entry(A, i, i);
    const real psi0 = a_ii;     /* identity initial guess: psi_0 = a_ii */
    real psi = psi0;
    int32_t reason = OR_STOP_KMAX, steps = 0;
    mark[i] = MARK_SELF;
    if (psi_tr) psi_tr[0] = (double)psi0;

    for (int32_t k = 1; k <= J->nsteps; ++k) {
        int32_t room = J->s;
        if (J->cap - 1 - m < room) room = J->cap - 1 - m;
        if (room <= 0) { reason = OR_STOP_CAP; break; }

        /* ---- candidate universe (R7): columns j < i of rows P-bar U {i}, minus P-bar */
        for (int64_t t = 0; t < ncand; ++t)
            if (mark[W->cand_j[t]] == MARK_CAND) mark[W->cand_j[t]] = MARK_NONE;
        ncand = 0;
        for (int32_t q = -1; q < m; ++q) {
            int64_t r = (q < 0) ? i : W->P[q];
            for (int64_t e = A->rowptr[r]; e < A->rowptr[r + 1]; ++e) {
                int32_t j = A->col[e];
                if (j >= i || mark[j] != MARK_NONE) continue;
                if (ncand == W->cand_cap) {
                    W->cand_cap *= 2;
                    W->cand_j = (int32_t *)realloc(W->cand_j, W->cand_cap * sizeof(int32_t));
                    W->cand = (or_cand *)realloc(W->cand, W->cand_cap * sizeof(or_cand));
                }
                mark[j] = MARK_CAND;
                W->cand_j[ncand++] = j;
            }
        }

        /* ---- Kaporin gradient, Eq. 15: acc_j = sum_r a_jr gt_ir (gt_ii = 1), row j of A
         *      read in storage (ascending column) order                       */
        int64_t nnz_c = 0;
        for (int64_t t = 0; t < ncand; ++t) {
            int32_t j = W->cand_j[t];
            real acc = +0.0;
            for (int64_t e = A->rowptr[j]; e < A->rowptr[j + 1]; ++e) {
                int32_t r = A->col[e];
                if (r == i) acc = R_FMA(A->val[e], (real)1.0, acc);
                else if (mark[r] >= 0) acc = R_FMA(A->val[e], W->g[mark[r]], acc);
            }
            if (acc != 0.0) { W->cand[nnz_c].j = j; W->cand[nnz_c].acc = acc; ++nnz_c; }
        }
        if (nnz_c == 0) { reason = OR_STOP_NOCAND; break; }

        /* ---- select the top `room` (full sort: plain) */
        qsort(W->cand, (size_t)nnz_c, sizeof(or_cand), cand_cmp);
        int32_t nsel = (nnz_c < room) ? (int32_t)nnz_c : room;
        if (mg_tr) {
            double top = fabs((double)W->cand[0].acc);   /* trace only: in double */
            mg_tr[k - 1] = (nnz_c > nsel) ? (fabs((double)W->cand[nsel - 1].acc) - fabs((double)W->cand[nsel].acc)) / top
                                         : INFINITY;
        }
        int32_t sel[1024];
        for (int32_t t = 0; t < nsel; ++t) sel[t] = W->cand[t].j;
        qsort(sel, (size_t)nsel, sizeof(int32_t), int_cmp);
        for (int32_t t = 0; t < nsel; ++t) { W->P[m + t] = sel[t]; mark[sel[t]] = m + t; }
        m += nsel;

        /* ---- refactor A[P,P] = L L^T from scratch (Eq. 7), forward-solve y = L^-1 (-A[P,i]) */
        for (int32_t q = 0; q < m; ++q) {
            const int64_t pq = W->P[q];
            for (int32_t c = 0; c <= q; ++c) W->arow[c] = +0.0;
            real b = +0.0;
            for (int64_t e = A->rowptr[pq]; e < A->rowptr[pq + 1]; ++e) {
                int32_t c = A->col[e];
                if (c == i) b = A->val[e];
                else if (mark[c] >= 0 && mark[c] <= q) W->arow[mark[c]] = A->val[e];
            }
            real *Lq = W->L + (int64_t)q * mmax;
            for (int32_t c = 0; c < q; ++c) {
                const real *Lc = W->L + (int64_t)c * mmax;
                real t = W->arow[c];
                for (int32_t kk = 0; kk < c; ++kk) t = R_FMA(-Lq[kk], Lc[kk], t);
                Lq[c] = t * W->inv[c];
            }
            real t = W->arow[q];
            for (int32_t kk = 0; kk < q; ++kk) t = R_FMA(-Lq[kk], Lq[kk], t);
            if (!(t > 1e-30)) { *bad_step = k; return OR_ENOTSPD; }
            W->inv[q] = (real)1.0 / R_SQRT(t);
            real ty = -b;
            for (int32_t kk = 0; kk < q; ++kk) ty = R_FMA(-Lq[kk], W->y[kk], ty);
            W->y[q] = ty * W->inv[q];
        }
        /* ---- psi = a_ii - ||y||^2 = a_ii + A[i,P] gt  (Eq. 9 denominator; R3) */
        psi = a_ii;
        for (int32_t q = 0; q < m; ++q) psi = R_FMA(-W->y[q], W->y[q], psi);
        if (!(psi > 0.0)) { *bad_step = k; return OR_ENOTSPD; }
        /* ---- back-substitution gt = L^-T y */
        for (int32_t q = m - 1; q >= 0; --q) {
            real t = W->y[q];
            for (int32_t kk = m - 1; kk > q; --kk) t = R_FMA(-W->L[(int64_t)kk * mmax + q], W->g[kk], t);
            W->g[q] = t * W->inv[q];
        }
        steps = k;
        if (psi_tr) psi_tr[k] = (double)psi;
        /* ---- exit test, Eq. 16 (literal ratio; R4) */
        if (psi / psi0 <= J->eps) { reason = OR_STOP_TOL; break; }
    }

    /* ---- scaling Eqs. 8-9 (with the square root, R1) and output sorted by column */
    const real d = (real)1.0 / R_SQRT(psi);
    for (int32_t q = 0; q < m; ++q) { W->ent[q].c = W->P[q]; W->ent[q].v = W->g[q] * d; }
    W->ent[m].c = (int32_t)i;
    W->ent[m].v = d;
    qsort(W->ent, (size_t)(m + 1), sizeof(or_entry), entry_cmp);
    J->out_nnz[idx] = m + 1;
    for (int32_t q = 0; q <= m; ++q) {
        J->out_col[idx * J->stride + q] = W->ent[q].c;
        J->out_val[idx * J->stride + q] = (double)W->ent[q].v;   /* G = double(G_s): exact */
    }
    J->out_steps[idx] = steps;
    J->out_reason[idx] = reason;

    /* reset marks */
    for (int64_t t = 0; t < ncand; ++t)
        if (mark[W->cand_j[t]] == MARK_CAND) mark[W->cand_j[t]] = MARK_NONE;
    for (int32_t q = 0; q < m; ++q) mark[W->P[q]] = MARK_NONE;
    mark[i] = MARK_NONE;
    return OR_OK;
}

static void *worker(void *arg) {
    or_job *J = (or_job *)arg;
    or_ws W;
    memset(&W, 0, sizeof W);
    int32_t mm = J->mmax + 1;
    W.mark = (int32_t *)malloc(J->A.n * sizeof(int32_t));
    W.P = (int32_t *)malloc(mm * sizeof(int32_t));
    W.cand_cap = 1024;
    W.cand_j = (int32_t *)malloc(W.cand_cap * sizeof(int32_t));
    W.cand = (or_cand *)malloc(W.cand_cap * sizeof(or_cand));
    W.L = (real *)malloc((size_t)mm * mm * sizeof(real));
    W.inv = (real *)malloc(mm * sizeof(real));
    W.y = (real *)malloc(mm * sizeof(real));
    W.g = (real *)malloc(mm * sizeof(real));
    W.arow = (real *)malloc(mm * sizeof(real));
    W.ent = (or_entry *)malloc(mm * sizeof(or_entry));
    if (!W.mark || !W.P || !W.cand_j || !W.cand || !W.L || !W.inv || !W.y || !W.g || !W.arow || !W.ent) {
        pthread_mutex_lock(&J->lock);
        J->status = OR_ENOMEM;
        pthread_mutex_unlock(&J->lock);
    } else {
        for (int64_t t = 0; t < J->A.n; ++t) W.mark[t] = MARK_NONE;
        for (;;) {
            pthread_mutex_lock(&J->lock);
            int64_t idx = (J->status == OR_OK && J->next < J->nrows) ? J->next++ : -1;
            pthread_mutex_unlock(&J->lock);
            if (idx < 0) break;
            int32_t bad = 0;
            int rc = setup_row(J, &W, idx, &bad);
            if (rc != OR_OK) {
                pthread_mutex_lock(&J->lock);
                if (J->status == OR_OK || J->rows[idx] < J->err_row) {
                    J->status = rc;
                    J->err_row = J->rows[idx];
                    J->err_step = bad;
                }
                pthread_mutex_unlock(&J->lock);
            }
        }
    }
    free(W.mark); free(W.P); free(W.cand_j); free(W.cand); free(W.L);
    free(W.inv); free(W.y); free(W.g); free(W.arow); free(W.ent);
    return NULL;
}

/*
 * oracle_setup_rows: aFSAI rows `rows[0..nrows)` of the full symmetric CSR A.
 * Output per requested row t: out_nnz[t] entries of G (sorted columns, the
 * diagonal included) at out_col/out_val[t*stride ...]; steps taken; stop
 * reason (0 kmax, 1 cap, 2 no candidates, 3 tolerance); psi per step
 * (out_psi[t*(nsteps+1) + k], k = 0..steps) and the selection margin
 * (out_margin[t*nsteps + k-1]); both optional (NULL).
 * Returns 0, or 2 (not SPD; err_row / err_step set to the lowest failing row).
 */
int oracle_setup_rows(int64_t n, const int64_t *rowptr, const int32_t *col, const real *val,
                      int32_t nsteps, int32_t s, double eps, int32_t max_row_nnz,
                      const int64_t *rows, int64_t nrows, int32_t stride,
                      int32_t *out_nnz, int32_t *out_col, double *out_val,
                      int32_t *out_steps, int32_t *out_reason, double *out_psi, double *out_margin,
                      int64_t *err_row, int32_t *err_step, int32_t nthreads) {
    if (n < 0 || nsteps < 0 || s < 1 || !(eps >= 0.0 && eps < 1.0) || max_row_nnz < 1) return OR_EINVAL;
    int64_t mmax = (int64_t)nsteps * s;
    if (mmax > max_row_nnz - 1) mmax = max_row_nnz - 1;
    if (mmax > n) mmax = n;
    if (stride < mmax + 1 || s > 1024) return OR_EINVAL;
    or_job J;
    memset(&J, 0, sizeof J);
    J.A.n = n; J.A.rowptr = rowptr; J.A.col = col; J.A.val = val;
    J.nsteps = nsteps; J.s = s; J.cap = max_row_nnz; J.eps = eps;
    J.rows = rows; J.nrows = nrows; J.stride = stride; J.mmax = (int32_t)mmax;
    J.out_nnz = out_nnz; J.out_col = out_col; J.out_val = out_val;
    J.out_steps = out_steps; J.out_reason = out_reason; J.out_psi = out_psi; J.out_margin = out_margin;
    J.status = OR_OK; J.err_row = INT64_MAX;
    pthread_mutex_init(&J.lock, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 512) nthreads = 512;
    pthread_t th[512];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &J);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&J.lock);
    if (J.status != OR_OK && err_row) { *err_row = J.err_row; *err_step = J.err_step; }
    return J.status;
}

#ifndef OR_FP32
/* Exact transpose: counting sort by column, stable in the row index, so
 * each row of G^T lists its entries in ascending original row. */
int oracle_transpose(int64_t n, const int64_t *rowptr, const int32_t *col, const double *val,
                     int64_t *t_rowptr, int32_t *t_col, double *t_val) {
    for (int64_t j = 0; j <= n; ++j) t_rowptr[j] = 0;
    for (int64_t e = 0; e < rowptr[n]; ++e) t_rowptr[col[e] + 1]++;
    for (int64_t j = 0; j < n; ++j) t_rowptr[j + 1] += t_rowptr[j];
    int64_t *cur = (int64_t *)malloc((n + 1) * sizeof(int64_t));
    if (!cur) return OR_ENOMEM;
    memcpy(cur, t_rowptr, (n + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            int64_t p = cur[col[e]]++;
            t_col[p] = (int32_t)i;
            t_val[p] = val[e];
        }
    free(cur);
    return OR_OK;
}

/* y = M x, each row summed in storage order: y_i = ((m_i1 x_1 + m_i2 x_2) + ...) */
static void spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v, const double *x, double *y) {
    for (int64_t i = 0; i < n; ++i) {
        double t = 0.0;
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) t = t + v[e] * x[ci[e]];
        y[i] = t;
    }
}

static double dot(int64_t n, const double *a, const double *b) {
    double t = 0.0;
    for (int64_t i = 0; i < n; ++i) t = t + a[i] * b[i];
    return t;
}

/* z = G^T (G r), Eq. 1, two sparse products; tmp: n doubles */
int oracle_apply(int64_t n, const int64_t *g_rp, const int32_t *g_ci, const double *g_v,
                 const int64_t *t_rp, const int32_t *t_ci, const double *t_v,
                 const double *r, double *z, double *tmp) {
    spmv(n, g_rp, g_ci, g_v, r, tmp);
    spmv(n, t_rp, t_ci, t_v, tmp, z);
    return OR_OK;
}

/*
 * PCG (R12): x0 = 0, r = b, z = M^-1 r, p = z;
 *   q = A p; alpha = (r,z)/(p,q); x += alpha p; r -= alpha q;
 *   stop when ||r||_2 / ||b||_2 <= tol (checked after the r update);
 *   z = M^-1 r; beta = (r,z)_new/(r,z)_old; p = z + beta p.
 * M^-1 = G^T G (Eq. 1).  If g_rp == NULL, M = I (plain CG).
 * Returns 0 (converged) or 6 (not converged in max_iters); *iters, *relres set;
 * res_hist (optional, max_iters+1) gets ||r_k||/||b||.
 */
int oracle_pcg(int64_t n, const int64_t *a_rp, const int32_t *a_ci, const double *a_v,
               const int64_t *g_rp, const int32_t *g_ci, const double *g_v,
               const int64_t *t_rp, const int32_t *t_ci, const double *t_v,
               const double *b, double *x, double tol, int32_t max_iters,
               int32_t *iters, double *relres, double *res_hist) {
    double *r = (double *)malloc(n * sizeof(double));
    double *z = (double *)malloc(n * sizeof(double));
    double *p = (double *)malloc(n * sizeof(double));
    double *q = (double *)malloc(n * sizeof(double));
    double *tmp = (double *)malloc(n * sizeof(double));
    if (!r || !z || !p || !q || !tmp) { free(r); free(z); free(p); free(q); free(tmp); return OR_ENOMEM; }
    for (int64_t k = 0; k < n; ++k) { x[k] = 0.0; r[k] = b[k]; }
    const double bnorm = sqrt(dot(n, b, b));
    int rc = 6;
    *iters = 0;
    *relres = 0.0;
    if (res_hist) res_hist[0] = 1.0;
    if (bnorm == 0.0) { rc = 0; goto done; }
    if (g_rp) oracle_apply(n, g_rp, g_ci, g_v, t_rp, t_ci, t_v, r, z, tmp);
    else memcpy(z, r, n * sizeof(double));
    memcpy(p, z, n * sizeof(double));
    double rz = dot(n, r, z);
    *relres = 1.0;
    for (int32_t it = 1; it <= max_iters; ++it) {
        spmv(n, a_rp, a_ci, a_v, p, q);
        const double alpha = rz / dot(n, p, q);
        for (int64_t k = 0; k < n; ++k) { x[k] = x[k] + alpha * p[k]; r[k] = r[k] - alpha * q[k]; }
        const double rel = sqrt(dot(n, r, r)) / bnorm;
        *iters = it;
        *relres = rel;
        if (res_hist) res_hist[it] = rel;
        if (rel <= tol) { rc = 0; break; }
        if (g_rp) oracle_apply(n, g_rp, g_ci, g_v, t_rp, t_ci, t_v, r, z, tmp);
        else memcpy(z, r, n * sizeof(double));
        const double rz_new = dot(n, r, z);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int64_t k = 0; k < n; ++k) p[k] = z[k] + beta * p[k];
    }
done:
    free(r); free(z); free(p); free(q); free(tmp);
    return rc;
}

/*
 * oracle_gradient: the Kaporin-gradient accumulator of Eq. 15 for
 * row i with a given off-diagonal pattern P[0..m) (insertion order) and values
 * gt[0..m): for every candidate j (j < i, j not in P, j a column of some row in
 * P U {i}) returns acc_j = sum_{r in P U {i}} a_jr gt_r (gt_i = 1), folded as
 * in setup_row; d psi / d gt_j = 2 acc_j.  Candidates with acc == 0 are KEPT
 * here (so tests can see them).  Output ascending in j; returns the count, or
 * -1 if max_out is too small.
 */
int64_t oracle_gradient(int64_t n, const int64_t *rowptr, const int32_t *col, const double *val,
                        int64_t i, int32_t m, const int32_t *P, const double *gt,
                        int32_t *out_j, double *out_acc, int64_t max_out) {
    int32_t *mark = (int32_t *)malloc(n * sizeof(int32_t));
    if (!mark) return -1;
    for (int64_t t = 0; t < n; ++t) mark[t] = MARK_NONE;
    for (int32_t q = 0; q < m; ++q) mark[P[q]] = q;
    mark[i] = MARK_SELF;
    int64_t cnt = 0;
    for (int64_t j = 0; j < i; ++j) {
        if (mark[j] != MARK_NONE) continue;
        int in_universe = 0;
        for (int32_t q = -1; q < m && !in_universe; ++q) {
            int64_t r = (q < 0) ? i : P[q];
            for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e)
                if (col[e] == j) { in_universe = 1; break; }
        }
        if (!in_universe) continue;
        double acc = +0.0;
        for (int64_t e = rowptr[j]; e < rowptr[j + 1]; ++e) {
            int32_t r = col[e];
            if (r == i) acc = fma(val[e], 1.0, acc);
            else if (mark[r] >= 0) acc = fma(val[e], gt[mark[r]], acc);
        }
        if (cnt == max_out) { free(mark); return -1; }
        out_j[cnt] = (int32_t)j;
        out_acc[cnt] = acc;
        ++cnt;
    }
    free(mark);
    return cnt;
}
#endif /* !OR_FP32 */
