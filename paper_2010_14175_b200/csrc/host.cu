// host.cu -- the C ABI of include/afsai.h: contexts, afsai_setup (validate ->
// per-row kernel -> assemble G -> transpose), afsai_apply, afsai_pcg and the
// factor accessors.  Every step of the path runs in this library's kernels;
// host code only sizes buffers, launches and checks status.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "afsai_internal.h"
#include "assemble.h"
#include "dist.h"
#include "setup_kernel.h"
#include "spmv.h"

namespace afsai {

int set_status(afsai_status_t *st, int code, const std::string &msg, int64_t row, int32_t step) {
    if (st) {
        st->code = code;
        st->row = row;
        st->step = step;
        std::snprintf(st->msg, sizeof st->msg, "%s", msg.c_str());
    }
    return code;
}

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// A device view of a caller CSR: device arrays used as-is, host arrays staged.
int stage_csr(afsai_ctx_t ctx, const afsai_csr_t *A, DeviceCsr *out, afsai_status_t *status) {
    out->n_rows = A->n_rows;
    out->n_cols = A->n_cols;
    out->row_begin = A->row_begin;
    out->nnz = A->nnz;
    const bool dev = is_device_ptr(A->rowptr);
    if (dev != is_device_ptr(A->col) || (A->nnz > 0 && dev != is_device_ptr(A->val)))
        return set_status(status, AFSAI_EINVAL, "rowptr/col/val must all be host or all be device memory");
    if (dev) {
        out->rowptr = A->rowptr;
        out->col = A->col;
        out->val = A->val;
        out->staged = false;
        // base = rowptr[0] and the end offset (read back; two tiny copies)
        int64_t last = 0;
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&out->base, A->rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&last, A->rowptr + A->n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                       ctx->stream));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        if (last - out->base != A->nnz)
            return set_status(status, AFSAI_EINVAL, "rowptr[n_rows] - rowptr[0] != nnz");
        return AFSAI_OK;
    }
    if (A->rowptr[A->n_rows] - A->rowptr[0] != A->nnz)
        return set_status(status, AFSAI_EINVAL, "rowptr[n_rows] - rowptr[0] != nnz");
    out->base = A->rowptr[0];
    out->staged = true;
    AFSAI_CUDA_TRY(out->b_rowptr.alloc((A->n_rows + 1) * sizeof(int64_t), ctx->stream));
    AFSAI_CUDA_TRY(out->b_col.alloc(std::max<int64_t>(A->nnz, 1) * sizeof(int32_t), ctx->stream));
    AFSAI_CUDA_TRY(out->b_val.alloc(std::max<int64_t>(A->nnz, 1) * sizeof(double), ctx->stream));
    AFSAI_CUDA_TRY(cudaMemcpyAsync(out->b_rowptr.p, A->rowptr, (A->n_rows + 1) * sizeof(int64_t),
                                   cudaMemcpyHostToDevice, ctx->stream));
    if (A->nnz > 0) {
        AFSAI_CUDA_TRY(cudaMemcpyAsync(out->b_col.p, A->col, A->nnz * sizeof(int32_t),
                                       cudaMemcpyHostToDevice, ctx->stream));
        AFSAI_CUDA_TRY(cudaMemcpyAsync(out->b_val.p, A->val, A->nnz * sizeof(double),
                                       cudaMemcpyHostToDevice, ctx->stream));
    }
    out->rowptr = out->b_rowptr.as<int64_t>();
    out->col = out->b_col.as<int32_t>();
    out->val = out->b_val.as<double>();
    // staged copies keep the caller's rowptr values (relative to base)
    return AFSAI_OK;
}

int grid_stream(afsai_ctx_t ctx) { return ctx->num_sms * 8; }

static float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

// Validate A (a0): structure, diagonal, finiteness; returns max row length.
int validate_csr(afsai_ctx_t ctx, const DeviceCsr &A, int64_t *max_row_len, afsai_status_t *status) {
    NvtxRange nv("afsai validate A");
    DevBuf err;
    AFSAI_CUDA_TRY(err.alloc(2 * sizeof(unsigned long long), ctx->stream));
    AFSAI_CUDA_TRY(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), ctx->stream));
    AFSAI_CUDA_TRY(cudaMemsetAsync(err.as<unsigned long long>() + 1, 0, sizeof(unsigned long long), ctx->stream));
    const int grid = std::max<int64_t>(1, std::min<int64_t>((A.n_rows * 32 + 255) / 256, grid_stream(ctx)));
    KTimer kt(ctx, AFSAI_K_ASSEMBLE);
    validate_rows_kernel<<<grid, 256, 0, ctx->stream>>>(A.rowptr, A.col, A.val, A.base, A.n_rows, A.row_begin,
                                                        A.n_cols, err.as<unsigned long long>());
    row_len_max_kernel<<<grid, 256, 0, ctx->stream>>>(A.rowptr, A.n_rows, err.as<unsigned long long>() + 1);
    ctx->launches += 2;
    // bitwise symmetry (contract C1: the hit-list kernels read a_jr from row r) is
    // checked by default (one binary search per entry; pairs inside this rank's
    // rows); AFSAI_VALIDATE=0 skips it
    const char *v = std::getenv("AFSAI_VALIDATE");
    if (!(v && v[0] == '0')) {
        symmetry_kernel<<<grid, 256, 0, ctx->stream>>>(A.rowptr, A.col, A.val, A.base, A.n_rows, A.row_begin,
                                                       err.as<unsigned long long>());
        ctx->launches += 1;
    }
    AFSAI_CUDA_TRY(cudaGetLastError());
    unsigned long long h[2];
    AFSAI_CUDA_TRY(cudaMemcpyAsync(h, err.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (h[0] != ~0ull) {
        static const char *why[] = {"",
                                    "decreasing rowptr",
                                    "column out of range",
                                    "columns not strictly increasing",
                                    "non-finite value",
                                    "diagonal not positive",
                                    "diagonal missing",
                                    "not bitwise symmetric"};
        const int r = (int)(h[0] & 0xff);
        return set_status(status, AFSAI_EINVAL, std::string("invalid A: ") + why[r < 8 ? r : 0],
                          (int64_t)(h[0] >> 8));
    }
    *max_row_len = (int64_t)h[1];
    return AFSAI_OK;
}

static int ilog2(int x) {
    int l = 0;
    while ((1 << l) < x) ++l;
    return l;
}

// Runs the per-row kernel over global rows [row_lo, row_lo + nrows) of a matrix
// whose rows [a_lo, a_hi) are in A_ext; writes scratch indexed by row - out_base.
int run_rows(afsai_ctx_t ctx, const DeviceCsr &Aext, int64_t a_lo, int64_t a_hi, int64_t row_lo, int64_t nrows,
             const afsai_params_t &p, int32_t mmax, int64_t max_row_len, SetupWork &W, afsai_setup_stats_t *stats,
             afsai_status_t *status) {
    // Kernel plan.  Short rows (stencils: max row length <= 9) use the hit-list
    // kernel, whose gradient needs no loads of candidate rows; everything else and
    // every retry uses the general kernel.  Lanes per row: 16 up to mmax 96, else 32.
    // The candidate table starts small (stencil universes are small); rows that
    // overflow an on-chip table are retried with 4x larger tables.
    // AFSAI_LPR / AFSAI_TABLE / AFSAI_HITS=0 override (experiments).
    NvtxRange nv("afsai set-up rows kernel");
    // the kernel instances of the set-up precision (afsai::dp fp64, afsai::sp fp32)
    const bool f32 = p.precision == AFSAI_PREC_FP32;
#ifdef AFSAI_NO_FP32  // a build without the afsai::sp instances (build.py fp32=False, the debug build)
    if (f32) return set_status(status, AFSAI_ELIMIT, "this build of the library has no fp32 set-up kernels");
    namespace kp = dp;
    auto scan_kernel_for = kp::scan_kernel_for;
    auto scan_row_bytes = kp::scan_row_bytes;
    auto hits_kernel_for = kp::hits_kernel_for;
    auto hits_row_bytes = kp::hits_row_bytes;
    auto lockstep_kernel_for = kp::lockstep_kernel_for;
    auto lockstep_row_bytes = kp::lockstep_row_bytes;
    auto prow_kernel_for = kp::prow_kernel_for;
    auto prow_row_bytes = kp::prow_row_bytes;
#else
    auto scan_kernel_for = f32 ? sp::scan_kernel_for : dp::scan_kernel_for;
    auto scan_row_bytes = f32 ? sp::scan_row_bytes : dp::scan_row_bytes;
    auto hits_kernel_for = f32 ? sp::hits_kernel_for : dp::hits_kernel_for;
    auto hits_row_bytes = f32 ? sp::hits_row_bytes : dp::hits_row_bytes;
    auto lockstep_kernel_for = f32 ? sp::lockstep_kernel_for : dp::lockstep_kernel_for;
    auto lockstep_row_bytes = f32 ? sp::lockstep_row_bytes : dp::lockstep_row_bytes;
    auto prow_kernel_for = f32 ? sp::prow_kernel_for : dp::prow_kernel_for;
    auto prow_row_bytes = f32 ? sp::prow_row_bytes : dp::prow_row_bytes;
#endif
    DevBuf val32;  // A_s = single(A) (fp32 set-up)
    if (f32) {
        AFSAI_CUDA_TRY(val32.alloc(std::max<int64_t>(Aext.nnz, 1) * sizeof(float), ctx->stream));
        DevBuf cerr;
        AFSAI_CUDA_TRY(cerr.alloc(sizeof(unsigned long long), ctx->stream));
        AFSAI_CUDA_TRY(cudaMemsetAsync(cerr.p, 0xff, sizeof(unsigned long long), ctx->stream));
        const int grid = std::max<int64_t>(1, std::min<int64_t>((Aext.n_rows * 32 + 255) / 256, grid_stream(ctx)));
        {
            KTimer kt(ctx, AFSAI_K_ASSEMBLE);
            cast_rows_f32_kernel<<<grid, 256, 0, ctx->stream>>>(Aext.rowptr, Aext.col, Aext.val, Aext.base,
                                                                 Aext.n_rows, Aext.row_begin, val32.as<float>(),
                                                                 cerr.as<unsigned long long>());
        }
        ctx->launches += 1;
        AFSAI_CUDA_TRY(cudaGetLastError());
        unsigned long long ce = 0;
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&ce, cerr.p, sizeof ce, cudaMemcpyDeviceToHost, ctx->stream));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        if (ce != ~0ull)
            return set_status(status, AFSAI_EINVAL,
                              "A_s = single(A) overflows fp32 or loses a positive diagonal (fp32 set-up)",
                              (int64_t)ce);
    }
    int lpr = mmax <= 96 ? 16 : 32;
    if (const char *e = std::getenv("AFSAI_LPR")) {
        const int l = std::atoi(e);
        if (l == 32 || (l == 16 && mmax <= 96)) lpr = l;
    }
    // one entry per lane at 16 lanes per row; hits may record int32 entry indices
    bool hits = max_row_len <= 9 && Aext.nnz < INT32_MAX;
    if (const char *e = std::getenv("AFSAI_HITS")) hits = hits && std::atoi(e) != 0;
    // lockstep: ls_lpr lanes per row, 32/ls_lpr rows per warp (rows <= ls_lpr entries, s <= 4)
    int ls_lpr = 16;
    if (const char *e = std::getenv("AFSAI_LOCKSTEP_LPR")) ls_lpr = std::atoi(e) == 8 ? 8 : 16;
    bool lockstep = hits && max_row_len <= ls_lpr && p.s <= 4;
    if (const char *e = std::getenv("AFSAI_LOCKSTEP")) lockstep = lockstep && std::atoi(e) != 0;
    const int lpr0 = lpr;
    const int hc = max_row_len <= 7 ? 6 : 8;
    // universe <= (pattern rows) x (row length); observed ~ (mmax+1) * len / 10
    // for FE (700 of 91 x 81), ~2.2 (mmax+1) for 7-point stencils
    int H = 1 << std::max(6, ilog2((int)std::min<int64_t>(1 << 13, std::max<int64_t>(
                                     4 * (mmax + 1), (int64_t)(mmax + 1) * max_row_len / 6))));
    if (hits) H = 1 << std::max(6, ilog2(3 * (mmax + 1)));
    if (const char *e = std::getenv("AFSAI_TABLE")) {
        const int h = std::atoi(e);
        if (h >= 64 && (h & (h - 1)) == 0) H = h;
    }
    int cact = 56;  // active candidate slots (7-point interior rows peak near 50)
    // the hit-list kernels encode active slot aa as int8 state -2 - aa
    constexpr int kMaxCact = 126;
    // the probe's growth cap on the active candidate slots (A/B knob)
    int cact_cap = kMaxCact;
    if (const char *e = std::getenv("AFSAI_CACT_MAX")) cact_cap = std::max(8, std::min(kMaxCact, std::atoi(e)));
    // pattern-row kernel for long rows (FE): universe ~ (mmax+1) * len / 10 keys,
    // table at most 3/4 full; lists hold every pattern row (no overflow)
    // (its row descriptors hold entry offsets relative to row i as int32)
    bool prow = !hits && prow_kernel_for(mmax, p.s, max_row_len) != nullptr && Aext.nnz < INT32_MAX;
    if (const char *e = std::getenv("AFSAI_PROW")) prow = prow && std::atoi(e) != 0;
    const int lcap = (int)std::min<int64_t>(1 << 15, (int64_t)(mmax + 1) * max_row_len);
    if (prow) {
        const int64_t u = std::max<int64_t>(48, (int64_t)(mmax + 1) * max_row_len / 10);
        H = 1 << ilog2((int)std::min<int64_t>(1 << 14, (u * 4 + 2) / 3));
        if (const char *e = std::getenv("AFSAI_TABLE")) {
            const int h = std::atoi(e);
            if (h >= 64 && (h & (h - 1)) == 0) H = h;
        }
        if (prow_row_bytes(H, mmax, p.s, lcap) > 200 * 1024) prow = false;
    }
    SetupKArgs a{};
    a.rowptr = Aext.rowptr;
    a.col = Aext.col;
    a.val = Aext.val;
    a.val32 = f32 ? val32.as<float>() : nullptr;
    a.base = Aext.base;
    a.nnz = Aext.nnz;
    a.a_lo = a_lo;
    a.a_hi = a_hi;
    a.rows = nullptr;
    a.row_lo = row_lo;
    a.nrows = nrows;
    a.nsteps = p.nsteps;
    a.s = p.s;
    a.cap = p.max_row_nnz;
    a.mmax = mmax;
    a.eps = p.eps;
    a.out_base = row_lo;
    a.stride = mmax + 1;
    a.scol = W.scol.as<int32_t>();
    a.sval = W.sval.as<double>();
    a.nnz_row = W.nnz_row.as<int32_t>();
    a.steps = W.steps;
    a.reason = W.reason;
    a.err = W.err.as<unsigned long long>();
    a.retry_rows = W.retry.as<int64_t>();
    a.retry_count = W.retry_count.as<int32_t>();
    a.work = W.work.as<unsigned long long>();
    a.counters = W.counters.as<unsigned long long>();
    a.lcap = lcap;
    bool first = true;
    DevBuf lu_buf;  // the pattern-row kernel's lu lists (global memory, one region per warp)
    // One pass of the current plan over rows (device list) or [row_lo, row_lo+n);
    // returns the number of rows that overflowed an on-chip table in *rc.
    unsigned long long why = 0;  // overflow reasons of the last pass (lockstep kernel): 1 table, 2 slots, 4 hits
    auto pass = [&](const int64_t *rows, int64_t n, int32_t *rc) -> int {
        if (H > (1 << 15)) return set_status(status, AFSAI_ELIMIT, "candidate table would exceed 32768 slots");
        a.H = H;
        a.log2H = ilog2(H);
        a.cact = cact;
        a.rows = rows;
        a.nrows = n;
        SetupKernFn f = nullptr;
        bool ls = false;
        if (hits && lockstep) {
            f = lockstep_kernel_for(ls_lpr, mmax, p.s, hc);
            if (f) { lpr = ls_lpr; ls = true; }
        }
        if (!f && prow) {
            f = prow_kernel_for(mmax, p.s, max_row_len);
            lpr = 32;
        }
        if (!f) {
            lpr = lpr0;
            f = hits ? hits_kernel_for(lpr, mmax, p.s, hc) : scan_kernel_for(lpr, mmax, p.s);
        }
        if (!f) return set_status(status, AFSAI_ELIMIT, "no kernel instance for this pattern size");
        const int64_t rb = ls ? lockstep_row_bytes(H, mmax, p.s, cact, hc)
                           : hits ? hits_row_bytes(H, mmax, p.s, cact, hc)
                           : prow ? prow_row_bytes(H, mmax, p.s, lcap)
                                  : scan_row_bytes(H, mmax, p.s);
        a.warp_smem = (int32_t)rb;
        const int rpw = 32 / lpr;  // rows per warp
        if (rb * rpw > 200 * 1024) return set_status(status, AFSAI_ELIMIT, "a warp's rows exceed shared memory");
        // CTA size (1..8 warps) maximising the rows resident per SM
        int wpc = 1, occ = 0, best = -1;
        cudaFuncAttributes fa;
        AFSAI_CUDA_TRY(cudaFuncGetAttributes(&fa, (const void *)f));
        const int wmax = std::max(1, std::min(8, fa.maxThreadsPerBlock / 32));
        for (int wc = 1; wc <= wmax; ++wc) {
            const size_t sm_ = (size_t)rb * wc * rpw;
            if (sm_ > 227 * 1024) break;
            if (cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_) !=
                cudaSuccess) { cudaGetLastError(); break; }
            int o = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, (const void *)f, wc * 32, sm_) != cudaSuccess) {
                cudaGetLastError();
                break;
            }
            if (o * wc > best) { best = o * wc; wpc = wc; occ = o; }
        }
        const int rows_per_cta = wpc * rpw;
        const size_t smem = (size_t)rb * rows_per_cta;
        AFSAI_CUDA_TRY(cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        occ = std::max(1, occ);
        int64_t grid = (int64_t)ctx->num_sms * occ;
        grid = std::max<int64_t>(1, std::min<int64_t>(grid, (n + rows_per_cta - 1) / rows_per_cta));
        if (f == prow_kernel_for(mmax, p.s, max_row_len)) {  // per-warp lu lists in global memory
            const size_t need = (size_t)grid * rows_per_cta * (size_t)lcap * sizeof(int16_t);
            if (lu_buf.bytes < need) AFSAI_CUDA_TRY(lu_buf.alloc(need, ctx->stream));
            a.lu_global = lu_buf.as<int16_t>();
        }
        if (first) {
            stats->table_size = H;
            stats->rows_per_cta = rows_per_cta;
            stats->plan = (hits && lockstep) ? AFSAI_PLAN_LOCKSTEP : prow ? AFSAI_PLAN_PROW
                                                             : hits ? AFSAI_PLAN_HITS : AFSAI_PLAN_SCAN;
            stats->lanes_per_row = lpr;
            stats->value_bytes = f32 ? 4 : 8;
        }
        AFSAI_CUDA_TRY(cudaMemsetAsync(W.work.p, 0, sizeof(unsigned long long), ctx->stream));
        AFSAI_CUDA_TRY(cudaMemsetAsync(W.retry_count.p, 0, sizeof(int32_t), ctx->stream));
        AFSAI_CUDA_TRY(cudaMemsetAsync(W.counters.as<unsigned long long>() + 20, 0, sizeof(unsigned long long),
                                       ctx->stream));
        if (std::getenv("AFSAI_DEBUG_PLAN"))
            std::fprintf(stderr,
                         "[afsai rank %d] pass: kernel=%s rows=%lld list=%d H=%d cact=%d lpr=%d rb=%lld "
                         "rows/cta=%d grid=%lld a_lo=%lld a_hi=%lld row_lo=%lld base=%lld\n",
                         ctx->rank, (hits && lockstep) ? "lockstep" : prow ? "prow" : hits ? "hits" : "scan",
                         (long long)n, rows != nullptr, H, cact, lpr, (long long)rb, rows_per_cta, (long long)grid,
                         (long long)a.a_lo, (long long)a.a_hi, (long long)a.row_lo, (long long)a.base);
        {
            KTimer kt(ctx, AFSAI_K_SETUP_ROWS);
            f<<<(unsigned)grid, rows_per_cta * lpr, smem, ctx->stream>>>(a);
            AFSAI_CUDA_TRY(cudaGetLastError());
        }
        ctx->launches += 1;
        AFSAI_CUDA_TRY(cudaMemcpyAsync(rc, W.retry_count.p, sizeof *rc, cudaMemcpyDeviceToHost, ctx->stream));
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&why, W.counters.as<unsigned long long>() + 20, sizeof why,
                                       cudaMemcpyDeviceToHost, ctx->stream));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        return AFSAI_OK;
    };
    // Table-size probe for the hit-list plans: the stencil's universe depends on
    // the coefficients (anisotropy spreads the pattern), so a strided sample of
    // rows is run first; while more than 1% of it overflows, table and active
    // candidate slots double (the sample's results are recomputed by the main pass).
    const bool probe_env = std::getenv("AFSAI_TABLE") == nullptr && std::getenv("AFSAI_NOPROBE") == nullptr;
    if (hits && probe_env && nrows >= 32768) {
        const int64_t ns = 2048, stride = nrows / ns;
        std::vector<int64_t> hs((size_t)ns);
        for (int64_t t = 0; t < ns; ++t) hs[(size_t)t] = row_lo + t * stride;
        DevBuf sample;
        AFSAI_CUDA_TRY(sample.alloc(ns * sizeof(int64_t), ctx->stream));
        AFSAI_CUDA_TRY(cudaMemcpyAsync(sample.p, hs.data(), ns * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        for (int it = 0; it < 3; ++it) {
            int32_t rc = 0;
            const int r = pass(sample.as<int64_t>(), ns, &rc);
            if (r != AFSAI_OK) return r;
            first = false;
            if (rc * 100 <= ns) break;
            // grow what overflowed (the lockstep kernel reports why; others: both)
            int nH = H, nC = cact;
            if (!(hits && lockstep) || why == 0) why = 3;
            if (why & 1) nH = 2 * H;
            if (why & 2) nC = std::min(cact_cap, cact + std::max(8, cact / 2));
            if (nH == H && nC == cact) break;  // hit lists full: the retries take those rows
            if (hits_row_bytes(nH, mmax, p.s, nC, hc) * 2 > 200 * 1024) break;
            H = nH;
            cact = nC;
        }
        AFSAI_CUDA_TRY(cudaMemsetAsync(W.counters.p, 0, 32 * sizeof(unsigned long long), ctx->stream));
        AFSAI_CUDA_TRY(cudaMemsetAsync(W.err.p, 0xff, sizeof(unsigned long long), ctx->stream));
        first = true;
    }
    int64_t todo = nrows;
    DevBuf retry_in;
    int32_t retried_total = 0;
    const int64_t *rows = nullptr;
    while (todo > 0) {
        int32_t rc = 0;
        const int r = pass(rows, todo, &rc);
        if (r != AFSAI_OK) return r;
        todo = rc;
        if (rc > 0 && rows == nullptr) {  // the first pass's overflow list: every retried row
            AFSAI_CUDA_TRY(W.retried.alloc(rc * sizeof(int64_t), ctx->stream));
            AFSAI_CUDA_TRY(cudaMemcpyAsync(W.retried.p, W.retry.p, rc * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                                           ctx->stream));
            W.n_retried = rc;
        }
        if (rc > 0) {
            retried_total += rc;
            AFSAI_CUDA_TRY(retry_in.alloc(rc * sizeof(int64_t), ctx->stream));
            AFSAI_CUDA_TRY(cudaMemcpyAsync(retry_in.p, W.retry.p, rc * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                                           ctx->stream));
            rows = retry_in.as<int64_t>();
            if (prow && prow_row_bytes(2 * H, mmax, p.s, lcap) <= 200 * 1024) {
                H *= 2;  // pattern-row kernel with a larger table
            } else if (hits && lockstep && 2 * cact <= kMaxCact &&
                       hits_row_bytes(2 * H, mmax, p.s, 2 * cact, hc) * 2 <= 200 * 1024) {
                H *= 2;  // hit-list kernel with a larger table and more candidate slots
                cact *= 2;
            } else {
                if (prow) H = 1 << std::max(6, ilog2((int)std::min<int64_t>(
                                  1 << 13, std::max<int64_t>(4 * (mmax + 1), (int64_t)(mmax + 1) * max_row_len / 6))));
                prow = false;
                H *= 4;
                hits = false;  // retries use the general kernel
            }
        }
        first = false;
    }
    stats->retried_rows += retried_total;
    return AFSAI_OK;
}

}  // namespace afsai

// One library-owned pool per device, shared by the contexts on that device and
// trimmed to zero when the last of them is destroyed (the device's default pool,
// which other libraries use, is left alone).
namespace {
constexpr int kMaxDev = 64;
std::mutex g_pool_mu;
cudaMemPool_t g_pool[kMaxDev] = {};
int g_pool_refs[kMaxDev] = {};
}  // namespace

namespace afsai {
cudaMemPool_t library_pool() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDev) return nullptr;
    return g_pool[d];
}
}  // namespace afsai

static cudaMemPool_t pool_acquire(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 0 || dev >= kMaxDev) return nullptr;
    if (!g_pool[dev]) {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.handleTypes = cudaMemHandleTypeNone;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        if (cudaMemPoolCreate(&g_pool[dev], &pp) != cudaSuccess) {
            cudaGetLastError();
            g_pool[dev] = nullptr;
            return nullptr;
        }
    }
    ++g_pool_refs[dev];
    return g_pool[dev];
}

static void pool_release(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 0 || dev >= kMaxDev || !g_pool[dev]) return;
    if (--g_pool_refs[dev] <= 0) {
        g_pool_refs[dev] = 0;
        cudaMemPoolTrimTo(g_pool[dev], 0);  // return every unused byte to the device
    }
}

using namespace afsai;

extern "C" {

const char *afsai_version(void) { return "afsai-b200 0.1 (sm_100a)"; }

const char *afsai_strerror(int code) {
    switch (code) {
        case AFSAI_OK: return "ok";
        case AFSAI_EINVAL: return "invalid argument";
        case AFSAI_ENOTSPD: return "matrix is not SPD (non-positive pivot or psi)";
        case AFSAI_ECUDA: return "CUDA error";
        case AFSAI_ENCCL: return "NCCL error";
        case AFSAI_ENOMEM: return "out of device memory";
        case AFSAI_ENOTCONV: return "PCG did not converge within max_iters";
        case AFSAI_ELIMIT: return "implementation limit exceeded";
        default: return "unknown error";
    }
}

static int ctx_init(afsai_ctx_t c, void *stream, afsai_status_t *status) {
    AFSAI_CUDA_TRY(cudaGetDevice(&c->device));
    // keep freed stream-ordered allocations cached in the library pool while a
    // context lives: the set-up scratch and G are re-allocated every call and
    // remapping them costs ms
    cudaMemPool_t pool = pool_acquire(c->device);
    c->pool_held = pool != nullptr;
    if (pool) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // Map device memory into the pool once (default 20% of the device, at most half
        // of what is free; AFSAI_POOL_PREWARM_GB overrides, 0 disables), so set-up calls
        // do not grow it: growth maps memory on the host thread while the GPU idles
        // (0.2-0.7 s for the multi-GB G^T buffers of M3 on 2 GPUs; measured run-to-run
        // T_p 357-902 ms without, 350-352 ms with 24 GB).
        size_t fr = 0, tot = 0;
        double gb = 0.0;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) gb = std::min(0.2 * (double)tot, 0.5 * (double)fr) / 1073741824.0;
        if (const char *e = std::getenv("AFSAI_POOL_PREWARM_GB")) gb = std::atof(e);
        if (gb > 0) {
            void *p = nullptr;
            if (cudaMallocFromPoolAsync(&p, (size_t)(gb * 1073741824.0), pool, (cudaStream_t)stream) == cudaSuccess) {
                cudaFreeAsync(p, (cudaStream_t)stream);
                cudaStreamSynchronize((cudaStream_t)stream);
            } else {
                cudaGetLastError();
            }
        }
    }
    AFSAI_CUDA_TRY(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    c->stream = (cudaStream_t)stream;
    for (auto &e : c->ev) AFSAI_CUDA_TRY(cudaEventCreate(&e));
    return AFSAI_OK;
}

int afsai_ctx_create(afsai_ctx_t *ctx, void *stream) {
    afsai_status_t *status = nullptr;
    if (!ctx) return AFSAI_EINVAL;
    auto *c = new afsai_ctx_s();
    int rc = ctx_init(c, stream, status);
    if (rc != AFSAI_OK) {
        delete c;
        return rc;
    }
    *ctx = c;
    return AFSAI_OK;
}

int afsai_nccl_unique_id(char id[128]) {
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return AFSAI_ENCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
    std::memcpy(id, &u, 128);
    return AFSAI_OK;
}

int afsai_ctx_create_nccl(afsai_ctx_t *ctx, void *stream, const char id[128], int32_t rank, int32_t nranks) {
    afsai_status_t *status = nullptr;
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return AFSAI_EINVAL;
    auto *c = new afsai_ctx_s();
    int rc = ctx_init(c, stream, status);
    if (rc != AFSAI_OK) {
        delete c;
        return rc;
    }
    c->rank = rank;
    c->nranks = nranks;
    if (nranks > 1) {
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        if (ncclCommInitRank(&c->comm, nranks, u, rank) != ncclSuccess) {
            delete c;
            return AFSAI_ENCCL;
        }
        // NCCL connects point-to-point channels lazily, on the first send/recv
        // between two ranks (0.1-0.3 s on a fresh communicator, measured inside the
        // first set-up's halo exchange in round 1): connect every pair and the
        // all-reduce ring once here, outside any timed call.
        DevBuf w;
        const size_t off = (2 * (size_t)nranks + 7) & ~(size_t)7;  // two doubles after the pair bytes
        bool ok = w.alloc(off + 16, c->stream) == cudaSuccess &&
                  cudaMemsetAsync(w.p, 0, off + 16, c->stream) == cudaSuccess;
        ok = ok && ncclGroupStart() == ncclSuccess;
        if (ok) {
            char *b = w.as<char>();
            for (int q = 0; q < nranks; ++q) {
                if (q == rank) continue;
                ncclSend(b + q, 1, ncclChar, q, c->comm, c->stream);
                ncclRecv(b + nranks + q, 1, ncclChar, q, c->comm, c->stream);
            }
            ok = ncclGroupEnd() == ncclSuccess;
        }
        ok = ok && ncclAllReduce(w.as<char>() + off, w.as<char>() + off + 8, 1, ncclDouble, ncclSum, c->comm,
                                 c->stream) == ncclSuccess;
        w.release();
        ok = ok && cudaStreamSynchronize(c->stream) == cudaSuccess;
        if (!ok) {
            ncclCommDestroy(c->comm);
            delete c;
            return AFSAI_ENCCL;
        }
    }
    *ctx = c;
    return AFSAI_OK;
}

int afsai_ctx_rank(afsai_ctx_t ctx, int32_t *rank, int32_t *nranks) {
    if (!ctx) return AFSAI_EINVAL;
    if (rank) *rank = ctx->rank;
    if (nranks) *nranks = ctx->nranks;
    return AFSAI_OK;
}

void afsai_ctx_destroy(afsai_ctx_t ctx) {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto &t : ctx->timed) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    for (auto e : ctx->pool) cudaEventDestroy(e);
    if (ctx->pool_held) pool_release(ctx->device);
    delete ctx;
}

int64_t afsai_ctx_launches(afsai_ctx_t ctx) { return ctx ? ctx->launches : 0; }

int afsai_ctx_set_timing(afsai_ctx_t ctx, int32_t enable) {
    if (!ctx) return AFSAI_EINVAL;
    cudaStreamSynchronize(ctx->stream);
    for (auto &t : ctx->timed) {
        ctx->pool.push_back(t.a);
        ctx->pool.push_back(t.b);
    }
    ctx->timed.clear();
    for (int k = 0; k < AFSAI_K_NCLASSES; ++k) {
        ctx->t_launch[k] = 0;
        ctx->t_ms[k] = 0.0;
    }
    ctx->timing = enable != 0;
    return AFSAI_OK;
}

int afsai_ctx_kernel_times(afsai_ctx_t ctx, int64_t launches[AFSAI_K_NCLASSES], double ms[AFSAI_K_NCLASSES]) {
    if (!ctx) return AFSAI_EINVAL;
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return AFSAI_ECUDA;
    for (auto &t : ctx->timed) {
        float e = 0.f;
        cudaEventElapsedTime(&e, t.a, t.b);
        ctx->t_launch[t.cls] += 1;
        ctx->t_ms[t.cls] += e;
        ctx->pool.push_back(t.a);
        ctx->pool.push_back(t.b);
    }
    ctx->timed.clear();
    for (int k = 0; k < AFSAI_K_NCLASSES; ++k) {
        if (launches) launches[k] = ctx->t_launch[k];
        if (ms) ms[k] = ctx->t_ms[k];
    }
    return AFSAI_OK;
}

int afsai_setup(afsai_ctx_t ctx, const afsai_csr_t *A, const afsai_params_t *p, afsai_factor_t *out,
                afsai_status_t *status) {
    NvtxRange nv("afsai_setup");
    set_status(status, AFSAI_OK, "");
    if (!ctx || !A || !p || !out) return set_status(status, AFSAI_EINVAL, "null argument");
    if (A->n_rows < 0 || A->n_cols < 1 || A->nnz < 0 || A->row_begin < 0 || A->row_begin + A->n_rows > A->n_cols ||
        A->n_cols >= (int64_t)INT32_MAX || (A->n_rows > 0 && (!A->rowptr || !A->col || !A->val)))
        return set_status(status, AFSAI_EINVAL, "bad matrix sizes or null arrays");
    if (p->nsteps < 0 || p->s < 1 || p->s > AFSAI_MAX_S || !(p->eps >= 0.0 && p->eps < 1.0) || p->max_row_nnz < 1 ||
        (p->precision != AFSAI_PREC_FP64 && p->precision != AFSAI_PREC_FP32) || p->halo_k < 0 || p->halo_k > 64)
        return set_status(status, AFSAI_EINVAL,
                          "params out of range (nsteps>=0, 1<=s<=16, 0<=eps<1, max_row_nnz>=1, precision 0|1, "
                          "0<=halo_k<=64)");
    const int64_t mmax64 = std::min<int64_t>((int64_t)p->nsteps * p->s, (int64_t)p->max_row_nnz - 1);
    if (mmax64 > AFSAI_MAX_MMAX)
        return set_status(status, AFSAI_ELIMIT, "min(nsteps*s, max_row_nnz-1) exceeds AFSAI_MAX_MMAX (128)");
    if (ctx->nranks > 1) return dist_setup(ctx, A, p, out, status);
    if (A->row_begin != 0 || A->n_rows != A->n_cols)
        return set_status(status, AFSAI_EINVAL, "single-GPU context needs the whole matrix (row_begin 0)");
    return local_setup(ctx, A, p, out, status);
}

}  // extern "C"

namespace afsai {

// Single-GPU set-up: validate -> rows kernel -> assemble -> transpose.
int local_setup(afsai_ctx_t ctx, const afsai_csr_t *Ain, const afsai_params_t *p, afsai_factor_t *out,
                afsai_status_t *status) {
    cudaStream_t st = ctx->stream;
    DeviceCsr A;
    int rc = stage_csr(ctx, Ain, &A, status);
    if (rc) return rc;
    const int64_t n = A.n_rows;
    const int32_t mmax = (int32_t)std::max<int64_t>(0, std::min<int64_t>((int64_t)p->nsteps * p->s,
                                                                          (int64_t)p->max_row_nnz - 1));
    auto *F = new afsai_factor_s();
    F->ctx = ctx;
    F->n_rows = n;
    F->n_global = A.n_cols;
    F->row_begin = 0;
    F->stats.n_rows = n;
    auto fail = [&](int code) {
        delete F;
        return code;
    };
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[0], st));
    int64_t maxlen = 0;
    rc = validate_csr(ctx, A, &maxlen, status);
    if (rc) return fail(rc);

    SetupWork W;
    rc = W.alloc(ctx, n, mmax, status);
    if (rc) return fail(rc);
    if (F->steps.alloc(std::max<int64_t>(n, 1) * sizeof(int32_t), st) != cudaSuccess ||
        F->reason.alloc(std::max<int64_t>(n, 1) * sizeof(int32_t), st) != cudaSuccess)
        return fail(set_status(status, AFSAI_ENOMEM, "trace buffers"));
    W.steps = F->steps.as<int32_t>();
    W.reason = F->reason.as<int32_t>();

    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[1], st));
    rc = run_rows(ctx, A, 0, n, 0, n, *p, mmax, maxlen, W, &F->stats, status);
    if (rc) return fail(rc);
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[2], st));
    rc = W.check_error(ctx, status);
    if (rc) return fail(rc);

    rc = assemble_G(ctx, F, W, n, mmax + 1, status);
    if (rc) return fail(rc);
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[3], st));
    rc = transpose_G(ctx, F, 0, n, status);
    if (rc) return fail(rc);
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[4], st));
    rc = W.read_stats(ctx, &F->stats, status);
    if (rc) return fail(rc);
    F->retried = std::move(W.retried);
    F->n_retried = W.n_retried;
    F->stats.nnz_G = F->nnz_G;
    F->stats.nnz_Gt = F->nnz_Gt;
    F->stats.ms_total = elapsed(ctx->ev[1], ctx->ev[4]);
    F->stats.ms_rows = elapsed(ctx->ev[1], ctx->ev[2]);
    F->stats.ms_assemble = elapsed(ctx->ev[2], ctx->ev[3]);
    F->stats.ms_transpose = elapsed(ctx->ev[3], ctx->ev[4]);
    F->g_lo = 0;
    F->gt_hi = n;
    if (A.staged) {
        F->src_rowptr = Ain->rowptr;
        F->src_col = Ain->col;
        F->src_val = Ain->val;
        F->staged_A = std::move(A);
    }
    *out = F;
    return AFSAI_OK;
}

int SetupWork::alloc(afsai_ctx_t ctx, int64_t n, int32_t mmax, afsai_status_t *status) {
    cudaStream_t st = ctx->stream;
    const int64_t stride = mmax + 1;
    const int64_t nn = std::max<int64_t>(n, 1);
    if (scol.alloc(nn * stride * sizeof(int32_t), st) != cudaSuccess ||
        sval.alloc(nn * stride * sizeof(double), st) != cudaSuccess ||
        nnz_row.alloc(nn * sizeof(int32_t), st) != cudaSuccess || err.alloc(sizeof(unsigned long long), st) ||
        retry.alloc(nn * sizeof(int64_t), st) != cudaSuccess || retry_count.alloc(sizeof(int32_t), st) ||
        work.alloc(sizeof(unsigned long long), st) || counters.alloc(32 * sizeof(unsigned long long), st))
        return set_status(status, AFSAI_ENOMEM, "set-up scratch");
    AFSAI_CUDA_TRY(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), st));
    AFSAI_CUDA_TRY(cudaMemsetAsync(counters.p, 0, 32 * sizeof(unsigned long long), st));
    AFSAI_CUDA_TRY(cudaMemsetAsync(nnz_row.p, 0, nn * sizeof(int32_t), st));
    return AFSAI_OK;
}

int SetupWork::check_error(afsai_ctx_t ctx, afsai_status_t *status) {
    unsigned long long e = 0;
    AFSAI_CUDA_TRY(cudaMemcpyAsync(&e, err.p, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (e != ~0ull) {
        const int code = (int)(e & 0xf);
        const int64_t row = (int64_t)(e >> 24);
        const int32_t step = (int32_t)((e >> 4) & 0xfffff);
        return set_status(status, code, "non-positive pivot or psi: A is not SPD", row, step);
    }
    return AFSAI_OK;
}

int SetupWork::read_stats(afsai_ctx_t ctx, afsai_setup_stats_t *s, afsai_status_t *status) {
    unsigned long long c[32];
    AFSAI_CUDA_TRY(cudaMemcpyAsync(c, counters.p, sizeof c, cudaMemcpyDeviceToHost, ctx->stream));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    s->steps_total = (int64_t)c[0];
    s->fma_border = (int64_t)c[1];
    s->fma_backsub = (int64_t)c[2];
    s->fma_grad = (int64_t)c[3];
    s->grad_entries = (int64_t)c[4];
    for (int r = 0; r < 4; ++r) s->rows_by_reason[r] = (int64_t)c[5 + r];
    for (int k = 0; k < 7; ++k) s->phase_cycles[k] = (int64_t)c[9 + k];
    s->max_universe = (int64_t)c[16];
    return AFSAI_OK;
}

// count -> scan -> fill (a7).  The scratch rows are already sorted by column.
int assemble_G(afsai_ctx_t ctx, afsai_factor_t F, SetupWork &W, int64_t n, int32_t stride, afsai_status_t *status) {
    NvtxRange nv("afsai assemble G");
    cudaStream_t st = ctx->stream;
    DevBuf tiles;
    AFSAI_CUDA_TRY(tiles.alloc(scan_tmp_elems(n) * sizeof(int64_t) + 16, st));
    AFSAI_CUDA_TRY(F->g_rowptr.alloc((n + 1) * sizeof(int64_t), st));
    KTimer kt(ctx, AFSAI_K_ASSEMBLE);
    AFSAI_CUDA_TRY(exclusive_scan(W.nnz_row.as<int32_t>(), n, F->g_rowptr.as<int64_t>(), tiles.as<int64_t>(), st,
                                  &ctx->launches));
    int64_t nnz = 0;
    AFSAI_CUDA_TRY(cudaMemcpyAsync(&nnz, F->g_rowptr.as<int64_t>() + n, sizeof nnz, cudaMemcpyDeviceToHost, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    F->nnz_G = nnz;
    if (F->g_col.alloc(std::max<int64_t>(nnz, 1) * sizeof(int32_t), st) != cudaSuccess ||
        F->g_val.alloc(std::max<int64_t>(nnz, 1) * sizeof(double), st) != cudaSuccess)
        return set_status(status, AFSAI_ENOMEM, "G");
    const int grid = std::max<int64_t>(1, std::min<int64_t>((n * 32 + 255) / 256, grid_stream(ctx)));
    fill_rows_kernel<<<grid, 256, 0, st>>>(n, W.scol.as<int32_t>(), W.sval.as<double>(), stride,
                                          F->g_rowptr.as<int64_t>(), F->g_col.as<int32_t>(), F->g_val.as<double>());
    ctx->launches += 1;
    AFSAI_CUDA_TRY(cudaGetLastError());
    return AFSAI_OK;
}

// G^T of the local G (1 GPU: col_lo = 0, n_out = n): count columns, scan,
// scatter, then sort each row by source row (C10).
int transpose_G(afsai_ctx_t ctx, afsai_factor_t F, int64_t col_lo, int64_t n_out, afsai_status_t *status) {
    NvtxRange nv("afsai transpose G");
    cudaStream_t st = ctx->stream;
    DevBuf cnt, tiles, tcol, tval;
    const int64_t nnz = F->nnz_G;
    AFSAI_CUDA_TRY(cnt.alloc(std::max<int64_t>(n_out, 1) * sizeof(int32_t), st));
    AFSAI_CUDA_TRY(tiles.alloc(scan_tmp_elems(n_out) * sizeof(int64_t) + 16, st));
    AFSAI_CUDA_TRY(F->t_rowptr.alloc((n_out + 1) * sizeof(int64_t), st));
    AFSAI_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, std::max<int64_t>(n_out, 1) * sizeof(int32_t), st));
    const int grid = grid_stream(ctx);
    KTimer kt(ctx, AFSAI_K_TRANSPOSE);
    count_cols_kernel<<<grid, 256, 0, st>>>(nnz, F->g_col.as<int32_t>(), col_lo, n_out, cnt.as<int32_t>());
    ctx->launches += 1;
    AFSAI_CUDA_TRY(exclusive_scan(cnt.as<int32_t>(), n_out, F->t_rowptr.as<int64_t>(), tiles.as<int64_t>(), st,
                                  &ctx->launches));
    F->nnz_Gt = nnz;  // one GPU: every entry lands locally
    if (F->t_col.alloc(std::max<int64_t>(nnz, 1) * sizeof(int32_t), st) != cudaSuccess ||
        F->t_val.alloc(std::max<int64_t>(nnz, 1) * sizeof(double), st) != cudaSuccess)
        return set_status(status, AFSAI_ENOMEM, "G^T");
    const char *tenv = std::getenv("AFSAI_TRANSPOSE");
    if (tenv && std::strcmp(tenv, "radix") == 0) {
        // stable radix sort by column (no atomics, no per-row sort; 27.7 vs 24.2 ms on
        // M3, so the atomic scatter + sort below stays the default)
        DevBuf rx;
        if (rx.alloc((size_t)radix_tmp_bytes(nnz, n_out), st) != cudaSuccess)
            return set_status(status, AFSAI_ENOMEM, "G^T radix scratch");
        AFSAI_CUDA_TRY(transpose_radix(F->n_rows, F->g_rowptr.as<int64_t>(), F->g_col.as<int32_t>(),
                                       F->g_val.as<double>(), nnz, col_lo, n_out, F->row_begin, rx.as<char>(),
                                       F->t_col.as<int32_t>(), F->t_val.as<double>(), grid, st, &ctx->launches));
        return AFSAI_OK;
    }
    // scatter with column cursors (atomics), then a per-row sort into source-row order
    if (tcol.alloc(std::max<int64_t>(nnz, 1) * sizeof(int32_t), st) != cudaSuccess ||
        tval.alloc(std::max<int64_t>(nnz, 1) * sizeof(double), st) != cudaSuccess)
        return set_status(status, AFSAI_ENOMEM, "G^T");
    AFSAI_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, std::max<int64_t>(n_out, 1) * sizeof(int32_t), st));
    scatter_t_kernel<<<grid, 256, 0, st>>>(F->n_rows, F->g_rowptr.as<int64_t>(), F->g_col.as<int32_t>(),
                                           F->g_val.as<double>(), F->row_begin, col_lo, n_out,
                                           F->t_rowptr.as<int64_t>(), cnt.as<int32_t>(), tcol.as<int32_t>(),
                                           tval.as<double>());
    sort_gt_rows(n_out, F->t_rowptr.as<int64_t>(), tcol.as<int32_t>(), tval.as<double>(), F->t_col.as<int32_t>(),
                 F->t_val.as<double>(), grid, st, &ctx->launches);
    ctx->launches += 1;
    AFSAI_CUDA_TRY(cudaGetLastError());
    return AFSAI_OK;
}

// ---------------------------------------------------------------- apply / PCG
int PcgWork::ensure(afsai_ctx_t ctx, int64_t n, afsai_status_t *status) {
    if (n_alloc >= n && vec.p) return AFSAI_OK;
    cudaStream_t st = ctx->stream;
    const int64_t nn = std::max<int64_t>(n, 1);
    nparts = grid_stream(ctx);
    if (vec.alloc(6 * nn * sizeof(double), st) != cudaSuccess ||
        parts.alloc((size_t)nparts * sizeof(double) * 2, st) != cudaSuccess ||
        counter.alloc(4 * sizeof(unsigned), st) != cudaSuccess || state.alloc(sizeof(PcgState), st) != cudaSuccess)
        return set_status(status, AFSAI_ENOMEM, "PCG workspace");
    AFSAI_CUDA_TRY(cudaMemsetAsync(counter.p, 0, 4 * sizeof(unsigned), st));
    AFSAI_CUDA_TRY(cudaMemsetAsync(state.p, 0, sizeof(PcgState), st));
    n_alloc = n;
    return AFSAI_OK;
}

static SpmvArgs spmv_args(int64_t n, const int64_t *rp, const int32_t *ci, const double *v, const double *x,
                          int64_t xoff, double *y) {
    SpmvArgs a{};
    a.n = n;
    a.rowptr = rp;
    a.col = ci;
    a.val = v;
    a.x = x;
    a.x_off = xoff;
    a.y = y;
    return a;
}

// t = G r ; z = G^T t   (+ optional fused dot(z, w) in `mode`)
void launch_apply_local(afsai_ctx_t ctx, afsai_factor_t F, const double *r, double *t, double *z, int mode,
                        const double *w, PcgWork *pw) {
    const int64_t n = F->n_rows;
    const int grid = grid_stream(ctx);
    SpmvArgs a = spmv_args(n, F->g_rowptr.as<int64_t>(), F->g_col.as<int32_t>(), F->g_val.as<double>(), r, 0, t);
    if (pw) a.st = pw->state.as<PcgState>();
    {
        KTimer kt(ctx, AFSAI_K_SPMV_G);
        launch_spmv(a, 0, spmv_group_width((double)F->nnz_G / std::max<int64_t>(n, 1), 1), grid, ctx->stream);
    }
    SpmvArgs b = spmv_args(n, F->t_rowptr.as<int64_t>(), F->t_col.as<int32_t>(), F->t_val.as<double>(), t, 0, z);
    if (pw) {
        b.st = pw->state.as<PcgState>();
        b.w = w;
        b.partials = pw->parts.as<double>();
        b.counter = pw->counter.as<unsigned>();
    }
    {
        KTimer kt(ctx, AFSAI_K_SPMV_GT);
        launch_spmv(b, mode, spmv_group_width((double)F->nnz_Gt / std::max<int64_t>(n, 1), 2), grid, ctx->stream);
    }
    ctx->launches += 2;
}

}  // namespace afsai

extern "C" {

int afsai_apply(afsai_ctx_t ctx, afsai_factor_t F, const double *r, double *z) {
    NvtxRange nv("afsai_apply");
    afsai_status_t *status = nullptr;
    if (!ctx || !F || !r || !z || r == z) return AFSAI_EINVAL;
    if (F->ctx != ctx || F->block) return AFSAI_EINVAL;  // another context's factor / a block factor (no G^T)
    if (ctx->nranks > 1) return dist_apply(ctx, F, r, z, status);
    const int64_t n = F->n_rows;
    cudaStream_t st = ctx->stream;
    const bool rdev = is_device_ptr(r), zdev = is_device_ptr(z);
    DevBuf rb, zb, tb;
    AFSAI_CUDA_TRY(tb.alloc(std::max<int64_t>(n, 1) * sizeof(double), st));
    const double *rd = r;
    double *zd = z;
    if (!rdev) {
        AFSAI_CUDA_TRY(rb.alloc(std::max<int64_t>(n, 1) * sizeof(double), st));
        AFSAI_CUDA_TRY(cudaMemcpyAsync(rb.p, r, n * sizeof(double), cudaMemcpyHostToDevice, st));
        rd = rb.as<double>();
    }
    if (!zdev) {
        AFSAI_CUDA_TRY(zb.alloc(std::max<int64_t>(n, 1) * sizeof(double), st));
        zd = zb.as<double>();
    }
    launch_apply_local(ctx, F, rd, tb.as<double>(), zd, 0, nullptr, nullptr);
    AFSAI_CUDA_TRY(cudaGetLastError());
    if (!zdev) {
        AFSAI_CUDA_TRY(cudaMemcpyAsync(z, zd, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return AFSAI_OK;
}

int afsai_pcg(afsai_ctx_t ctx, const afsai_csr_t *Ain, afsai_factor_t F, const double *b, double *x, double tol,
              int32_t max_iters, afsai_pcg_report_t *rep, afsai_status_t *status) {
    NvtxRange nv("afsai_pcg");
    set_status(status, AFSAI_OK, "");
    if (!ctx || !Ain || !F || !b || !x || !(tol > 0.0) || max_iters < 1)
        return set_status(status, AFSAI_EINVAL, "bad PCG arguments");
    if (F->ctx != ctx || F->block)
        return set_status(status, AFSAI_EINVAL, "factor belongs to another context or is a block factor (no G^T)");
    if (Ain->n_rows != F->n_rows || Ain->row_begin != F->row_begin)
        return set_status(status, AFSAI_EINVAL, "A does not match the factor's rows");
    if (ctx->nranks > 1) return dist_pcg(ctx, Ain, F, b, x, tol, max_iters, rep, status);
    return local_pcg(ctx, Ain, F, b, x, tol, max_iters, rep, status);
}

}  // extern "C"

namespace afsai {

// PCG on one GPU (R12, §4.4).  Five kernels per iteration; the scalars
// live on the device; the host polls the `done` flag every kPoll iterations.
int local_pcg(afsai_ctx_t ctx, const afsai_csr_t *Ain, afsai_factor_t F, const double *b, double *x, double tol,
              int32_t max_iters, afsai_pcg_report_t *rep, afsai_status_t *status) {
    cudaStream_t st = ctx->stream;
    DeviceCsr Aown;
    const DeviceCsr *Ap = &Aown;
    if (F->staged_A.staged && Ain->rowptr == F->src_rowptr && Ain->col == F->src_col && Ain->val == F->src_val) {
        Ap = &F->staged_A;
    } else {
        int rc0 = stage_csr(ctx, Ain, &Aown, status);
        if (rc0) return rc0;
    }
    const DeviceCsr &A = *Ap;
    int rc = AFSAI_OK;
    const int64_t n = A.n_rows;
    PcgWork &W = F->pcg;
    rc = W.ensure(ctx, n, status);
    if (rc) return rc;
    double *V = W.vec.as<double>();
    double *r = V, *p = V + n, *q = V + 2 * n, *z = V + 3 * n, *t = V + 4 * n, *xs = V + 5 * n;
    const bool bdev = is_device_ptr(b), xdev = is_device_ptr(x);
    DevBuf bb;
    const double *bd = b;
    if (!bdev) {
        AFSAI_CUDA_TRY(bb.alloc(std::max<int64_t>(n, 1) * sizeof(double), st));
        AFSAI_CUDA_TRY(cudaMemcpyAsync(bb.p, b, n * sizeof(double), cudaMemcpyHostToDevice, st));
        bd = bb.as<double>();
    }
    double *xd = xdev ? x : xs;
    PcgState *S = W.state.as<PcgState>();
    double *parts = W.parts.as<double>();
    unsigned *cnt = W.counter.as<unsigned>();
    const int grid = grid_stream(ctx);
    // A with absolute offsets: rowptr - base handled by passing shifted col/val
    const int64_t *arp = A.rowptr;
    const int32_t *aci = A.col - A.base;
    const double *av = A.val - A.base;
    const int wA = spmv_group_width((double)A.nnz / std::max<int64_t>(n, 1), 0);

    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[5], st));
    {
        KTimer kt(ctx, AFSAI_K_VECTOR);
        launch_pcg_init(n, bd, xd, r, parts, cnt, S, grid, st);
    }
    // z = M^-1 r = G^T (G r): two deterministic SpMVs (G, then G^T with the fused
    // r.z), or with AFSAI_APPLY=single one pass over G with fp64 reductions into z
    // (12 instead of 24 bytes per nonzero), then r.z
    const char *apply_env = std::getenv("AFSAI_APPLY");
    const bool single = apply_env && std::strcmp(apply_env, "single") == 0;
    const int wG1 = spmv_group_width((double)F->nnz_G / std::max<int64_t>(n, 1), 1);
    auto apply_rz = [&](int first) {
        if (single) {
            cudaMemsetAsync(z, 0, n * sizeof(double), st);
            {
                KTimer kt(ctx, AFSAI_K_SPMV_G);
                launch_apply_single_pass(n, F->g_rowptr.as<int64_t>(), F->g_col.as<int32_t>(), F->g_val.as<double>(),
                                         r, z, S, wG1, grid, st);
            }
            {
                KTimer kt(ctx, AFSAI_K_VECTOR);
                launch_pcg_rz(n, r, z, parts, cnt, S, first, grid, st);
            }
            ctx->launches += 2;
        } else {
            launch_apply_local(ctx, F, r, t, z, first ? 3 : 2, r, &W);
        }
    };
    apply_rz(1);  // z = M^-1 r, rz = r.z
    {
        KTimer kt(ctx, AFSAI_K_VECTOR);
        launch_pcg_update_p(n, p, z, S, 1, grid, st);  // p = z
    }
    ctx->launches += 2;
    PcgState hs{};
    const int kPoll = 8;
    int it = 0;
    for (;;) {
        for (int k = 0; k < kPoll && it < max_iters; ++k, ++it) {
            SpmvArgs aq = spmv_args(n, arp, aci, av, p, 0, q);
            aq.w = p;
            aq.partials = parts;
            aq.counter = cnt;
            aq.st = S;
            {
                KTimer kt(ctx, AFSAI_K_SPMV_A);
                launch_spmv(aq, 1, wA, grid, st);  // q = A p, alpha
            }
            {
                KTimer kt(ctx, AFSAI_K_VECTOR);
                launch_pcg_axpy(n, xd, r, p, q, parts, cnt, S, tol, max_iters, grid, st);  // x, r, test
            }
            apply_rz(0);  // z = M^-1 r, beta
            {
                KTimer kt(ctx, AFSAI_K_VECTOR);
                launch_pcg_update_p(n, p, z, S, 0, grid, st);  // p = z + beta p
            }
            ctx->launches += 3;
        }
        AFSAI_CUDA_TRY(cudaGetLastError());
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&hs, S, sizeof hs, cudaMemcpyDeviceToHost, st));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
        if (hs.done || it >= max_iters) break;
    }
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[6], st));
    // explicit residual ||b - A x|| / ||b||
    {
        SpmvArgs ax = spmv_args(n, arp, aci, av, xd, 0, q);
        launch_spmv(ax, 0, wA, grid, st);
        launch_residual(n, bd, q, parts, cnt, &S->true_rr, grid, st);
        ctx->launches += 2;
    }
    AFSAI_CUDA_TRY(cudaMemcpyAsync(&hs, S, sizeof hs, cudaMemcpyDeviceToHost, st));
    if (!xdev) AFSAI_CUDA_TRY(cudaMemcpyAsync(x, xd, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    if (rep) {
        rep->iters = hs.iters;
        rep->converged = hs.done == 1 || hs.bnorm2 == 0.0;
        rep->rel_res = hs.rel;
        rep->true_rel_res = hs.bnorm2 > 0 ? std::sqrt(hs.true_rr) / std::sqrt(hs.bnorm2) : 0.0;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[5], ctx->ev[6]);
        rep->ms_solve = ms;
        rep->ms_per_iter = hs.iters > 0 ? ms / hs.iters : 0.0;
    }
    const bool conv = hs.done == 1 || hs.bnorm2 == 0.0;
    return conv ? AFSAI_OK : set_status(status, AFSAI_ENOTCONV, "PCG reached max_iters");
}

}  // namespace afsai

extern "C" {

int afsai_factor_nnz(afsai_factor_t F, int64_t *nnz_G, int64_t *nnz_Gt) {
    if (!F) return AFSAI_EINVAL;
    if (nnz_G) *nnz_G = F->nnz_G;
    if (nnz_Gt) *nnz_Gt = F->nnz_Gt;
    return AFSAI_OK;
}

int afsai_factor_copy(afsai_factor_t F, int32_t which, int64_t *rowptr, int32_t *col, double *val) {
    afsai_status_t *status = nullptr;
    if (!F || (which != 0 && which != 1) || (which == 1 && F->block)) return AFSAI_EINVAL;
    cudaStream_t st = F->ctx->stream;
    const int64_t n = F->n_rows, nnz = which ? F->nnz_Gt : F->nnz_G;
    const DevBuf &rp = which ? F->t_rowptr : F->g_rowptr;
    const DevBuf &ci = which ? F->t_col : F->g_col;
    const DevBuf &v = which ? F->t_val : F->g_val;
    if (rowptr) AFSAI_CUDA_TRY(cudaMemcpyAsync(rowptr, rp.p, (n + 1) * sizeof(int64_t), cudaMemcpyDefault, st));
    if (col && nnz) AFSAI_CUDA_TRY(cudaMemcpyAsync(col, ci.p, nnz * sizeof(int32_t), cudaMemcpyDefault, st));
    if (val && nnz) AFSAI_CUDA_TRY(cudaMemcpyAsync(val, v.p, nnz * sizeof(double), cudaMemcpyDefault, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    return AFSAI_OK;
}

int afsai_factor_trace(afsai_factor_t F, int32_t *steps, int32_t *reason) {
    afsai_status_t *status = nullptr;
    if (!F) return AFSAI_EINVAL;
    cudaStream_t st = F->ctx->stream;
    if (steps && F->n_rows)
        AFSAI_CUDA_TRY(cudaMemcpyAsync(steps, F->steps.p, F->n_rows * sizeof(int32_t), cudaMemcpyDefault, st));
    if (reason && F->n_rows)
        AFSAI_CUDA_TRY(cudaMemcpyAsync(reason, F->reason.p, F->n_rows * sizeof(int32_t), cudaMemcpyDefault, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    return AFSAI_OK;
}

int afsai_factor_retried(afsai_factor_t F, int64_t *rows, int64_t max_rows, int64_t *count) {
    afsai_status_t *status = nullptr;
    if (!F || !count || max_rows < 0) return AFSAI_EINVAL;
    *count = F->n_retried;
    const int64_t k = std::min(max_rows, F->n_retried);
    if (rows && k > 0) {
        AFSAI_CUDA_TRY(cudaMemcpyAsync(rows, F->retried.p, k * sizeof(int64_t), cudaMemcpyDefault, F->ctx->stream));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(F->ctx->stream));
    }
    return AFSAI_OK;
}

int afsai_factor_stats(afsai_factor_t F, afsai_setup_stats_t *s) {
    if (!F || !s) return AFSAI_EINVAL;
    *s = F->stats;
    return AFSAI_OK;
}

void afsai_factor_destroy(afsai_factor_t F) {
    if (!F) return;
    cudaStreamSynchronize(F->ctx->stream);
    dist_free(F);
    delete F;
}

int afsai_probe_dfma_peak(afsai_ctx_t ctx, double *flops_per_s, double *ms_out) {
    afsai_status_t *status = nullptr;
    if (!ctx) return AFSAI_EINVAL;
    DevBuf out;
    AFSAI_CUDA_TRY(out.alloc(sizeof(double), ctx->stream));
    const int grid = ctx->num_sms * 8;
    const int iters = 4096;
    launch_dfma_probe(out.as<double>(), 64, grid, ctx->stream);  // warm-up
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[0], ctx->stream));
    launch_dfma_probe(out.as<double>(), iters, grid, ctx->stream);
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[1], ctx->stream));
    ctx->launches += 2;
    AFSAI_CUDA_TRY(cudaEventSynchronize(ctx->ev[1]));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    const double flops = 2.0 * 8 * 16 * (double)iters * grid * 256;
    if (flops_per_s) *flops_per_s = flops / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    return AFSAI_OK;
}

}  // extern "C"
