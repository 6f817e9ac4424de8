// dist.cu -- multi-GPU aFSAI (one process per GPU, NCCL over NVLink/NVSwitch).
//
// Rows are block-partitioned: rank p owns the contiguous rows [b_p, e_p).
// (PAPER.md P:815-839 stripes.)
//  - set-up halo, once: every pattern entry of row i lies within graph distance
//    k_max of i (each step adds neighbours of P U {i}) and the kernels
//    only read rows < i, so the rows [b_p - k_max*beta, b_p) of A (beta = global
//    bandwidth) are exactly sufficient; they are gathered with grouped
//    ncclSend/ncclRecv of contiguous row ranges (lengths first, then col/val).
//    The set-up kernel then runs on the local rows unchanged: G is bitwise the
//    1-GPU G (pin P12).
//  - G^T: entries (i, j) of the local G go to the owner of column j (grouped
//    send/recv of (col, row, val) triples); each rank builds its G^T rows sorted
//    by source row.
//  - PCG: per iteration three range halos (p for A p: [b - beta_A, e + beta_A);
//    r for G r: [b - beta_G, b); t for G^T t: [e, e + beta_G)) and two
//    all-reduces (p.q; then r.r and r.z packed in one).  Contiguous ranges need no packing:
//    NCCL sends and receives straight from/into the extended vectors.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "assemble.h"
#include "dist.h"
#include "setup_kernel.h"
#include "spmv.h"

namespace afsai {

struct Seg {
    int peer;
    int64_t begin, count;  // global index range [begin, begin + count)
};

// A range halo for one distributed vector: this rank holds [b, e) and needs
// the extended range [lo, hi).
struct RangePlan {
    int64_t lo = 0, hi = 0, b = 0, e = 0;
    std::vector<Seg> sends, recvs;
};

// Host-side plan: ranks own [bounds[q], bounds[q+1]); rank q needs [lo[q], hi[q]).
static RangePlan make_range_plan(int me, int nranks, const std::vector<int64_t> &bounds,
                                 const std::vector<int64_t> &lo, const std::vector<int64_t> &hi) {
    RangePlan P;
    P.b = bounds[me];
    P.e = bounds[me + 1];
    P.lo = lo[me];
    P.hi = hi[me];
    for (int q = 0; q < nranks; ++q) {
        if (q == me) continue;
        // what q needs from me
        const int64_t s0 = std::max(P.b, lo[q]), s1 = std::min(P.e, hi[q]);
        if (s1 > s0) P.sends.push_back({q, s0, s1 - s0});
        // what I need from q
        const int64_t r0 = std::max(bounds[q], P.lo), r1 = std::min(bounds[q + 1], P.hi);
        if (r1 > r0) P.recvs.push_back({q, r0, r1 - r0});
    }
    return P;
}

// Wait for the context stream while polling NCCL's asynchronous error state: a
// failed or vanished peer would otherwise leave cudaStreamSynchronize waiting
// forever inside a collective.  On an NCCL error the communicator is aborted
// (the context then refuses further collective calls) and AFSAI_ENCCL returned.
static int sync_poll(afsai_ctx_t ctx, afsai_status_t *status) {
    for (;;) {
        const cudaError_t e = cudaStreamQuery(ctx->stream);
        if (e == cudaSuccess) return AFSAI_OK;
        if (e != cudaErrorNotReady)
            return set_status(status, AFSAI_ECUDA, std::string("stream error: ") + cudaGetErrorString(e));
        ncclResult_t r = ncclSuccess;
        if (ctx->comm && ncclCommGetAsyncError(ctx->comm, &r) == ncclSuccess && r != ncclSuccess &&
            r != ncclInProgress) {
            ncclCommAbort(ctx->comm);
            ctx->comm = nullptr;
            return set_status(status, AFSAI_ENCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(r));
        }
        std::this_thread::yield();
    }
}

// exchange a RangePlan on an extended buffer ext (index = global - lo) of `elem` bytes
static ncclResult_t range_exchange(const RangePlan &P, void *ext, size_t elem, ncclComm_t comm, cudaStream_t st) {
    char *base = static_cast<char *>(ext);
    ncclResult_t r = ncclGroupStart();
    if (r != ncclSuccess) return r;
    for (const Seg &s : P.recvs)
        if ((r = ncclRecv(base + (s.begin - P.lo) * elem, s.count * elem, ncclChar, s.peer, comm, st)) != ncclSuccess)
            break;
    if (r == ncclSuccess)
        for (const Seg &s : P.sends)
            if ((r = ncclSend(base + (s.begin - P.lo) * elem, s.count * elem, ncclChar, s.peer, comm, st)) !=
                ncclSuccess)
                break;
    const ncclResult_t r2 = ncclGroupEnd();  // always close the group
    return r != ncclSuccess ? r : r2;
}

// an NCCL group that is always closed, also when a call inside it fails
struct NcclGroup {
    bool open = false;
    ncclResult_t start() {
        const ncclResult_t r = ncclGroupStart();
        open = r == ncclSuccess;
        return r;
    }
    ncclResult_t end() {
        open = false;
        return ncclGroupEnd();
    }
    ~NcclGroup() {
        if (open) ncclGroupEnd();
    }
};

struct DistState {
    std::vector<int64_t> bounds;  // nranks + 1
    RangePlan planA, planG, planT;
    int64_t betaA = 0, betaG = 0;
    DevBuf ext;  // p_ext | r_ext | t_ext (PCG / apply)
};

static DistState *dstate(afsai_factor_t F) { return static_cast<DistState *>(F->dist); }

void dist_free(afsai_factor_t F) {
    if (F && F->dist) {
        delete dstate(F);
        F->dist = nullptr;
    }
}

// all-gather of one int64 per rank (via a device buffer)
static int allgather_i64(afsai_ctx_t ctx, int64_t v, std::vector<int64_t> &out, afsai_status_t *status) {
    DevBuf d;
    AFSAI_CUDA_TRY(d.alloc((ctx->nranks + 1) * sizeof(int64_t), ctx->stream));
    AFSAI_CUDA_TRY(cudaMemcpyAsync(d.as<int64_t>() + ctx->nranks, &v, sizeof v, cudaMemcpyHostToDevice, ctx->stream));
    AFSAI_NCCL_TRY(ncclAllGather(d.as<int64_t>() + ctx->nranks, d.p, 1, ncclInt64, ctx->comm, ctx->stream));
    out.assign(ctx->nranks, 0);
    AFSAI_CUDA_TRY(cudaMemcpyAsync(out.data(), d.p, ctx->nranks * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return AFSAI_OK;
}

__global__ void bandwidth_kernel(const int64_t *rowptr, const int32_t *col, int64_t base, int64_t n_rows,
                                 int64_t row_begin, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e0 = rowptr[r] - base, e1 = rowptr[r + 1] - base;
        if (e1 > e0) {
            const int64_t gi = r + row_begin;
            const int64_t d0 = gi - (int64_t)col[e0], d1 = (int64_t)col[e1 - 1] - gi;
            const unsigned long long d = (unsigned long long)(d0 > d1 ? d0 : d1);
            m = d > m ? d : m;
        }
    }
    atomicMax(out, m);
}

// max over ranks of a local non-negative int64
static int allreduce_max(afsai_ctx_t ctx, int64_t v, int64_t *out, afsai_status_t *status) {
    std::vector<int64_t> all;
    int rc = allgather_i64(ctx, v, all, status);
    if (rc) return rc;
    *out = *std::max_element(all.begin(), all.end());
    return AFSAI_OK;
}

// Error agreement: after a step that can fail on one rank only (staging,
// validation, an allocation, a non-SPD row), every rank learns whether any rank
// failed, so no rank walks into a collective a failed rank will never join.
// Returns rc if this rank failed, else the lowest failing rank's code (AFSAI_OK if none).
static int agree(afsai_ctx_t ctx, int rc, afsai_status_t *status) {
    std::vector<int64_t> all;
    afsai_status_t tmp{};
    const int r2 = allgather_i64(ctx, rc, all, &tmp);
    if (r2) return rc ? rc : set_status(status, r2, tmp.msg);
    if (rc) return rc;
    for (int q = 0; q < ctx->nranks; ++q)
        if (all[q])
            return set_status(status, (int)all[q],
                              "rank " + std::to_string(q) + " failed (" + afsai_strerror((int)all[q]) + ")");
    return AFSAI_OK;
}

// G rows [row_lo, row_lo + nrows) from a matrix holding rows [a_lo, a_hi)
// (validated); fills F's G (global columns), trace and stats.
int block_rows_to_G(afsai_ctx_t ctx, const DeviceCsr &Aext, int64_t a_lo, int64_t a_hi, int64_t row_lo,
                           int64_t nrows, const afsai_params_t *p, int64_t maxlen, afsai_factor_t F,
                           afsai_status_t *status) {
    cudaStream_t st = ctx->stream;
    const int32_t mmax = (int32_t)std::max<int64_t>(
        0, std::min<int64_t>((int64_t)p->nsteps * p->s, (int64_t)p->max_row_nnz - 1));
    SetupWork W;
    int rc = W.alloc(ctx, nrows, mmax, status);
    if (rc) return rc;
    if (F->steps.alloc(std::max<int64_t>(nrows, 1) * sizeof(int32_t), st) != cudaSuccess ||
        F->reason.alloc(std::max<int64_t>(nrows, 1) * sizeof(int32_t), st) != cudaSuccess)
        return set_status(status, AFSAI_ENOMEM, "trace buffers");
    W.steps = F->steps.as<int32_t>();
    W.reason = F->reason.as<int32_t>();
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[1], st));
    rc = run_rows(ctx, Aext, a_lo, a_hi, row_lo, nrows, *p, mmax, maxlen, W, &F->stats, status);
    if (rc) return rc;
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[2], st));
    rc = W.check_error(ctx, status);
    if (rc) return rc;
    rc = assemble_G(ctx, F, W, nrows, mmax + 1, status);
    if (rc) return rc;
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[3], st));
    rc = W.read_stats(ctx, &F->stats, status);
    if (rc) return rc;
    F->retried = std::move(W.retried);
    F->n_retried = W.n_retried;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]);
    F->stats.ms_rows = ms;
    cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
    F->stats.ms_assemble = ms;
    F->stats.nnz_G = F->nnz_G;
    return AFSAI_OK;
}

// out[k] = in[idx[k]] (a few scattered values of a device array for the host)
__global__ void gather_i64_kernel(const int64_t *in, const int64_t *idx, int n, int64_t *out) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) out[k] = in[idx[k]];
}

// Gather rows [lo, b) of A from lower ranks (exact set-up halo) and build the
// extended CSR of rows [lo, e).
static int gather_halo(afsai_ctx_t ctx, const DeviceCsr &A, const std::vector<int64_t> &bounds, int64_t lo,
                       DeviceCsr *X, afsai_status_t *status) {
    NvtxRange nv("afsai set-up halo exchange");
    cudaStream_t st = ctx->stream;
    const int me = ctx->rank, np = ctx->nranks;
    const int64_t b = bounds[me], e = bounds[me + 1];
    // every rank's needed lower range [lo_q, b_q): recompute from each rank's lo
    std::vector<int64_t> los;
    int rc = allgather_i64(ctx, lo, los, status);
    if (rc) return rc;
    std::vector<int64_t> his(np);
    for (int q = 0; q < np; ++q) his[q] = bounds[q];  // lower halo only
    RangePlan P = make_range_plan(me, np, bounds, los, his);
    // stage 1: row lengths (int32) over the extended row range [lo, e)
    const int64_t next = e - lo;
    DevBuf len, rp, tiles;
    AFSAI_CUDA_TRY(len.alloc(std::max<int64_t>(next, 1) * sizeof(int32_t), st));
    AFSAI_CUDA_TRY(rp.alloc((next + 1) * sizeof(int64_t), st));
    AFSAI_CUDA_TRY(tiles.alloc(scan_tmp_elems(next) * sizeof(int64_t) + 16, st));
    const int grid = grid_stream(ctx);
    row_lengths_kernel<<<grid, 256, 0, st>>>(A.rowptr, A.n_rows, len.as<int32_t>() + (b - lo));
    ctx->launches += 1;
    {
        KTimer kt(ctx, AFSAI_K_COMM);
        // sends read my local lengths (their global rows lie in [b, e) == ext index >= b - lo)
        RangePlan P1 = P;
        P1.lo = lo;
        AFSAI_NCCL_TRY(range_exchange(P1, len.p, sizeof(int32_t), ctx->comm, st));
    }
    AFSAI_CUDA_TRY(exclusive_scan(len.as<int32_t>(), next, rp.as<int64_t>(), tiles.as<int64_t>(), st, &ctx->launches));
    // the host needs the extended row pointer only at segment boundaries (entry
    // ranges of the sends / receives), at b and at the end: gather those few values
    // on the device instead of copying the whole (n_rows + halo) row pointer
    std::vector<int64_t> need = {next, b - lo};
    for (const Seg &sg : P.recvs) need.insert(need.end(), {sg.begin - lo, sg.begin + sg.count - lo});
    for (const Seg &sg : P.sends) need.insert(need.end(), {sg.begin - lo, sg.begin + sg.count - lo});
    DevBuf dneed;
    AFSAI_CUDA_TRY(dneed.alloc(2 * need.size() * sizeof(int64_t), st));
    AFSAI_CUDA_TRY(cudaMemcpyAsync(dneed.p, need.data(), need.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    gather_i64_kernel<<<1, 256, 0, st>>>(rp.as<int64_t>(), dneed.as<int64_t>(), (int)need.size(),
                                         dneed.as<int64_t>() + need.size());
    ctx->launches += 1;
    std::vector<int64_t> vals(need.size());
    AFSAI_CUDA_TRY(cudaMemcpyAsync(vals.data(), dneed.as<int64_t>() + need.size(), need.size() * sizeof(int64_t),
                                   cudaMemcpyDeviceToHost, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    std::unordered_map<int64_t, int64_t> hrp;  // extended row index -> entry offset
    for (size_t k = 0; k < need.size(); ++k) hrp[need[k]] = vals[k];
    const int64_t nnz_ext = hrp[next];
    // stage 2: col / val of the halo rows straight into the extended arrays;
    // sends come from my local arrays (entry ranges from my host row pointer)
    X->b_rowptr = std::move(rp);
    X->rowptr = X->b_rowptr.as<int64_t>();
    AFSAI_CUDA_TRY(X->b_col.alloc(std::max<int64_t>(nnz_ext, 1) * sizeof(int32_t), st));
    AFSAI_CUDA_TRY(X->b_val.alloc(std::max<int64_t>(nnz_ext, 1) * sizeof(double), st));
    X->col = X->b_col.as<int32_t>();
    X->val = X->b_val.as<double>();
    X->base = 0;
    X->n_rows = next;
    X->n_cols = A.n_cols;
    X->row_begin = lo;
    X->nnz = nnz_ext;
    X->staged = true;
    const int64_t loc_off = hrp[b - lo];  // local rows start here in the extended arrays
    AFSAI_CUDA_TRY(cudaMemcpyAsync(X->b_col.as<int32_t>() + loc_off, A.col, A.nnz * sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, st));
    AFSAI_CUDA_TRY(cudaMemcpyAsync(X->b_val.as<double>() + loc_off, A.val, A.nnz * sizeof(double),
                                   cudaMemcpyDeviceToDevice, st));
    {
        KTimer kt(ctx, AFSAI_K_COMM);
        NcclGroup grp;
        AFSAI_NCCL_TRY(grp.start());
        for (const Seg &s : P.recvs) {
            const int64_t e0 = hrp[s.begin - lo], e1 = hrp[s.begin + s.count - lo];
            AFSAI_NCCL_TRY(ncclRecv(X->b_col.as<int32_t>() + e0, (e1 - e0), ncclInt32, s.peer, ctx->comm, st));
            AFSAI_NCCL_TRY(ncclRecv(X->b_val.as<double>() + e0, (e1 - e0), ncclDouble, s.peer, ctx->comm, st));
        }
        for (const Seg &s : P.sends) {
            // entries of my rows [s.begin, s.begin + count) are at the same place in the
            // extended arrays (local part copied above)
            const int64_t e0 = hrp[s.begin - lo], e1 = hrp[s.begin + s.count - lo];
            AFSAI_NCCL_TRY(ncclSend(X->b_col.as<int32_t>() + e0, (e1 - e0), ncclInt32, s.peer, ctx->comm, st));
            AFSAI_NCCL_TRY(ncclSend(X->b_val.as<double>() + e0, (e1 - e0), ncclDouble, s.peer, ctx->comm, st));
        }
        AFSAI_NCCL_TRY(grp.end());
    }
    return AFSAI_OK;
}

// G^T of the distributed G.  G is lower triangular, so an entry (i, j) of a local
// row lies either in a local G^T row (j >= b) or in a G^T row owned by a lower
// rank.  Local entries go through the 1-GPU count / scan / scatter path; the
// few entries for each lower rank q are extracted in row order (per-row
// counts, scan, fill) and sent as (col, row, val) triples; received triples
// (from higher ranks) join the local G^T rows, which are then sorted by row.
struct DbgTimer {
    bool on = false;
    cudaStream_t st;
    std::vector<cudaEvent_t> ev;
    std::vector<const char *> nm;
    explicit DbgTimer(cudaStream_t s) : st(s) { on = std::getenv("AFSAI_DEBUG_TIMING") != nullptr; }
    void mark(const char *name) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        ev.push_back(e);
        nm.push_back(name);
    }
    ~DbgTimer() {
        if (!on || ev.empty()) return;
        cudaEventSynchronize(ev.back());
        for (size_t k = 1; k < ev.size(); ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[k - 1], ev[k]);
            std::fprintf(stderr, "[afsai timing] %-28s %8.3f ms\n", nm[k], ms);
        }
        for (auto e : ev) cudaEventDestroy(e);
    }
};

static int dist_transpose(afsai_ctx_t ctx, afsai_factor_t F, const std::vector<int64_t> &bounds,
                          afsai_status_t *status) {
    NvtxRange nv("afsai G^T exchange + transpose");
    cudaStream_t st = ctx->stream;
    DbgTimer dt(st);
    dt.mark("start");
    const int np = ctx->nranks, me = ctx->rank;
    const int64_t b = bounds[me], e = bounds[me + 1], n = F->n_rows;
    const int grid = grid_stream(ctx);
    const int64_t *grp = F->g_rowptr.as<int64_t>();
    const int32_t *gci = F->g_col.as<int32_t>();
    const double *gv = F->g_val.as<double>();
    // ---- outgoing triples, one contiguous buffer per lower rank
    DevBuf rc32, roff, tiles_r;
    AFSAI_CUDA_TRY(rc32.alloc(std::max<int64_t>(n, 1) * 4, st));
    AFSAI_CUDA_TRY(roff.alloc((n + 1) * 8, st));
    AFSAI_CUDA_TRY(tiles_r.alloc(scan_tmp_elems(n) * 8 + 16, st));
    std::vector<int64_t> scnt(np, 0);
    std::vector<DevBuf> sc(np), sr(np), sv(np);
    for (int q = 0; q < me; ++q) {
        band_count_kernel<<<grid, 256, 0, st>>>(n, grp, gci, bounds[q], bounds[q + 1], rc32.as<int32_t>());
        AFSAI_CUDA_TRY(exclusive_scan(rc32.as<int32_t>(), n, roff.as<int64_t>(), tiles_r.as<int64_t>(), st,
                                      &ctx->launches));
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&scnt[q], roff.as<int64_t>() + n, 8, cudaMemcpyDeviceToHost, st));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
        AFSAI_CUDA_TRY(sc[q].alloc(std::max<int64_t>(scnt[q], 1) * 4, st));
        AFSAI_CUDA_TRY(sr[q].alloc(std::max<int64_t>(scnt[q], 1) * 4, st));
        AFSAI_CUDA_TRY(sv[q].alloc(std::max<int64_t>(scnt[q], 1) * 8, st));
        band_fill_kernel<<<grid, 256, 0, st>>>(n, grp, gci, gv, F->row_begin, bounds[q], bounds[q + 1],
                                               roff.as<int64_t>(), sc[q].as<int32_t>(), sr[q].as<int32_t>(),
                                               sv[q].as<double>());
        ctx->launches += 2;
    }
    dt.mark("extract remote");
    // ---- exchange counts (each rank sends to lower ranks, receives from higher ranks)
    DevBuf dcnt;
    AFSAI_CUDA_TRY(dcnt.alloc(2 * np * 8, st));
    AFSAI_CUDA_TRY(cudaMemcpyAsync(dcnt.p, scnt.data(), np * 8, cudaMemcpyHostToDevice, st));
    {
        KTimer kt(ctx, AFSAI_K_COMM);
        NcclGroup grp;
        AFSAI_NCCL_TRY(grp.start());
        for (int q = 0; q < me; ++q) AFSAI_NCCL_TRY(ncclSend(dcnt.as<int64_t>() + q, 1, ncclInt64, q, ctx->comm, st));
        for (int q = me + 1; q < np; ++q)
            AFSAI_NCCL_TRY(ncclRecv(dcnt.as<int64_t>() + np + q, 1, ncclInt64, q, ctx->comm, st));
        AFSAI_NCCL_TRY(grp.end());
    }
    std::vector<int64_t> rcnt(np, 0), hall(2 * np);
    AFSAI_CUDA_TRY(cudaMemcpyAsync(hall.data(), dcnt.p, 2 * np * 8, cudaMemcpyDeviceToHost, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    int64_t total_r = 0;
    std::vector<int64_t> rbase(np, 0);
    for (int q = me + 1; q < np; ++q) {
        rcnt[q] = hall[np + q];
        rbase[q] = total_r;
        total_r += rcnt[q];
    }
    DevBuf rc_, rr_, rv_;
    AFSAI_CUDA_TRY(rc_.alloc(std::max<int64_t>(total_r, 1) * 4, st));
    AFSAI_CUDA_TRY(rr_.alloc(std::max<int64_t>(total_r, 1) * 4, st));
    AFSAI_CUDA_TRY(rv_.alloc(std::max<int64_t>(total_r, 1) * 8, st));
    {
        KTimer kt(ctx, AFSAI_K_COMM);
        NcclGroup grp;
        AFSAI_NCCL_TRY(grp.start());
        for (int q = 0; q < me; ++q)
            if (scnt[q] > 0) {
                AFSAI_NCCL_TRY(ncclSend(sc[q].p, scnt[q], ncclInt32, q, ctx->comm, st));
                AFSAI_NCCL_TRY(ncclSend(sr[q].p, scnt[q], ncclInt32, q, ctx->comm, st));
                AFSAI_NCCL_TRY(ncclSend(sv[q].p, scnt[q], ncclDouble, q, ctx->comm, st));
            }
        for (int q = me + 1; q < np; ++q)
            if (rcnt[q] > 0) {
                AFSAI_NCCL_TRY(ncclRecv(rc_.as<int32_t>() + rbase[q], rcnt[q], ncclInt32, q, ctx->comm, st));
                AFSAI_NCCL_TRY(ncclRecv(rr_.as<int32_t>() + rbase[q], rcnt[q], ncclInt32, q, ctx->comm, st));
                AFSAI_NCCL_TRY(ncclRecv(rv_.as<double>() + rbase[q], rcnt[q], ncclDouble, q, ctx->comm, st));
            }
        AFSAI_NCCL_TRY(grp.end());
    }
    dt.mark("exchange");
    // ---- local G^T rows [b, e): local entries + received triples
    const int64_t n_out = e - b;
    DevBuf cnt, tiles, tcol, tval;
    AFSAI_CUDA_TRY(cnt.alloc(std::max<int64_t>(n_out, 1) * 4, st));
    AFSAI_CUDA_TRY(tiles.alloc(scan_tmp_elems(n_out) * 8 + 16, st));
    AFSAI_CUDA_TRY(F->t_rowptr.alloc((n_out + 1) * 8, st));
    AFSAI_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, std::max<int64_t>(n_out, 1) * 4, st));
    KTimer kt(ctx, AFSAI_K_TRANSPOSE);
    count_cols_kernel<<<grid, 256, 0, st>>>(F->nnz_G, gci, b, n_out, cnt.as<int32_t>());
    count_triples_kernel<<<grid, 256, 0, st>>>(total_r, rc_.as<int32_t>(), b, n_out, cnt.as<int32_t>());
    ctx->launches += 2;
    AFSAI_CUDA_TRY(exclusive_scan(cnt.as<int32_t>(), n_out, F->t_rowptr.as<int64_t>(), tiles.as<int64_t>(), st,
                                  &ctx->launches));
    dt.mark("count+scan");
    int64_t total = 0;
    AFSAI_CUDA_TRY(cudaMemcpyAsync(&total, F->t_rowptr.as<int64_t>() + n_out, 8, cudaMemcpyDeviceToHost, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    F->nnz_Gt = total;
    if (F->t_col.alloc(std::max<int64_t>(total, 1) * 4, st) != cudaSuccess ||
        F->t_val.alloc(std::max<int64_t>(total, 1) * 8, st) != cudaSuccess ||
        tcol.alloc(std::max<int64_t>(total, 1) * 4, st) != cudaSuccess ||
        tval.alloc(std::max<int64_t>(total, 1) * 8, st) != cudaSuccess)
        return set_status(status, AFSAI_ENOMEM, "G^T");
    AFSAI_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, std::max<int64_t>(n_out, 1) * 4, st));
    dt.mark("alloc");
    scatter_t_kernel<<<grid, 256, 0, st>>>(n, grp, gci, gv, F->row_begin, b, n_out, F->t_rowptr.as<int64_t>(),
                                           cnt.as<int32_t>(), tcol.as<int32_t>(), tval.as<double>());
    scatter_triples_kernel<<<grid, 256, 0, st>>>(total_r, rc_.as<int32_t>(), rr_.as<int32_t>(), rv_.as<double>(), b,
                                                 n_out, F->t_rowptr.as<int64_t>(), cnt.as<int32_t>(),
                                                 tcol.as<int32_t>(), tval.as<double>());
    dt.mark("scatter");
    sort_gt_rows(n_out, F->t_rowptr.as<int64_t>(), tcol.as<int32_t>(), tval.as<double>(), F->t_col.as<int32_t>(),
                 F->t_val.as<double>(), grid, st, &ctx->launches);
    dt.mark("sort");
    ctx->launches += 2;
    AFSAI_CUDA_TRY(cudaGetLastError());
    return AFSAI_OK;
}

// ---- bounded-communication set-up
// owner of a global row / column: the rank q with bounds[q] <= x < bounds[q+1]
__device__ __forceinline__ int owner_of(const int64_t *bounds, int np, int64_t x) {
    int lo = 0, hi = np;  // bounds[lo] <= x < bounds[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (bounds[mid] <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

// this rank's row of the communication matrix A-hat: bit q set iff a local row has
// a column owned by rank q
__global__ void comm_row_kernel(const int64_t *rowptr, const int32_t *col, int64_t base, int64_t n_rows,
                                const int64_t *bounds, int np, unsigned long long *mask) {
    unsigned long long m = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x)
        for (int64_t e = rowptr[r] - base; e < rowptr[r + 1] - base; ++e) m |= 1ull << owner_of(bounds, np, col[e]);
    atomicOr(mask, m);
}

// N_p = { q <= p : (A-hat^k)_pq != 0 } as a bit mask.  A-hat is gathered from all
// ranks; its diagonal is nonzero (diagonal entries), so A-hat^k's pattern is the
// set of ranks reachable from p in at most k steps (a few boolean products).
static int comm_neighbours(afsai_ctx_t ctx, const DeviceCsr &A, const std::vector<int64_t> &bounds, int k,
                           uint64_t *nmask, afsai_status_t *status) {
    cudaStream_t st = ctx->stream;
    const int np = ctx->nranks;
    if (np > 64) return set_status(status, AFSAI_ELIMIT, "the bounded-communication set-up supports <= 64 ranks");
    DevBuf db, dm;
    AFSAI_CUDA_TRY(db.alloc((np + 1) * sizeof(int64_t), st));
    AFSAI_CUDA_TRY(dm.alloc(sizeof(unsigned long long), st));
    AFSAI_CUDA_TRY(cudaMemcpyAsync(db.p, bounds.data(), (np + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    AFSAI_CUDA_TRY(cudaMemsetAsync(dm.p, 0, sizeof(unsigned long long), st));
    comm_row_kernel<<<grid_stream(ctx), 256, 0, st>>>(A.rowptr, A.col, A.base, A.n_rows, db.as<int64_t>(), np,
                                                      dm.as<unsigned long long>());
    ctx->launches += 1;
    unsigned long long mine = 0;
    AFSAI_CUDA_TRY(cudaMemcpyAsync(&mine, dm.p, sizeof mine, cudaMemcpyDeviceToHost, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<int64_t> rows;  // A-hat, one bit row per rank
    int rc = allgather_i64(ctx, (int64_t)mine, rows, status);
    if (rc) return rc;
    std::vector<uint64_t> ur(rows.begin(), rows.end());
    if (afsai_bounded_stripes(ctx->rank, np, ur.data(), k, nmask) != AFSAI_OK)
        return set_status(status, AFSAI_EINVAL, "bad communication matrix");
    return AFSAI_OK;
}

// keep entry (r, c) of the extended rows iff owner(r) and owner(c) are in nmask:
// X becomes A[I_p, I_p] (rows of the other stripes empty; they are never read)
__global__ void stripe_count_kernel(const int64_t *rowptr, const int32_t *col, int64_t base, int64_t n_rows,
                                    int64_t row_begin, const int64_t *bounds, int np, unsigned long long nmask,
                                    int32_t *cnt) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        int c = 0;
        if ((nmask >> owner_of(bounds, np, r + row_begin)) & 1ull)
            for (int64_t e = rowptr[r] - base; e < rowptr[r + 1] - base; ++e)
                c += (int)((nmask >> owner_of(bounds, np, col[e])) & 1ull);
        cnt[r] = c;
    }
}

__global__ void stripe_fill_kernel(const int64_t *rowptr, const int32_t *col, const double *val, int64_t base,
                                   int64_t n_rows, int64_t row_begin, const int64_t *bounds, int np,
                                   unsigned long long nmask, const int64_t *orp, int32_t *ocol, double *oval) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        if (!((nmask >> owner_of(bounds, np, r + row_begin)) & 1ull)) continue;
        int64_t o = orp[r];
        for (int64_t e = rowptr[r] - base; e < rowptr[r + 1] - base; ++e)
            if ((nmask >> owner_of(bounds, np, col[e])) & 1ull) {
                ocol[o] = col[e];
                oval[o] = val[e];
                ++o;
            }
    }
}

static int truncate_to_stripes(afsai_ctx_t ctx, const DeviceCsr &X, const std::vector<int64_t> &bounds,
                               uint64_t nmask, DeviceCsr *T, afsai_status_t *status) {
    cudaStream_t st = ctx->stream;
    const int np = ctx->nranks;
    const int64_t n = X.n_rows;
    DevBuf db, cnt, tiles;
    AFSAI_CUDA_TRY(db.alloc((np + 1) * sizeof(int64_t), st));
    AFSAI_CUDA_TRY(cudaMemcpyAsync(db.p, bounds.data(), (np + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    AFSAI_CUDA_TRY(cnt.alloc(std::max<int64_t>(n, 1) * sizeof(int32_t), st));
    AFSAI_CUDA_TRY(tiles.alloc(scan_tmp_elems(n) * sizeof(int64_t) + 16, st));
    AFSAI_CUDA_TRY(T->b_rowptr.alloc((n + 1) * sizeof(int64_t), st));
    const int grid = grid_stream(ctx);
    stripe_count_kernel<<<grid, 256, 0, st>>>(X.rowptr, X.col, X.base, n, X.row_begin, db.as<int64_t>(), np, nmask,
                                              cnt.as<int32_t>());
    ctx->launches += 1;
    AFSAI_CUDA_TRY(exclusive_scan(cnt.as<int32_t>(), n, T->b_rowptr.as<int64_t>(), tiles.as<int64_t>(), st,
                                  &ctx->launches));
    int64_t nnz = 0;
    AFSAI_CUDA_TRY(cudaMemcpyAsync(&nnz, T->b_rowptr.as<int64_t>() + n, sizeof nnz, cudaMemcpyDeviceToHost, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    AFSAI_CUDA_TRY(T->b_col.alloc(std::max<int64_t>(nnz, 1) * sizeof(int32_t), st));
    AFSAI_CUDA_TRY(T->b_val.alloc(std::max<int64_t>(nnz, 1) * sizeof(double), st));
    stripe_fill_kernel<<<grid, 256, 0, st>>>(X.rowptr, X.col, X.val, X.base, n, X.row_begin, db.as<int64_t>(), np,
                                             nmask, T->b_rowptr.as<int64_t>(), T->b_col.as<int32_t>(),
                                             T->b_val.as<double>());
    ctx->launches += 1;
    AFSAI_CUDA_TRY(cudaGetLastError());
    T->rowptr = T->b_rowptr.as<int64_t>();
    T->col = T->b_col.as<int32_t>();
    T->val = T->b_val.as<double>();
    T->base = 0;
    T->n_rows = n;
    T->n_cols = X.n_cols;
    T->row_begin = X.row_begin;
    T->nnz = nnz;
    T->staged = true;
    return AFSAI_OK;
}

int dist_setup(afsai_ctx_t ctx, const afsai_csr_t *Ain, const afsai_params_t *p, afsai_factor_t *out,
               afsai_status_t *status) {
    if (!ctx->comm) return set_status(status, AFSAI_ENCCL, "the context's communicator was aborted");
    cudaStream_t st = ctx->stream;
    DeviceCsr A;
    int rc = agree(ctx, stage_csr(ctx, Ain, &A, status), status);
    if (rc) return rc;
    auto *F = new afsai_factor_s();
    F->ctx = ctx;
    F->n_rows = A.n_rows;
    F->n_global = A.n_cols;
    F->row_begin = A.row_begin;
    F->stats.n_rows = A.n_rows;
    auto fail = [&](int code) {
        dist_free(F);
        delete F;
        return code;
    };
    auto *D = new DistState();
    F->dist = D;
    // partition (contiguous, rank order == row order)
    std::vector<int64_t> begins;
    rc = allgather_i64(ctx, A.row_begin, begins, status);
    if (rc) return fail(rc);
    D->bounds.assign(begins.begin(), begins.end());
    D->bounds.push_back(A.n_cols);
    // every rank sees the same bounds, so these two checks agree by themselves
    if (D->bounds[0] != 0)
        return fail(set_status(status, AFSAI_EINVAL, "rank 0's block must start at row 0"));
    for (int q = 0; q < ctx->nranks; ++q)
        if (D->bounds[q + 1] < D->bounds[q])
            return fail(set_status(status, AFSAI_EINVAL, "row blocks must be contiguous in rank order"));
    rc = D->bounds[ctx->rank + 1] != A.row_begin + A.n_rows
             ? set_status(status, AFSAI_EINVAL, "row blocks must tile [0, n) in rank order")
             : AFSAI_OK;
    if ((rc = agree(ctx, rc, status))) return fail(rc);
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[0], st));
    int64_t maxlen = 0;
    rc = agree(ctx, validate_csr(ctx, A, &maxlen, status), status);
    if (rc) return fail(rc);
    rc = allreduce_max(ctx, maxlen, &maxlen, status);  // same kernel plan on every rank
    if (rc) return fail(rc);
    // global bandwidth of A
    DevBuf bw;
    AFSAI_CUDA_TRY(bw.alloc(8, st));
    AFSAI_CUDA_TRY(cudaMemsetAsync(bw.p, 0, 8, st));
    bandwidth_kernel<<<grid_stream(ctx), 256, 0, st>>>(A.rowptr, A.col, A.base, A.n_rows, A.row_begin,
                                                       bw.as<unsigned long long>());
    ctx->launches += 1;
    int64_t hbw = 0;
    AFSAI_CUDA_TRY(cudaMemcpyAsync(&hbw, bw.p, 8, cudaMemcpyDeviceToHost, st));
    AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    rc = allreduce_max(ctx, hbw, &D->betaA, status);
    if (rc) return fail(rc);
    // exact set-up halo: rows [b - kmax*beta, b)
    const int64_t b = A.row_begin, e = b + A.n_rows;
    const int64_t reach = std::min<int64_t>(b, (int64_t)p->nsteps * D->betaA);
    int64_t lo = b - reach;
    // bounded-communication set-up: G-hat <= lower(A-hat^k); the
    // rank gathers the stripes q <= p with (A-hat^k)_pq != 0 and sets up on the
    // principal submatrix A[I_p, I_p] of their rows (entries outside are zero)
    uint64_t nmask = 0;
    if (p->halo_k > 0) {
        rc = agree(ctx, comm_neighbours(ctx, A, D->bounds, p->halo_k, &nmask, status), status);
        if (rc) return fail(rc);
        int q0 = 0;
        while (!((nmask >> q0) & 1ull)) ++q0;
        lo = D->bounds[q0];
    }
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[5], st));
    DeviceCsr X;
    rc = agree(ctx, gather_halo(ctx, A, D->bounds, lo, &X, status), status);
    if (rc) return fail(rc);
    int64_t halo_entries = 0;
    {
        int64_t h0 = 0;
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&h0, X.rowptr + (b - lo), sizeof h0, cudaMemcpyDeviceToHost, st));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
        halo_entries = h0;  // entries of the received rows [lo, b)
    }
    if (p->halo_k > 0) {
        DeviceCsr T;
        rc = agree(ctx, truncate_to_stripes(ctx, X, D->bounds, nmask, &T, status), status);
        if (rc) return fail(rc);
        X = std::move(T);
    }
#ifdef AFSAI_BOUNDS_CHECK
    {   // debug build: the gathered halo-extended matrix must be a valid CSR
        int64_t ml = 0;
        rc = validate_csr(ctx, X, &ml, status);
        if (rc) {
            std::fprintf(stderr, "[afsai rank %d] halo-extended A invalid: %s\n", ctx->rank,
                         status ? status->msg : "?");
            return fail(rc);
        }
    }
#endif
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[6], st));
    F->stats.halo_rows = (int32_t)(b - lo);
    F->stats.halo_bytes = halo_entries * (int64_t)(sizeof(int32_t) + sizeof(double)) + (b - lo) * 4;
    F->stats.halo_mask = (int64_t)nmask;
    rc = agree(ctx, block_rows_to_G(ctx, X, lo, e, b, A.n_rows, p, maxlen, F, status), status);
    if (rc) return fail(rc);
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[3], st));
    rc = agree(ctx, dist_transpose(ctx, F, D->bounds, status), status);
    if (rc) return fail(rc);
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[4], st));
    // G's lower reach (for the r halo of G r and the t halo of G^T t)
    {
        DevBuf gb;
        AFSAI_CUDA_TRY(gb.alloc(8, st));
        AFSAI_CUDA_TRY(cudaMemsetAsync(gb.p, 0, 8, st));
        bandwidth_kernel<<<grid_stream(ctx), 256, 0, st>>>(F->g_rowptr.as<int64_t>(), F->g_col.as<int32_t>(), 0,
                                                           F->n_rows, b, gb.as<unsigned long long>());
        ctx->launches += 1;
        int64_t g = 0;
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&g, gb.p, 8, cudaMemcpyDeviceToHost, st));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
        rc = allreduce_max(ctx, g, &D->betaG, status);
        if (rc) return fail(rc);
    }
    // per-iteration halo plans (every rank derives all ranges from the bounds)
    const int np = ctx->nranks;
    const int64_t n = A.n_cols;
    std::vector<int64_t> lo_(np), hi_(np);
    for (int q = 0; q < np; ++q) {
        lo_[q] = std::max<int64_t>(0, D->bounds[q] - D->betaA);
        hi_[q] = std::min<int64_t>(n, D->bounds[q + 1] + D->betaA);
    }
    D->planA = make_range_plan(ctx->rank, np, D->bounds, lo_, hi_);
    for (int q = 0; q < np; ++q) {
        lo_[q] = std::max<int64_t>(0, D->bounds[q] - D->betaG);
        hi_[q] = D->bounds[q + 1];
    }
    D->planG = make_range_plan(ctx->rank, np, D->bounds, lo_, hi_);
    for (int q = 0; q < np; ++q) {
        lo_[q] = D->bounds[q];
        hi_[q] = std::min<int64_t>(n, D->bounds[q + 1] + D->betaG);
    }
    D->planT = make_range_plan(ctx->rank, np, D->bounds, lo_, hi_);
    F->stats.nnz_Gt = F->nnz_Gt;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[5], ctx->ev[6]);
    F->stats.ms_halo = ms;
    cudaEventElapsedTime(&ms, ctx->ev[3], ctx->ev[4]);
    F->stats.ms_transpose = ms;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[4]);
    F->stats.ms_total = ms;
    F->g_lo = std::max<int64_t>(0, b - D->betaG);
    F->gt_hi = std::min<int64_t>(n, e + D->betaG);
    if (A.staged) {
        F->src_rowptr = Ain->rowptr;
        F->src_col = Ain->col;
        F->src_val = Ain->val;
        F->staged_A = std::move(A);
    }
    *out = F;
    return AFSAI_OK;
}

// extended vectors of the factor: p_ext (A plan) | r_ext (G plan) | t_ext (G^T plan)
static int ensure_ext(afsai_ctx_t ctx, afsai_factor_t F, double **pe, double **re, double **te,
                      afsai_status_t *status) {
    DistState *D = dstate(F);
    const int64_t nA = D->planA.hi - D->planA.lo, nG = D->planG.hi - D->planG.lo, nT = D->planT.hi - D->planT.lo;
    const size_t need = (size_t)(nA + nG + nT) * sizeof(double);
    if (D->ext.bytes < need) {
        AFSAI_CUDA_TRY(D->ext.alloc(need, ctx->stream));
        AFSAI_CUDA_TRY(cudaMemsetAsync(D->ext.p, 0, need, ctx->stream));
    }
    *pe = D->ext.as<double>();
    *re = *pe + nA;
    *te = *re + nG;
    return AFSAI_OK;
}

static SpmvArgs sargs(int64_t n, const int64_t *rp, const int32_t *ci, const double *v, const double *x, int64_t xoff,
                      double *y) {
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

// t = G r (r in r_ext), z = G^T t (t in t_ext); halos for r and t; optional dot(z, w) -> st->sum[2]
static int dist_apply_ext(afsai_ctx_t ctx, afsai_factor_t F, double *re, double *te, double *z, const double *w,
                          PcgWork *pw, afsai_status_t *status) {
    DistState *D = dstate(F);
    cudaStream_t st = ctx->stream;
    const int64_t n = F->n_rows, b = F->row_begin;
    const int grid = grid_stream(ctx);
    {
        KTimer kt(ctx, AFSAI_K_COMM);
        AFSAI_NCCL_TRY(range_exchange(D->planG, re, sizeof(double), ctx->comm, st));
    }
    SpmvArgs a = sargs(n, F->g_rowptr.as<int64_t>(), F->g_col.as<int32_t>(), F->g_val.as<double>(), re, D->planG.lo,
                       te + (b - D->planT.lo));
    if (pw) a.st = pw->state.as<PcgState>();
    {
        KTimer kt(ctx, AFSAI_K_SPMV_G);
        launch_spmv(a, 0, spmv_group_width((double)F->nnz_G / std::max<int64_t>(n, 1), 1), grid, st);
    }
    {
        KTimer kt(ctx, AFSAI_K_COMM);
        AFSAI_NCCL_TRY(range_exchange(D->planT, te, sizeof(double), ctx->comm, st));
    }
    SpmvArgs c = sargs(n, F->t_rowptr.as<int64_t>(), F->t_col.as<int32_t>(), F->t_val.as<double>(), te, D->planT.lo,
                       z);
    int mode = 0;
    if (pw) {
        c.st = pw->state.as<PcgState>();
        c.w = w;
        c.partials = pw->parts.as<double>();
        c.counter = pw->counter.as<unsigned>();
        c.sum_idx = 2;
        mode = 4;
    }
    {
        KTimer kt(ctx, AFSAI_K_SPMV_GT);
        launch_spmv(c, mode, spmv_group_width((double)F->nnz_Gt / std::max<int64_t>(n, 1), 2), grid, st);
    }
    ctx->launches += 2;
    AFSAI_CUDA_TRY(cudaGetLastError());
    return AFSAI_OK;
}

int dist_apply(afsai_ctx_t ctx, afsai_factor_t F, const double *r, double *z, afsai_status_t *status) {
    if (!ctx->comm) return set_status(status, AFSAI_ENCCL, "the context's communicator was aborted");
    if (!F->dist) return set_status(status, AFSAI_EINVAL, "factor was not built on this communicator");
    DistState *D = dstate(F);
    cudaStream_t st = ctx->stream;
    const int64_t n = F->n_rows, b = F->row_begin;
    double *pe, *re, *te;
    int rc = ensure_ext(ctx, F, &pe, &re, &te, status);
    if (rc) return rc;
    AFSAI_CUDA_TRY(cudaMemcpyAsync(re + (b - D->planG.lo), r, n * sizeof(double), cudaMemcpyDefault, st));
    const bool zdev = is_device_ptr(z);
    DevBuf zb;
    double *zd = z;
    if (!zdev) {
        AFSAI_CUDA_TRY(zb.alloc(std::max<int64_t>(n, 1) * sizeof(double), st));
        zd = zb.as<double>();
    }
    rc = dist_apply_ext(ctx, F, re, te, zd, nullptr, nullptr, status);
    if (rc) return rc;
    if (!zdev) {
        AFSAI_CUDA_TRY(cudaMemcpyAsync(z, zd, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        AFSAI_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return AFSAI_OK;
}

// PCG on N GPUs (R12, §6): same recurrence as local_pcg; dot products
// are reduced locally by the producing kernel and all-reduced: p.q, then r.r and
// r.z together (two all-reduces per iteration).
int dist_pcg(afsai_ctx_t ctx, const afsai_csr_t *Ain, afsai_factor_t F, const double *b_in, double *x, double tol,
             int32_t max_iters, afsai_pcg_report_t *rep, afsai_status_t *status) {
    if (!ctx->comm) return set_status(status, AFSAI_ENCCL, "the context's communicator was aborted");
    if (!F->dist) return set_status(status, AFSAI_EINVAL, "factor was not built on this communicator");
    DistState *D = dstate(F);
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
    const int64_t n = A.n_rows, b = A.row_begin;
    PcgWork &W = F->pcg;
    int rc = W.ensure(ctx, n, status);
    if (rc) return rc;
    double *pe, *re, *te;
    rc = ensure_ext(ctx, F, &pe, &re, &te, status);
    if (rc) return rc;
    double *V = W.vec.as<double>();
    double *q = V + n, *z = V + 3 * n, *xs = V + 5 * n;
    double *p = pe + (b - D->planA.lo);  // local parts of the extended vectors
    double *r = re + (b - D->planG.lo);
    const bool bdev = is_device_ptr(b_in), xdev = is_device_ptr(x);
    DevBuf bb;
    const double *bd = b_in;
    if (!bdev) {
        AFSAI_CUDA_TRY(bb.alloc(std::max<int64_t>(n, 1) * sizeof(double), st));
        AFSAI_CUDA_TRY(cudaMemcpyAsync(bb.p, b_in, n * sizeof(double), cudaMemcpyHostToDevice, st));
        bd = bb.as<double>();
    }
    double *xd = xdev ? x : xs;
    PcgState *S = W.state.as<PcgState>();
    double *parts = W.parts.as<double>();
    unsigned *cnt = W.counter.as<unsigned>();
    const int grid = grid_stream(ctx);
    const int64_t *arp = A.rowptr;
    const int32_t *aci = A.col - A.base;
    const double *av = A.val - A.base;
    const int wA = spmv_group_width((double)A.nnz / std::max<int64_t>(n, 1), 0);
    auto allreduce = [&](int k) -> int {
        KTimer kt(ctx, AFSAI_K_COMM);
        AFSAI_NCCL_TRY(ncclAllReduce(&S->sum[k], &S->sum[k], 1, ncclDouble, ncclSum, ctx->comm, st));
        return AFSAI_OK;
    };
    auto allreduce2 = [&](int k) -> int {  // sum[k], sum[k+1]
        KTimer kt(ctx, AFSAI_K_COMM);
        AFSAI_NCCL_TRY(ncclAllReduce(&S->sum[k], &S->sum[k], 2, ncclDouble, ncclSum, ctx->comm, st));
        return AFSAI_OK;
    };
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[5], st));
    {
        KTimer kt(ctx, AFSAI_K_VECTOR);
        launch_pcg_init_dist(n, bd, xd, r, parts, cnt, S, grid, st);
    }
    if ((rc = allreduce(1))) return rc;
    rc = dist_apply_ext(ctx, F, re, te, z, r, &W, status);  // z = M^-1 r, sum[2] = r.z
    if (rc) return rc;
    if ((rc = allreduce(2))) return rc;
    launch_pcg_start_dist(S, st);
    {
        KTimer kt(ctx, AFSAI_K_VECTOR);
        launch_pcg_update_p_dist(n, p, z, S, 1, grid, st);
    }
    ctx->launches += 3;
    PcgState hs{};
    const int kPoll = 8;
    int it = 0;
    for (;;) {
        for (int k = 0; k < kPoll && it < max_iters; ++k, ++it) {
            {
                KTimer kt(ctx, AFSAI_K_COMM);
                AFSAI_NCCL_TRY(range_exchange(D->planA, pe, sizeof(double), ctx->comm, st));
            }
            SpmvArgs aq = sargs(n, arp, aci, av, pe, D->planA.lo, q);
            aq.w = p;
            aq.partials = parts;
            aq.counter = cnt;
            aq.st = S;
            aq.sum_idx = 0;
            {
                KTimer kt(ctx, AFSAI_K_SPMV_A);
                launch_spmv(aq, 4, wA, grid, st);  // q = A p, sum[0] = p.q
            }
            if ((rc = allreduce(0))) return rc;
            {
                KTimer kt(ctx, AFSAI_K_VECTOR);
                launch_pcg_axpy_dist(n, xd, r, p, q, parts, cnt, S, grid, st);  // sum[1] = r.r
            }
            rc = dist_apply_ext(ctx, F, re, te, z, r, &W, status);  // sum[2] = r.z
            if (rc) return rc;
            // r.r and r.z in one all-reduce; the convergence test on r.r follows it
            // (same value, same iteration count; the converged iteration's apply runs)
            if ((rc = allreduce2(1))) return rc;
            launch_pcg_check_dist(S, tol, max_iters, st);
            {
                KTimer kt(ctx, AFSAI_K_VECTOR);
                launch_pcg_update_p_dist(n, p, z, S, 0, grid, st);
            }
            launch_pcg_rz_dist(S, st);
            ctx->launches += 5;
        }
        AFSAI_CUDA_TRY(cudaGetLastError());
        AFSAI_CUDA_TRY(cudaMemcpyAsync(&hs, S, sizeof hs, cudaMemcpyDeviceToHost, st));
        if ((rc = sync_poll(ctx, status))) return rc;
        if (hs.done || it >= max_iters) break;
    }
    AFSAI_CUDA_TRY(cudaEventRecord(ctx->ev[6], st));
    // explicit residual ||b - A x||: x into p_ext for its halo
    AFSAI_CUDA_TRY(cudaMemcpyAsync(p, xd, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    {
        KTimer kt(ctx, AFSAI_K_COMM);
        AFSAI_NCCL_TRY(range_exchange(D->planA, pe, sizeof(double), ctx->comm, st));
    }
    {
        SpmvArgs ax = sargs(n, arp, aci, av, pe, D->planA.lo, q);
        launch_spmv(ax, 0, wA, grid, st);
        launch_residual(n, bd, q, parts, cnt, &S->sum[3], grid, st);
        ctx->launches += 2;
    }
    if ((rc = allreduce(3))) return rc;
    AFSAI_CUDA_TRY(cudaMemcpyAsync(&hs, S, sizeof hs, cudaMemcpyDeviceToHost, st));
    if (!xdev) AFSAI_CUDA_TRY(cudaMemcpyAsync(x, xd, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    if ((rc = sync_poll(ctx, status))) return rc;
    const bool conv = hs.done == 1 || hs.bnorm2 == 0.0;
    if (rep) {
        rep->iters = hs.iters;
        rep->converged = conv;
        rep->rel_res = hs.rel;
        rep->true_rel_res = hs.bnorm2 > 0 ? std::sqrt(hs.sum[3]) / std::sqrt(hs.bnorm2) : 0.0;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[5], ctx->ev[6]);
        rep->ms_solve = ms;
        rep->ms_per_iter = hs.iters > 0 ? ms / hs.iters : 0.0;
    }
    return conv ? AFSAI_OK : set_status(status, AFSAI_ENOTCONV, "PCG reached max_iters");
}

// ---- host-side plan helper exported for tests (no GPU needed)
int plan_ranges(int32_t me, int32_t nranks, const int64_t *bounds, const int64_t *lo, const int64_t *hi,
                int64_t *out, int32_t max_out) {
    std::vector<int64_t> B(bounds, bounds + nranks + 1), L(lo, lo + nranks), Hh(hi, hi + nranks);
    RangePlan P = make_range_plan(me, nranks, B, L, Hh);
    int32_t k = 0;
    for (const Seg &s : P.sends) {
        if (k >= max_out) return -1;
        out[4 * k] = 0; out[4 * k + 1] = s.peer; out[4 * k + 2] = s.begin; out[4 * k + 3] = s.count;
        ++k;
    }
    for (const Seg &s : P.recvs) {
        if (k >= max_out) return -1;
        out[4 * k] = 1; out[4 * k + 1] = s.peer; out[4 * k + 2] = s.begin; out[4 * k + 3] = s.count;
        ++k;
    }
    return k;
}

}  // namespace afsai

extern "C" {

int afsai_setup_block(afsai_ctx_t ctx, const afsai_csr_t *Ain, int64_t row_lo, int64_t n_rows,
                      const afsai_params_t *p, afsai_factor_t *out, afsai_status_t *status) {
    using namespace afsai;
    set_status(status, AFSAI_OK, "");
    if (!ctx || !Ain || !p || !out) return set_status(status, AFSAI_EINVAL, "null argument");
    const int64_t a_lo = Ain->row_begin, a_hi = Ain->row_begin + Ain->n_rows;
    if (Ain->n_rows < 1 || Ain->n_cols < 1 || a_hi > Ain->n_cols || n_rows < 0 || row_lo < a_lo ||
        row_lo + n_rows > a_hi || !Ain->rowptr || !Ain->col || !Ain->val)
        return set_status(status, AFSAI_EINVAL, "block must lie inside A_ext");
    if (p->nsteps < 0 || p->s < 1 || p->s > AFSAI_MAX_S || !(p->eps >= 0.0 && p->eps < 1.0) || p->max_row_nnz < 1 ||
        (p->precision != AFSAI_PREC_FP64 && p->precision != AFSAI_PREC_FP32))
        return set_status(status, AFSAI_EINVAL, "params out of range");
    if (std::min<int64_t>((int64_t)p->nsteps * p->s, (int64_t)p->max_row_nnz - 1) > AFSAI_MAX_MMAX)
        return set_status(status, AFSAI_ELIMIT, "min(nsteps*s, max_row_nnz-1) exceeds AFSAI_MAX_MMAX (128)");
    DeviceCsr A;
    int rc = stage_csr(ctx, Ain, &A, status);
    if (rc) return rc;
    int64_t maxlen = 0;
    rc = validate_csr(ctx, A, &maxlen, status);
    if (rc) return rc;
    auto *F = new afsai_factor_s();
    F->ctx = ctx;
    F->n_rows = n_rows;
    F->n_global = Ain->n_cols;
    F->row_begin = row_lo;
    F->stats.n_rows = n_rows;
    F->block = true;
    rc = block_rows_to_G(ctx, A, a_lo, a_hi, row_lo, n_rows, p, maxlen, F, status);
    if (rc) {
        delete F;
        return rc;
    }
    *out = F;
    return AFSAI_OK;
}

int afsai_bounded_stripes(int32_t me, int32_t nranks, const uint64_t *ahat_rows, int32_t k, uint64_t *mask) {
    if (nranks < 1 || nranks > 64 || me < 0 || me >= nranks || k < 0 || !ahat_rows || !mask) return AFSAI_EINVAL;
    // (A-hat^k)_me,q != 0  <=>  q reachable from me in at most k steps (A-hat has a nonzero diagonal)
    uint64_t reach = 1ull << me;
    for (int t = 0; t < k; ++t) {
        uint64_t nx = reach;
        for (int q = 0; q < nranks; ++q)
            if ((reach >> q) & 1ull) nx |= ahat_rows[q];
        reach = nx;
    }
    const uint64_t lower = me == 63 ? ~0ull : ((2ull << me) - 1ull);
    *mask = reach & lower;
    return AFSAI_OK;
}

int afsai_plan_ranges(int32_t me, int32_t nranks, const int64_t *bounds, const int64_t *lo, const int64_t *hi,
                      int64_t *out, int32_t max_out) {
    if (nranks < 1 || me < 0 || me >= nranks || !bounds || !lo || !hi || !out) return -1;
    return afsai::plan_ranges(me, nranks, bounds, lo, hi, out, max_out);
}

}  // extern "C"
