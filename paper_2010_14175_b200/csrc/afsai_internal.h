// Internal declarations of libafsai_b200.so (not part of the C ABI).
// The public ABI is include/afsai.h; this header is shared only by the
// library's own translation units (never by oracle/).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/afsai.h"

namespace afsai {

constexpr int kWarp = 32;
constexpr int kMaxGroup = 4;  // new rows bordered in lockstep

struct Status {
    int code = AFSAI_OK;
    int64_t row = -1;
    int32_t step = -1;
    std::string msg;
};

// Fill the optional caller status struct.
int set_status(afsai_status_t *st, int code, const std::string &msg, int64_t row = -1, int32_t step = -1);

#define AFSAI_CUDA_TRY(expr)                                                                        \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            return ::afsai::set_status(status, AFSAI_ECUDA,                                         \
                                       std::string(#expr " failed at ") + __FILE__ ":" +             \
                                           std::to_string(__LINE__) + ": " + cudaGetErrorString(_e));  \
    } while (0)

#define AFSAI_NCCL_TRY(expr)                                                                        \
    do {                                                                                            \
        ncclResult_t _r = (expr);                                                                   \
        if (_r != ncclSuccess)                                                                      \
            return ::afsai::set_status(status, AFSAI_ENCCL,                                         \
                                       std::string(#expr " failed: ") + ncclGetErrorString(_r));    \
    } while (0)

// The library's own stream-ordered memory pool on the current device (created by
// the first context on the device; the device's default pool is never touched).
cudaMemPool_t library_pool();

// Stream-ordered device buffer (allocated from library_pool() on the context stream).
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    cudaStream_t stream = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept { *this = std::move(o); }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p; bytes = o.bytes; stream = o.stream;
            o.p = nullptr; o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    cudaError_t alloc(size_t nbytes, cudaStream_t s) {
        release();
        stream = s;
        bytes = nbytes;
        if (nbytes == 0) return cudaSuccess;
        cudaMemPool_t pool = library_pool();
        return pool ? cudaMallocFromPoolAsync(&p, nbytes, pool, s) : cudaMallocAsync(&p, nbytes, s);
    }
    void release() {
        if (p) cudaFreeAsync(p, stream);
        p = nullptr;
        bytes = 0;
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// A device view of a CSR (row block): entries of local row r are
// [rowptr[r] - base, rowptr[r+1] - base) of col/val.
struct DeviceCsr {
    int64_t n_rows = 0, n_cols = 0, row_begin = 0, nnz = 0, base = 0;
    const int64_t *rowptr = nullptr;
    const int32_t *col = nullptr;
    const double *val = nullptr;
    bool staged = false;
    DevBuf b_rowptr, b_col, b_val;  // owned copies when staged from host
};

// Scratch of one afsai_setup call.
struct SetupWork {
    DevBuf scol, sval, nnz_row, err, retry, retry_count, work, counters;
    DevBuf retried;          // global rows the first pass overflowed (recomputed with larger tables)
    int64_t n_retried = 0;
    int32_t *steps = nullptr, *reason = nullptr;  // point into the factor
    int alloc(afsai_ctx_t ctx, int64_t n, int32_t mmax, afsai_status_t *status);
    int check_error(afsai_ctx_t ctx, afsai_status_t *status);
    int read_stats(afsai_ctx_t ctx, afsai_setup_stats_t *s, afsai_status_t *status);
};

// PCG workspace cached in the factor.
struct PcgWork {
    DevBuf vec, parts, counter, state, halo;
    int64_t n_alloc = 0;
    int nparts = 0;
    int ensure(afsai_ctx_t ctx, int64_t n, afsai_status_t *status);
};

}  // namespace afsai

// ---- opaque handle types of the ABI
struct afsai_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    ncclComm_t comm = nullptr;  // null on one GPU
    int32_t rank = 0, nranks = 1;
    int64_t launches = 0;       // kernels launched by this library on this context
    bool pool_held = false;     // holds a reference on the device's library pool
    cudaEvent_t ev[8] = {};
    // optional per-class kernel timing (afsai_ctx_set_timing)
    bool timing = false;
    struct Timed {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Timed> timed;
    std::vector<cudaEvent_t> pool;
    int64_t t_launch[AFSAI_K_NCLASSES] = {};
    double t_ms[AFSAI_K_NCLASSES] = {};
    cudaEvent_t take_event() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};

namespace afsai {
// NVTX range of one phase of a call (header-only NVTX v3: a no-op unless a tool
// such as Nsight Systems is attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// RAII: events around the launches of one kernel class when timing is enabled
struct KTimer {
    afsai_ctx_t c;
    int cls;
    cudaEvent_t a = nullptr;
    KTimer(afsai_ctx_t ctx, int k) : c(ctx), cls(k) {
        if (c->timing) {
            a = c->take_event();
            cudaEventRecord(a, c->stream);
        }
    }
    ~KTimer() {
        if (a) {
            cudaEvent_t b = c->take_event();
            cudaEventRecord(b, c->stream);
            c->timed.push_back({cls, a, b});
        }
    }
};
}  // namespace afsai

// Per-iteration halo plan for one CSR operand on N GPUs.
struct afsai_halo_plan {
    // global rows of the extended vector: [ext_lo, ext_hi) with the local block
    // [row_begin, row_end) inside it; lower part from ranks < rank, upper from ranks > rank
    int64_t ext_lo = 0, ext_hi = 0;
};

struct afsai_factor_s {
    afsai_ctx_t ctx = nullptr;
    int64_t n_rows = 0, n_global = 0, row_begin = 0;
    // G: local rows, global columns
    afsai::DevBuf g_rowptr, g_col, g_val;
    int64_t nnz_G = 0;
    // G^T: local rows (global row index row_begin + k), global columns
    afsai::DevBuf t_rowptr, t_col, t_val;
    int64_t nnz_Gt = 0;
    // per-row trace
    afsai::DevBuf steps, reason;
    afsai::DevBuf retried;       // global rows recomputed by a retry pass (afsai_factor_retried)
    int64_t n_retried = 0;
    afsai_setup_stats_t stats{};
    // multi-GPU: column reach of G below / above the local block (for halos)
    int64_t g_lo = 0;   // min column of G over local rows
    int64_t gt_hi = 0;  // max column + 1 of G^T over local rows
    afsai::PcgWork pcg;
    void *dist = nullptr;  // multi-GPU halo plans (dist.cu)
    bool block = false;    // made by afsai_setup_block: G rows only (no G^T), not appliable
    // device copy of a HOST A staged by afsai_setup, reused by afsai_pcg when
    // it is called with the same host arrays (one H2D of A per solve cycle)
    afsai::DeviceCsr staged_A;
    const void *src_rowptr = nullptr, *src_col = nullptr, *src_val = nullptr;
};

namespace afsai {
bool is_device_ptr(const void *p);
int stage_csr(afsai_ctx_t ctx, const afsai_csr_t *A, DeviceCsr *out, afsai_status_t *status);
int grid_stream(afsai_ctx_t ctx);
int validate_csr(afsai_ctx_t ctx, const DeviceCsr &A, int64_t *max_row_len, afsai_status_t *status);
int run_rows(afsai_ctx_t ctx, const DeviceCsr &Aext, int64_t a_lo, int64_t a_hi, int64_t row_lo, int64_t nrows,
             const afsai_params_t &p, int32_t mmax, int64_t max_row_len, SetupWork &W, afsai_setup_stats_t *stats,
             afsai_status_t *status);
int assemble_G(afsai_ctx_t ctx, afsai_factor_t F, SetupWork &W, int64_t n, int32_t stride, afsai_status_t *status);
int transpose_G(afsai_ctx_t ctx, afsai_factor_t F, int64_t col_lo, int64_t n_out, afsai_status_t *status);
void launch_apply_local(afsai_ctx_t ctx, afsai_factor_t F, const double *r, double *t, double *z, int mode,
                        const double *w, PcgWork *pw);
int local_setup(afsai_ctx_t ctx, const afsai_csr_t *A, const afsai_params_t *p, afsai_factor_t *out,
                afsai_status_t *status);
int local_pcg(afsai_ctx_t ctx, const afsai_csr_t *A, afsai_factor_t F, const double *b, double *x, double tol,
              int32_t max_iters, afsai_pcg_report_t *rep, afsai_status_t *status);
}  // namespace afsai

