// assemble.cu -- input validation, CSR assembly of G (count -> scan -> fill,
// SURVEY §8(a) a7) and the deterministic transpose G^T (a8).
#include <cuda_runtime.h>

#include <cstdint>

#include "afsai_internal.h"
#include "assemble.h"

namespace afsai {

constexpr unsigned kFullA = 0xffffffffu;

// ---------------------------------------------------------------- validation
// One warp per row: columns strictly increasing and in [0, n_cols), diagonal
// present and > 0, values finite.  err gets atomicMin((row << 8) | reason).
__global__ void validate_rows_kernel(const int64_t *rowptr, const int32_t *col, const double *val, int64_t base,
                                     int64_t n_rows, int64_t row_begin, int64_t n_cols,
                                     unsigned long long *err) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nw) {
        const int64_t e0 = rowptr[r] - base, e1 = rowptr[r + 1] - base;
        const int64_t gi = r + row_begin;
        int bad = 0;
        bool diag = false;
        if (e1 < e0) bad = 1;
        for (int64_t e = e0 + lane; e < e1 && !bad; e += 32) {
            const int32_t c = col[e];
            const double v = val[e];
            if (c < 0 || c >= n_cols) bad = 2;
            else if (e > e0 && col[e - 1] >= c) bad = 3;
            else if (!isfinite(v)) bad = 4;
            else if (c == gi) {
                diag = true;
                if (!(v > 0.0)) bad = 5;
            }
        }
        bad = __reduce_max_sync(kFullA, bad);
        const bool has_diag = __any_sync(kFullA, diag);
        if (!bad && !has_diag) bad = 6;
        if (bad && lane == 0) atomicMin(err, ((unsigned long long)gi << 8) | (unsigned long long)bad);
    }
}

// max row length (sizes the per-row candidate table)
__global__ void row_len_max_kernel(const int64_t *rowptr, int64_t n_rows, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long l = (unsigned long long)(rowptr[r + 1] - rowptr[r]);
        m = l > m ? l : m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(kFullA, m, o);
        m = x > m ? x : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// bitwise symmetry (AFSAI_VALIDATE=1): for each stored (i, j) with row j held
// locally, (j, i) must exist with identical bits.
__global__ void symmetry_kernel(const int64_t *rowptr, const int32_t *col, const double *val, int64_t base,
                                int64_t n_rows, int64_t row_begin, unsigned long long *err) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < n_rows; r += nt) {
        const int64_t gi = r + row_begin;
        for (int64_t e = rowptr[r] - base; e < rowptr[r + 1] - base; ++e) {
            const int64_t j = col[e];
            if (j < row_begin || j >= row_begin + n_rows) continue;
            int64_t lo = rowptr[j - row_begin] - base, hi = rowptr[j - row_begin + 1] - base;
            bool ok = false;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (col[mid] < gi) lo = mid + 1;
                else hi = mid;
            }
            if (lo < rowptr[j - row_begin + 1] - base && col[lo] == gi)
                ok = (__double_as_longlong(val[lo]) == __double_as_longlong(val[e]));
            if (!ok) atomicMin(err, ((unsigned long long)gi << 8) | 7ull);
        }
    }
}

// A_s = single(A) for the fp32 set-up (the paper casts on the
// host before the copy; here A is already on the device).  Round to nearest even
// (__double2float_rn, numpy's astype(float32)).  Flags (lowest row) a value that
// overflows to +-inf or a diagonal that is no longer > 0.
__global__ void cast_rows_f32_kernel(const int64_t *rowptr, const int32_t *col, const double *val, int64_t base,
                                     int64_t n_rows, int64_t row_begin, float *out, unsigned long long *err) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nw) {
        const int64_t e0 = rowptr[r] - base, e1 = rowptr[r + 1] - base;
        bool bad = false;
        for (int64_t e = e0 + lane; e < e1; e += 32) {
            const float f = __double2float_rn(val[e]);
            out[e] = f;
            bad |= isinf(f) || (col[e] == r + row_begin && !(f > 0.0f));
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(err, (unsigned long long)(r + row_begin));
    }
}

// ---------------------------------------------------------------- exclusive scan
// int32 counts -> int64 offsets, out[n] = total.  Three passes over tiles of
// kScanTile elements: tile sums, scan of tile sums (one block), tile scans.
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t *total) {
    __shared__ int64_t warp_tot[kScanThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFullA, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t w = (lane < kScanThreads / 32) ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(kFullA, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kScanThreads / 32) warp_tot[lane] = w;
    }
    __syncthreads();
    const int64_t before = (wid > 0 ? warp_tot[wid - 1] : 0) + (x - v);
    *total = warp_tot[kScanThreads / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void scan_tile_sums(const int32_t *in, int64_t n, int64_t *tile_sums) {
    const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
    int64_t s = 0;
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t idx = t0 + (int64_t)k * kScanThreads + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    int64_t tot;
    block_exclusive_scan(s, &tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void scan_tile_offsets(int64_t *tile_sums, int64_t ntiles) {
    // single block, sequential chunks
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < ntiles; c0 += kScanThreads) {
        const int64_t idx = c0 + threadIdx.x;
        const int64_t v = idx < ntiles ? tile_sums[idx] : 0;
        int64_t tot;
        const int64_t ex = block_exclusive_scan(v, &tot);
        if (idx < ntiles) tile_sums[idx] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) tile_sums[ntiles] = carry;
}

__global__ void scan_tiles(const int32_t *in, int64_t n, const int64_t *tile_off, int64_t *out) {
    // each thread owns kScanItems consecutive elements
    const int64_t t0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int32_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (t0 + k < n) ? in[t0 + k] : 0;
        s += v[k];
    }
    int64_t tot;
    int64_t ex = block_exclusive_scan(s, &tot) + tile_off[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (t0 + k < n) out[t0 + k] = ex;
        ex += v[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = tile_off[gridDim.x];
}

cudaError_t exclusive_scan(const int32_t *in, int64_t n, int64_t *out, int64_t *tmp_tiles, cudaStream_t st,
                           int64_t *launches) {
    const int64_t ntiles = (n + kScanTile - 1) / kScanTile > 0 ? (n + kScanTile - 1) / kScanTile : 1;
    scan_tile_sums<<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, n, tmp_tiles);
    scan_tile_offsets<<<1, kScanThreads, 0, st>>>(tmp_tiles, ntiles);
    scan_tiles<<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, n, tmp_tiles, out);
    *launches += 3;
    return cudaGetLastError();
}

int64_t scan_tmp_elems(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

// ---------------------------------------------------------------- fill G
// warp per row: copy the fixed-stride scratch row (already sorted) into CSR.
__global__ void fill_rows_kernel(int64_t n_rows, const int32_t *scol, const double *sval, int32_t stride,
                                 const int64_t *rowptr, int32_t *col, double *val) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nw) {
        const int64_t o = rowptr[r];
        const int k = (int)(rowptr[r + 1] - o);
        const int32_t *sc = scol + r * stride;
        const double *sv = sval + r * stride;
        for (int t = lane; t < k; t += 32) {
            col[o + t] = sc[t];
            val[o + t] = sv[t];
        }
    }
}

// ---------------------------------------------------------------- transpose
// count entries per column (columns mapped to [0, n_out) by subtracting col_lo)
__global__ void count_cols_kernel(int64_t nnz, const int32_t *col, int64_t col_lo, int64_t n_out, int32_t *cnt) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = tid; e < nnz; e += nt) {
        const int64_t c = (int64_t)col[e] - col_lo;
        if (c >= 0 && c < n_out) atomicAdd(&cnt[c], 1);
    }
}

// scatter entry (row, c, v) to rowptr_t[c] + cursor; order within a row fixed later
__global__ void scatter_t_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, const double *val,
                                 int64_t row_begin, int64_t col_lo, int64_t n_out, const int64_t *t_rowptr,
                                 int32_t *cursor, int32_t *t_col, double *t_val) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nw) {
        for (int64_t e = rowptr[r] + lane; e < rowptr[r + 1]; e += 32) {
            const int64_t c = (int64_t)col[e] - col_lo;
            if (c < 0 || c >= n_out) continue;
            const int p = atomicAdd(&cursor[c], 1);
            t_col[t_rowptr[c] + p] = (int32_t)(r + row_begin);
            t_val[t_rowptr[c] + p] = val[e];
        }
    }
}

// Rows of G^T are sorted by source row (C10): the scatter above places entries
// in atomic (arbitrary) order.  Short rows (<= kLongRow entries, every stencil and
// FE row) are rank-sorted by one warp; a hub column can make a G^T row as long
// as n, so longer rows take an O(k log^2 k) CTA sort (sort_long_rows_kernel).
constexpr int kLongRow = 256;

// warp per short row of G^T: rank sort by column (row index of G), ascending
__global__ void sort_rows_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *in_col, const double *in_val,
                                 int32_t *out_col, double *out_val) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nw) {
        const int64_t o = rowptr[r];
        const int k = (int)(rowptr[r + 1] - o);
        if (k > kLongRow) continue;  // sort_long_rows_kernel
        for (int t = lane; t < k; t += 32) {
            const int32_t c = in_col[o + t];
            int rank = 0;
            for (int u = 0; u < k; ++u) rank += (in_col[o + u] < c);
            out_col[o + rank] = c;
            out_val[o + rank] = in_val[o + t];
        }
    }
}

// first index in the sorted run key[0, len) with key >= x
__device__ __forceinline__ int64_t lower_bound_i32(const int32_t *key, int64_t len, int32_t x) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One CTA per long row (> kLongRow entries).  Keys (source rows) are unique in a
// row, so the sorted order is unique.  Tiles of kSortTile keys are rank-sorted in
// shared memory into out_*, then runs are merged pairwise (each element's place
// = its index in its run + its rank in the partner run, a binary search), ping-
// ponging between out_* and in_* (in_* is scratch); the result ends in out_*.
constexpr int kSortTile = 1024;
__global__ void __launch_bounds__(256) sort_long_rows_kernel(int64_t n_rows, const int64_t *rowptr, int32_t *in_col,
                                                             double *in_val, int32_t *out_col, double *out_val) {
    __shared__ int32_t skey[kSortTile];
    __shared__ int64_t slist[256];
    __shared__ int nlist;
    for (int64_t r0 = (int64_t)blockIdx.x * 256; r0 < n_rows; r0 += (int64_t)gridDim.x * 256) {
        if (threadIdx.x == 0) nlist = 0;
        __syncthreads();
        const int64_t r = r0 + threadIdx.x;
        if (r < n_rows && rowptr[r + 1] - rowptr[r] > kLongRow) slist[atomicAdd(&nlist, 1)] = r;
        __syncthreads();
        const int nl = nlist;
        for (int li = 0; li < nl; ++li) {
            const int64_t row = slist[li];
            const int64_t o = rowptr[row], k = rowptr[row + 1] - o;
            // tiles: rank sort in shared memory, in_* -> out_*
            for (int64_t t0 = 0; t0 < k; t0 += kSortTile) {
                const int tl = (int)(k - t0 < kSortTile ? k - t0 : kSortTile);
                for (int t = threadIdx.x; t < tl; t += blockDim.x) skey[t] = in_col[o + t0 + t];
                __syncthreads();
                for (int t = threadIdx.x; t < tl; t += blockDim.x) {
                    const int32_t c = skey[t];
                    int rank = 0;
                    for (int u = 0; u < tl; ++u) rank += (skey[u] < c);
                    out_col[o + t0 + rank] = c;
                    out_val[o + t0 + rank] = in_val[o + t0 + t];
                }
                __syncthreads();
            }
            // merge passes
            int32_t *sc = out_col + o, *dc = in_col + o;
            double *sv = out_val + o, *dv = in_val + o;
            for (int64_t w = kSortTile; w < k; w *= 2) {
                for (int64_t p = threadIdx.x; p < k; p += blockDim.x) {
                    const int64_t s0 = (p / (2 * w)) * (2 * w);
                    const int64_t aend = s0 + w < k ? s0 + w : k, bend = s0 + 2 * w < k ? s0 + 2 * w : k;
                    const int32_t x = sc[p];
                    int64_t pos;
                    if (p < aend) pos = (p - s0) + lower_bound_i32(sc + aend, bend - aend, x);
                    else pos = (p - aend) + lower_bound_i32(sc + s0, aend - s0, x);
                    dc[s0 + pos] = x;
                    dv[s0 + pos] = sv[p];
                }
                __syncthreads();
                int32_t *tc = sc; sc = dc; dc = tc;
                double *tv = sv; sv = dv; dv = tv;
            }
            if (sc != out_col + o) {
                for (int64_t p = threadIdx.x; p < k; p += blockDim.x) {
                    out_col[o + p] = sc[p];
                    out_val[o + p] = sv[p];
                }
            }
            __syncthreads();
        }
    }
}

void sort_gt_rows(int64_t n_rows, const int64_t *rowptr, int32_t *in_col, double *in_val, int32_t *out_col,
                  double *out_val, int grid, cudaStream_t st, int64_t *launches) {
    sort_rows_kernel<<<grid, 256, 0, st>>>(n_rows, rowptr, in_col, in_val, out_col, out_val);
    const int64_t g2 = (n_rows + 255) / 256;
    sort_long_rows_kernel<<<(unsigned)(g2 < grid ? (g2 > 0 ? g2 : 1) : grid), 256, 0, st>>>(n_rows, rowptr, in_col,
                                                                                              in_val, out_col, out_val);
    *launches += 2;
}

// ---------------------------------------------------------------- transpose by stable radix sort
// G^T as a stable LSD radix sort of G's entries by column (8-bit digits): the input
// is G in row-major order, so every column's entries come out in ascending row --
// the deterministic order C10 asks for, with no atomics and no per-row sort.
// A pass = per-tile digit histograms, one exclusive scan (digit-major), a stable
// scatter (ranks inside a tile from warp match masks and per-warp digit counts).
constexpr int kRxThreads = 256, kRxItems = 16, kRxTile = kRxThreads * kRxItems;

// keys (column - col_lo) and row ids of G's entries, in storage order
__global__ void rx_init_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, int64_t col_lo,
                               int64_t row_begin, int32_t *key, int32_t *row) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nw)
        for (int64_t e = rowptr[r] + lane; e < rowptr[r + 1]; e += 32) {
            key[e] = (int32_t)(col[e] - col_lo);
            row[e] = (int32_t)(r + row_begin);
        }
}

__global__ void __launch_bounds__(kRxThreads) rx_hist_kernel(int64_t nnz, const int32_t *key, int shift,
                                                             int64_t ntiles, int32_t *hist) {
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * kRxTile;
#pragma unroll 4
    for (int k = 0; k < kRxItems; ++k) {
        const int64_t e = t0 + k * kRxThreads + threadIdx.x;
        if (e < nnz) atomicAdd(&h[(key[e] >> shift) & 255], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter of one digit pass.  Items of a tile are taken in storage order
// (iteration k: items t0 + 256 k + thread); an item's place in its digit bucket =
// the bucket's start for this tile (scanned histogram) + items of the digit in
// earlier iterations + in earlier warps of this iteration + earlier lanes of its warp.
__global__ void __launch_bounds__(kRxThreads) rx_scatter_kernel(int64_t nnz, const int32_t *key,
                                                                const int32_t *row, const double *val, int shift,
                                                                int64_t ntiles, const int64_t *off, int32_t *okey,
                                                                int32_t *orow, double *oval) {
    constexpr int NW = kRxThreads / 32;
    __shared__ int64_t base[256];
    __shared__ int run[256];
    __shared__ int wcnt[NW][256];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    base[tid] = off[(int64_t)tid * ntiles + blockIdx.x];
    run[tid] = 0;
    const int64_t t0 = (int64_t)blockIdx.x * kRxTile;
    for (int k = 0; k < kRxItems; ++k) {
#pragma unroll
        for (int x = 0; x < NW; ++x) wcnt[x][tid] = 0;
        __syncthreads();
        const int64_t e = t0 + k * kRxThreads + tid;
        const bool valid = e < nnz;
        const int32_t kk = valid ? key[e] : 0;
        const int d = valid ? (kk >> shift) & 255 : 256;  // 256: no digit
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (valid && rank == 0) wcnt[w][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int pre = 0;
            for (int x = 0; x < w; ++x) pre += wcnt[x][d];
            const int64_t pos = base[d] + run[d] + pre + rank;
            if (okey) okey[pos] = kk;
            orow[pos] = row[e];
            oval[pos] = val[e];
        }
        __syncthreads();
        int add = 0;
#pragma unroll
        for (int x = 0; x < NW; ++x) add += wcnt[x][tid];
        run[tid] += add;
    }
}

int64_t radix_tmp_bytes(int64_t nnz, int64_t n_out) {
    const int64_t ntiles = (nnz + kRxTile - 1) / kRxTile;
    const int64_t nh = 256 * (ntiles > 0 ? ntiles : 1);
    return nnz * (4 + 4 + 4 + 4 + 8 + 8) + nh * 4 + (nh + 1) * 8 + scan_tmp_elems(nh) * 8 + 64 * 6;
}

cudaError_t transpose_radix(int64_t n_rows, const int64_t *rowptr, const int32_t *col, const double *val,
                            int64_t nnz, int64_t col_lo, int64_t n_out, int64_t row_begin, char *tmp,
                            int32_t *t_col, double *t_val, int grid, cudaStream_t st, int64_t *launches) {
    if (nnz == 0) return cudaSuccess;
    const int64_t ntiles = (nnz + kRxTile - 1) / kRxTile;
    const int64_t nh = 256 * ntiles;
    auto carve = [&](size_t bytes) {
        char *p = tmp;
        tmp += (bytes + 63) & ~(size_t)63;
        return p;
    };
    int32_t *key0 = (int32_t *)carve(nnz * 4), *row0 = (int32_t *)carve(nnz * 4);
    int32_t *key1 = (int32_t *)carve(nnz * 4), *row1 = (int32_t *)carve(nnz * 4);
    double *val0 = (double *)carve(nnz * 8), *val1 = (double *)carve(nnz * 8);
    int32_t *hist = (int32_t *)carve(nh * 4);
    int64_t *off = (int64_t *)carve((nh + 1) * 8);
    int64_t *stiles = (int64_t *)carve(scan_tmp_elems(nh) * 8);
    int bits = 1;
    while (bits < 31 && (int64_t(1) << bits) < n_out) ++bits;
    const int passes = (bits + 7) / 8;
    rx_init_kernel<<<grid, 256, 0, st>>>(n_rows, rowptr, col, col_lo, row_begin, key0, row0);
    *launches += 1;
    const int32_t *ik = key0, *ir = row0;
    const double *iv = val;
    for (int ps = 0; ps < passes; ++ps) {
        const bool last = ps == passes - 1;
        int32_t *ok = last ? nullptr : (ps & 1 ? key0 : key1);
        int32_t *orr = last ? t_col : (ps & 1 ? row0 : row1);
        double *ov = last ? t_val : (ps & 1 ? val0 : val1);
        rx_hist_kernel<<<(unsigned)ntiles, kRxThreads, 0, st>>>(nnz, ik, 8 * ps, ntiles, hist);
        cudaError_t e = exclusive_scan(hist, nh, off, stiles, st, launches);
        if (e != cudaSuccess) return e;
        rx_scatter_kernel<<<(unsigned)ntiles, kRxThreads, 0, st>>>(nnz, ik, ir, iv, 8 * ps, ntiles, off, ok, orr, ov);
        *launches += 2;
        ik = ok;
        ir = orr;
        iv = ov;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- multi-GPU helpers
// lengths of local rows (int32) from a row pointer
__global__ void row_lengths_kernel(const int64_t *rowptr, int64_t n_rows, int32_t *len) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x)
        len[r] = (int32_t)(rowptr[r + 1] - rowptr[r]);
}

// G entries -> (col, row, val) triples, row = global row of the entry
__global__ void g_triples_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, const double *val,
                                 int64_t row_begin, int32_t *tc, int32_t *tr, double *tv) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nw)
        for (int64_t e = rowptr[r] + lane; e < rowptr[r + 1]; e += 32) {
            tc[e] = col[e];
            tr[e] = (int32_t)(r + row_begin);
            tv[e] = val[e];
        }
}

// triples with col in [lo, hi) (one destination rank), compacted in input order
// into out arrays at per-destination cursor; counts in cnt[dest]
__global__ void count_dest_kernel(int64_t nnz, const int32_t *tc, const int64_t *bounds, int nranks,
                                  unsigned long long *cnt) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = tc[e];
        int q = 0;
        while (q + 1 < nranks && c >= bounds[q + 1]) ++q;
        atomicAdd(&cnt[q], 1ull);
    }
}

__global__ void scatter_dest_kernel(int64_t nnz, const int32_t *tc, const int32_t *tr, const double *tv,
                                    const int64_t *bounds, int nranks, const unsigned long long *off,
                                    unsigned long long *cur, int32_t *oc, int32_t *orow, double *ov) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = tc[e];
        int q = 0;
        while (q + 1 < nranks && c >= bounds[q + 1]) ++q;
        const unsigned long long p = off[q] + atomicAdd(&cur[q], 1ull);
        oc[p] = tc[e];
        orow[p] = tr[e];
        ov[p] = tv[e];
    }
}

// entries of the local G with column in [lo, hi): per-row counts, then (after a
// scan of the counts) the (col, row, val) triples in row-major order
__global__ void band_count_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, int64_t lo, int64_t hi,
                                  int32_t *cnt) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        int c = 0;
        for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
            const int64_t j = col[e];
            c += (j >= lo && j < hi);
        }
        cnt[r] = c;
    }
}

__global__ void band_fill_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, const double *val,
                                 int64_t row_begin, int64_t lo, int64_t hi, const int64_t *off, int32_t *tc,
                                 int32_t *tr, double *tv) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = off[r];
        for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
            const int64_t j = col[e];
            if (j >= lo && j < hi) {
                tc[p] = (int32_t)j;
                tr[p] = (int32_t)(r + row_begin);
                tv[p] = val[e];
                ++p;
            }
        }
    }
}

// G^T of a set of triples whose columns lie in [col_lo, col_lo + n_out):
// count, (scan on host side), scatter, sort each row by source row (C10)
__global__ void count_triples_kernel(int64_t nnz, const int32_t *tc, int64_t col_lo, int64_t n_out, int32_t *cnt) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = (int64_t)tc[e] - col_lo;
        if (c >= 0 && c < n_out) atomicAdd(&cnt[c], 1);
    }
}

__global__ void scatter_triples_kernel(int64_t nnz, const int32_t *tc, const int32_t *tr, const double *tv,
                                       int64_t col_lo, int64_t n_out, const int64_t *t_rowptr, int32_t *cursor,
                                       int32_t *t_col, double *t_val) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = (int64_t)tc[e] - col_lo;
        if (c < 0 || c >= n_out) continue;
        const int p = atomicAdd(&cursor[c], 1);
        t_col[t_rowptr[c] + p] = tr[e];
        t_val[t_rowptr[c] + p] = tv[e];
    }
}

}  // namespace afsai
