// setup_kernel.cu -- the per-row adaptive FSAI set-up on sm_100a.
//
// One warp owns one row i of G at a time (persistent grid, atomic row queue).
// For that row it runs the whole k_max loop of PAPER.md P:383-396 with all
// state on chip (shared memory + registers):
//   phase G  Kaporin gradient (Eq. 15): for every candidate j,
//            acc_j = sum_{r in P U {i}} a_jr g~_r read from row j of A in storage
//            order (C3), one lane per candidate;
//   phase S  top-s selection with the (|acc| desc, j asc) total order (P:383-387,
//            DESIGN.md R5) by warp-shuffle argmax;
//   phase A  gather of the new rows of A[P,P] and A[P,i] (Eq. 7),
//            which also extends the candidate universe (R7);
//   phase B  bordered (incremental) Cholesky + forward solve + psi (Eq. 9
//            denominator) for the new rows only, as a right-looking column sweep
//            in which every lane folds its own entries in ascending k
//            (C5-C6);
//   phase U  back-substitution g~ = L^-T y as a descending column sweep (C7);
//   exit     Eq. 16 (C8); output scaled by psi^-1/2 (Eqs. 8-9, C9).
// The candidate/pattern set of a row lives in a per-warp open-addressing hash
// table in shared memory.  Compiled with -fmad=false: the only fused
// multiply-adds are the explicit fma() of the contract.
#include <cuda_runtime.h>

#include <cstdint>

#include "afsai_internal.h"
#include "setup_kernel.h"

namespace afsai {

constexpr unsigned kFull = 0xffffffffu;
constexpr int32_t kEmpty = -1;
constexpr int32_t kCand = -2;
constexpr int32_t kSel = -3;

__device__ __forceinline__ uint32_t hslot(int32_t key, int log2H) {
    return ((uint32_t)key * 2654435761u) >> (32 - log2H);
}

__device__ __forceinline__ int hfind(const int32_t *hkey, int H, int log2H, int32_t key) {
    uint32_t msk = (uint32_t)H - 1u, sl = hslot(key, log2H);
    for (int pr = 0; pr < H; ++pr) {
        int32_t k = hkey[sl];
        if (k == key) return (int)sl;
        if (k == kEmpty) return -1;
        sl = (sl + 1u) & msk;
    }
    return -1;
}

// insert-if-absent; returns slot (or -1 if the table is full); *ins = newly inserted
__device__ __forceinline__ int hinsert(int32_t *hkey, int H, int log2H, int32_t key, bool *ins) {
    uint32_t msk = (uint32_t)H - 1u, sl = hslot(key, log2H);
    for (int pr = 0; pr < H; ++pr) {
        int32_t k = hkey[sl];
        if (k == key) { *ins = false; return (int)sl; }
        if (k == kEmpty) {
            int32_t old = atomicCAS(&hkey[sl], kEmpty, key);
            if (old == kEmpty) { *ins = true; return (int)sl; }
            if (old == key) { *ins = false; return (int)sl; }
        }
        sl = (sl + 1u) & msk;
    }
    *ins = false;
    return -1;
}

// strictly-lower packed row-major L: L[q][c], c < q, at q(q-1)/2 + c
__device__ __forceinline__ int tri(int q) { return (q * (q - 1)) >> 1; }

struct WarpState {
    int32_t *hkey, *hval, *P, *sel, *selslot, *misc, *glen;
    int64_t *gstart;
    int16_t *clist;  // compact list of candidate slots
    double *hacc, *inv, *y, *g, *L, *arow, *brow, *dscr, *zero;
    int M;  // mmax: arow row stride
};

__device__ __forceinline__ WarpState carve(char *base, const SetupKArgs &a) {
    WarpState w;
    const int H = a.H, M = a.mmax, S = a.s;
    w.M = M;
    double *d = reinterpret_cast<double *>(base);
    w.hacc = d; d += H;
    w.inv = d; d += M;
    w.y = d; d += M;
    w.g = d; d += M;
    w.L = d; d += (M * (M - 1)) / 2 + 1;
    w.arow = d; d += S * M;
    w.brow = d; d += S;
    w.dscr = d; d += 2;
    w.zero = d; d += M + 1;
    w.gstart = reinterpret_cast<int64_t *>(d); d += S;
    int32_t *ip = reinterpret_cast<int32_t *>(d);
    w.hkey = ip; ip += H;
    w.hval = ip; ip += H;
    w.P = ip; ip += M;
    w.sel = ip; ip += S;
    w.selslot = ip; ip += S;
    w.glen = ip; ip += S;
    w.misc = ip; ip += 4;
    w.clist = reinterpret_cast<int16_t *>(ip);
    return w;
}

// bytes of one warp's state (must match carve)
__host__ __device__ inline int64_t warp_state_bytes(int H, int M, int S) {
    int64_t dbl = (int64_t)H + 3 * M + (M * (M - 1)) / 2 + 1 + (int64_t)S * M + S + 2 + S + M + 1;
    int64_t i32 = 2 * (int64_t)H + M + 3 * S + 4;
    int64_t b = dbl * 8 + i32 * 4 + 2 * (int64_t)H;
    return (b + 15) & ~int64_t(15);
}

// (|a|, ja) better than (|b|, jb)?  |acc| descending, then column ascending.
__device__ __forceinline__ bool better(double aa, int32_t ja, double ab, int32_t jb) {
    return (aa > ab) || (aa == ab && ja < jb);
}

__device__ __forceinline__ int64_t rp_of(const SetupKArgs &a, int64_t r) { return a.rowptr[r - a.a_lo] - a.base; }

template <int GS>
__device__ __forceinline__ double pick(const double (&v)[GS], int u) {
    double r = v[0];
#pragma unroll
    for (int k = 1; k < GS; ++k)
        if (u == k) r = v[k];
    return r;
}

// Bordered Cholesky of the group of new rows q = qf .. qf+gs-1 (gathered rows in
// arow/brow slots ug .. ug+gs-1), forward solve and psi update.  Right-looking
// column sweep: at stage k the owner lane of column k turns its accumulator into
// L[q][k] = t * inv[k] and broadcasts it; every lane then folds
// fma(-L[q][k], L[c][k], t_c) into its own columns.  Per accumulator the fold
// order is k ascending -- DESIGN.md C5.  Accumulators of columns c <= k (already
// finalized) or c > q_u (not part of row u) are dead, so the fold runs without
// per-lane predicates; their loads read a zero row (w.zero) to stay in bounds.
// Returns false on a pivot !(> 1e-30).
template <int NT, int GS>
__device__ bool border_group(const WarpState &w, int lane, int qf, int gs, int ug, double &psi) {
    const int ql = qf + gs - 1;
    const int M = w.M;
    double t[GS][NT];
    double ty[GS];
    double *Lnew[GS];
    const double *Lr[NT];
    int unew[NT];
    bool isold[NT];
#pragma unroll
    for (int u = 0; u < GS; ++u) {
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) {
            const int c = lane + 32 * tt;
            t[u][tt] = (u < gs && c <= qf + u) ? w.arow[(ug + u) * M + c] : 0.0;
        }
        ty[u] = (u < gs) ? -w.brow[ug + u] : 0.0;
        Lnew[u] = w.L + tri(qf + u);
    }
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        const int c = lane + 32 * tt;
        isold[tt] = c < qf;
        Lr[tt] = isold[tt] ? w.L + tri(c) : w.zero;
        unew[tt] = (c >= qf && c <= ql) ? c - qf : 0;
    }
    // ---- stages over the old columns k < qf: every group row is active
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        int lnend = qf - 32 * tt;
        if (lnend > 32) lnend = 32;
        for (int ln = 0; ln < lnend; ++ln) {
            const int k = 32 * tt + ln;
            const double inv_k = w.inv[k];
            const double y_k = w.y[k];
            double lsm[NT];
#pragma unroll
            for (int t2 = 0; t2 < NT; ++t2) lsm[t2] = Lr[t2][k];
            double l[GS];
#pragma unroll
            for (int u = 0; u < GS; ++u) l[u] = __shfl_sync(kFull, t[u][tt] * inv_k, ln);
            if (lane == ln) {
#pragma unroll
                for (int u = 0; u < GS; ++u)
                    if (u < gs) Lnew[u][k] = l[u];
            }
#pragma unroll
            for (int t2 = 0; t2 < NT; ++t2) {
                const double lc = isold[t2] ? lsm[t2] : pick<GS>(l, unew[t2]);
#pragma unroll
                for (int u = 0; u < GS; ++u) t[u][t2] = fma(-l[u], lc, t[u][t2]);
            }
#pragma unroll
            for (int u = 0; u < GS; ++u) ty[u] = fma(-l[u], y_k, ty[u]);
        }
    }
    // ---- stages over the group's own columns k = qf .. ql: finalize row k - qf,
    //      then fold it into the later group rows
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        int lnbeg = qf - 32 * tt, lnend = ql + 1 - 32 * tt;
        if (lnbeg < 0) lnbeg = 0;
        if (lnend > 32) lnend = 32;
        for (int ln = lnbeg; ln < lnend; ++ln) {
            const int k = 32 * tt + ln;
            const int uf = k - qf;
            double tv[GS];
#pragma unroll
            for (int u = 0; u < GS; ++u) tv[u] = t[u][tt];
            const double piv = __shfl_sync(kFull, pick<GS>(tv, uf), ln);
            if (!(piv > 1e-30)) return false;
            const double dq = sqrt(piv);          // C5.2: two correctly rounded operations
            const double inv_k = 1.0 / dq;
            const double y_k = pick<GS>(ty, uf) * inv_k;
            psi = fma(-y_k, y_k, psi);             // C6
            if (lane == 0) {
                w.inv[k] = inv_k;
                w.y[k] = y_k;
            }
            if (k == ql) break;
            double l[GS];
#pragma unroll
            for (int u = 0; u < GS; ++u) {
                l[u] = 0.0;
                if (u < gs && u > uf) {
                    l[u] = __shfl_sync(kFull, t[u][tt] * inv_k, ln);
                    if (lane == ln) Lnew[u][k] = l[u];
                }
            }
#pragma unroll
            for (int t2 = 0; t2 < NT; ++t2) {
                const int c = lane + 32 * t2;
                if (c > k && c <= ql) {
                    const double lnw = pick<GS>(l, unew[t2]);
#pragma unroll
                    for (int u = 0; u < GS; ++u) {
                        if (u < gs && u > uf && c <= qf + u) t[u][t2] = fma(-l[u], lnw, t[u][t2]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < GS; ++u)
                if (u < gs && u > uf) ty[u] = fma(-l[u], y_k, ty[u]);
        }
    }
    __syncwarp();
    return true;
}

// Back-substitution g~ = L^-T y (C7): descending column sweep; lane c
// folds fma(-L[k][c], g[k], t_c) for k = m-1 down to c+1.  Accumulators with
// c >= k are already final (dead), so the fold is unpredicated; column indices
// past the row are clamped to stay inside L.
template <int NT>
__device__ void back_substitute(const WarpState &w, int lane, int m) {
    double tb[NT];
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        const int c = lane + 32 * tt;
        tb[tt] = (c < m) ? w.y[c] : 0.0;
    }
#pragma unroll
    for (int tt = NT - 1; tt >= 0; --tt) {
        int ln0 = m - 1 - 32 * tt;
        if (ln0 > 31) ln0 = 31;
        for (int ln = ln0; ln >= 0; --ln) {
            const int k = 32 * tt + ln;
            const double iv = w.inv[k];
            const double *Lk = w.L + tri(k);
            double lk[NT];
#pragma unroll
            for (int t2 = 0; t2 <= tt; ++t2) {
                const int c = lane + 32 * t2;
                lk[t2] = Lk[c < k ? c : 0];
            }
            const double gk = __shfl_sync(kFull, tb[tt] * iv, ln);
            if (lane == ln) w.g[k] = gk;
#pragma unroll
            for (int t2 = 0; t2 <= tt; ++t2) tb[t2] = fma(-lk[t2], gk, tb[t2]);
        }
    }
    __syncwarp();
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// insert column c (< i) into the universe; appends new slots to the candidate list
__device__ __forceinline__ int universe_insert(const WarpState &w, int H, int log2H, int32_t c) {
    bool ins;
    const int sl = hinsert(w.hkey, H, log2H, c, &ins);
    if (sl < 0) {
        w.misc[1] = 1;
    } else if (ins) {
        const int p = atomicAdd(&w.misc[2], 1);
        w.clist[p] = (int16_t)sl;
        atomicAdd(&w.misc[0], 1);
    }
    return ins ? -1 : sl;  // slot of an already present key, else -1
}

constexpr int kGradChunk = 8;  // row entries loaded per batch in the gradient

template <int NT, int GS>
__global__ void __launch_bounds__(256) afsai_setup_rows_kernel(SetupKArgs a) {
    extern __shared__ __align__(16) char smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    WarpState w = carve(smem + (size_t)wid * a.warp_smem, a);
    const int H = a.H, log2H = a.log2H;
    unsigned long long c_steps = 0, c_border = 0, c_back = 0, c_gfma = 0, c_gent = 0;
    unsigned long long c_r0 = 0, c_r1 = 0, c_r2 = 0, c_r3 = 0, c_univ = 0;
    // per-phase SM cycles (lane 0): prologue, gradient, select, gather, border, backsub, output
    long long ph[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int x = lane; x <= a.mmax; x += 32) w.zero[x] = 0.0;
    __syncwarp();
    long long tph = clock64();
#define PHASE(idx)                      \
    {                                   \
        const long long t1_ = clock64(); \
        ph[idx] += t1_ - tph;           \
        tph = t1_;                      \
    }

    for (;;) {
        unsigned long long t_idx = 0;
        if (lane == 0) t_idx = atomicAdd(a.work, 1ull);
        t_idx = __shfl_sync(kFull, t_idx, 0);
        if ((int64_t)t_idx >= a.nrows) break;
        const int64_t i64 = a.rows ? a.rows[t_idx] : a.row_lo + (int64_t)t_idx;
        const int32_t i = (int32_t)i64;
        const int64_t orow = i64 - a.out_base;

        tph = clock64();
        // ---- prologue: empty table, universe = columns j < i of row i, a_ii
        for (int sl = lane; sl < H; sl += 32) {
            w.hkey[sl] = kEmpty;
            w.hval[sl] = kCand;  // every key starts as a candidate
        }
        if (lane == 0) {
            w.misc[0] = 0;  // keys inserted
            w.misc[1] = 0;  // overflow
            w.misc[2] = 0;  // candidate list length
            w.dscr[0] = 0.0;
        }
        __syncwarp();
        {
            const int64_t e0 = rp_of(a, i64), e1 = rp_of(a, i64 + 1);
            for (int64_t e = e0 + lane; e < e1; e += 32) {
                const int32_t c = a.col[e];
                if (c == i) w.dscr[0] = a.val[e];
                else if (c < i) universe_insert(w, H, log2H, c);
            }
        }
        __syncwarp();
        const double a_ii = w.dscr[0];
        const double psi0 = a_ii;
        double psi = psi0;
        int m = 0, steps = 0, reason = AFSAI_STOP_KMAX;
        bool fail = false, overflow = (w.misc[1] != 0);
        int fail_code = 0, fail_step = 0;
        PHASE(0)

        for (int k = 1; k <= a.nsteps && !overflow; ++k) {
            int room = a.s;
            if (a.cap - 1 - m < room) room = a.cap - 1 - m;
            if (room <= 0) { reason = AFSAI_STOP_CAP; break; }

            // ---- phase G: gradient (C3), one lane per candidate; each candidate row
            //      j is read in batches of kGradChunk independent loads, folded in
            //      storage (ascending r) order
            const int ncl = w.misc[2];
            int nc = 0;
            for (int base = 0; base < ncl; base += 32) {
                const int t = base + lane;
                if (t < ncl) {
                    const int sl = w.clist[t];
                    const int32_t j = w.hkey[sl];
                    double acc = 0.0;
                    const int64_t e0 = rp_of(a, j), e1 = rp_of(a, (int64_t)j + 1);
                    for (int64_t eb = e0; eb < e1; eb += kGradChunk) {
                        int32_t cc[kGradChunk];
                        double vv[kGradChunk];
#pragma unroll
                        for (int u = 0; u < kGradChunk; ++u) {
                            const bool in = eb + u < e1;
                            cc[u] = in ? __ldg(a.col + eb + u) : 0x7fffffff;
                            vv[u] = in ? __ldg(a.val + eb + u) : 0.0;
                        }
                        double gv[kGradChunk];
                        bool hit[kGradChunk];
#pragma unroll
                        for (int u = 0; u < kGradChunk; ++u) {
                            const int32_t r = cc[u];
                            hit[u] = false;
                            gv[u] = 1.0;
                            if (r == i) hit[u] = true;
                            else if (r < i) {
                                const int s2 = hfind(w.hkey, H, log2H, r);
                                if (s2 >= 0) {
                                    const int st = w.hval[s2];
                                    if (st >= 0) {
                                        hit[u] = true;
                                        gv[u] = w.g[st];
                                    }
                                }
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kGradChunk; ++u) {
                            if (hit[u]) {
                                acc = fma(vv[u], gv[u], acc);
                                ++c_gfma;
                            }
                            c_gent += (cc[u] <= i);
                        }
                        if (cc[kGradChunk - 1] >= i) break;  // sorted: nothing of P U {i} beyond
                    }
                    w.hacc[sl] = acc;
                    if (acc != 0.0) ++nc;
                }
            }
            nc = warp_sum_i(nc);
            __syncwarp();
            PHASE(1)
            if (nc == 0) { reason = AFSAI_STOP_NOCAND; break; }
            const int nsel = nc < room ? nc : room;

            // ---- phase S: top-nsel under the total order (|acc| desc, j asc)
            if (a.s <= GS) {
                // one pass: every lane keeps its best GS candidates (sorted, in
                // registers), then nsel rounds of warp argmax over the list heads
                double ba[GS];
                int32_t bj[GS], bs[GS];
#pragma unroll
                for (int q = 0; q < GS; ++q) { ba[q] = -1.0; bj[q] = 0x7fffffff; bs[q] = -1; }
                for (int t = lane; t < ncl; t += 32) {
                    const int sl = w.clist[t];
                    double ca = fabs(w.hacc[sl]);
                    if (ca == 0.0) continue;
                    int32_t cj = w.hkey[sl];
                    int32_t cs = sl;
#pragma unroll
                    for (int q = 0; q < GS; ++q) {
                        if (better(ca, cj, ba[q], bj[q])) {
                            const double ta = ba[q]; const int32_t tj = bj[q], ts = bs[q];
                            ba[q] = ca; bj[q] = cj; bs[q] = cs;
                            ca = ta; cj = tj; cs = ts;
                        }
                    }
                }
                for (int u = 0; u < nsel; ++u) {
                    double wa = ba[0];
                    int32_t wj = bj[0];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double oa = __shfl_xor_sync(kFull, wa, o);
                        const int32_t oj = __shfl_xor_sync(kFull, wj, o);
                        if (better(oa, oj, wa, wj)) { wa = oa; wj = oj; }
                    }
                    if (bj[0] == wj) {  // column indices are unique: exactly one lane
                        w.sel[u] = wj;
                        w.selslot[u] = bs[0];
#pragma unroll
                        for (int q = 0; q + 1 < GS; ++q) { ba[q] = ba[q + 1]; bj[q] = bj[q + 1]; bs[q] = bs[q + 1]; }
                        ba[GS - 1] = -1.0; bj[GS - 1] = 0x7fffffff; bs[GS - 1] = -1;
                    }
                }
                __syncwarp();
            } else {
                // s > 4: nsel rounds of warp argmax over the candidate list
                for (int u = 0; u < nsel; ++u) {
                    double ba = -1.0;
                    int32_t bj = 0x7fffffff;
                    int bs = -1;
                    for (int t = lane; t < ncl; t += 32) {
                        const int sl = w.clist[t];
                        if (w.hval[sl] != kCand) continue;
                        const double aa = fabs(w.hacc[sl]);
                        if (aa == 0.0) continue;
                        const int32_t j = w.hkey[sl];
                        if (better(aa, j, ba, bj)) { ba = aa; bj = j; bs = sl; }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double oa = __shfl_xor_sync(kFull, ba, o);
                        const int32_t oj = __shfl_xor_sync(kFull, bj, o);
                        const int os = __shfl_xor_sync(kFull, bs, o);
                        if (better(oa, oj, ba, bj)) { ba = oa; bj = oj; bs = os; }
                    }
                    if (lane == 0) { w.sel[u] = bj; w.selslot[u] = bs; w.hval[bs] = kSel; }
                    __syncwarp();
                }
            }
            // append in ascending column order (R9); rows of A to gather
            if (lane < nsel) {
                const int32_t j = w.sel[lane];
                int rank = 0;
                for (int u = 0; u < nsel; ++u) rank += (w.sel[u] < j);
                w.P[m + rank] = j;
                w.hval[w.selslot[lane]] = m + rank;
                const int64_t g0 = rp_of(a, j), g1 = rp_of(a, (int64_t)j + 1);
                w.gstart[rank] = g0;
                w.glen[rank] = (int32_t)(g1 - g0);
            }
            __syncwarp();
            // drop the selected slots from the candidate list (stable in-warp compaction)
            {
                int wr = 0;
                for (int base = 0; base < ncl; base += 32) {
                    const int t = base + lane;
                    const int sl = t < ncl ? w.clist[t] : 0;
                    const bool keep = t < ncl && w.hval[sl] == kCand;
                    const unsigned bal = __ballot_sync(kFull, keep);
                    __syncwarp();
                    if (keep) w.clist[wr + __popc(bal & ((1u << lane) - 1u))] = (int16_t)sl;
                    wr += __popc(bal);
                    __syncwarp();
                }
                if (lane == 0) w.misc[2] = wr;
            }
            // zero the gathered rows
            for (int x = lane; x < nsel * w.M; x += 32) w.arow[x] = 0.0;
            if (lane < nsel) w.brow[lane] = 0.0;
            __syncwarp();
            PHASE(2)

            // ---- phase A: gather rows P_q (q = m..m+nsel-1) of A, all rows at once;
            //      extend the universe with their columns (R7)
            {
                int total = 0;
                for (int u = 0; u < nsel; ++u) total += w.glen[u];
                for (int t = lane; t < total; t += 32) {
                    int u = 0, off = t;
                    while (off >= w.glen[u]) { off -= w.glen[u]; ++u; }
                    const int64_t e = w.gstart[u] + off;
                    const int32_t c = __ldg(a.col + e);
                    if (c == i) w.brow[u] = __ldg(a.val + e);
                    else if (c < i) {
                        const int sl = universe_insert(w, H, log2H, c);
                        if (sl >= 0) {
                            const int st = w.hval[sl];
                            if (st >= 0 && st <= m + u) w.arow[u * w.M + st] = __ldg(a.val + e);
                        }
                    }
                }
            }
            __syncwarp();
            PHASE(3)
            if (w.misc[1] != 0 || w.misc[0] * 4 > H * 3) { overflow = true; break; }

            // ---- phase B: bordered Cholesky of the new rows, in lockstep groups of GS
            for (int ug = 0; ug < nsel && !fail; ug += GS) {
                const int gs = (nsel - ug) < GS ? (nsel - ug) : GS;
                if (!border_group<NT, GS>(w, lane, m + ug, gs, ug, psi)) {
                    fail = true; fail_code = AFSAI_ENOTSPD; fail_step = k;
                }
            }
            if (fail) break;
            for (int u = 0; u < nsel; ++u) {
                const long q = m + u;
                c_border += (unsigned long long)(q * (q - 1) / 2 + 2 * q + 1);
            }
            m += nsel;
            if (!(psi > 0.0)) { fail = true; fail_code = AFSAI_ENOTSPD; fail_step = k; break; }
            PHASE(4)

            // ---- phase U: back-substitution
            back_substitute<NT>(w, lane, m);
            c_back += (unsigned long long)(m * (m - 1) / 2);
            steps = k;
            PHASE(5)
            // ---- Eq. 16 exit test (C8)
            if (psi / psi0 <= a.eps) { reason = AFSAI_STOP_TOL; break; }
        }

        if (overflow) {
            if (lane == 0) {
                const int p = atomicAdd(a.retry_count, 1);
                a.retry_rows[p] = i64;
            }
            continue;
        }
        if (fail) {
            if (lane == 0) {
                const unsigned long long code = ((unsigned long long)i64 << 24) |
                                                ((unsigned long long)(fail_step & 0xfffff) << 4) |
                                                (unsigned long long)fail_code;
                atomicMin(a.err, code);
                a.nnz_row[orow] = 0;
            }
            continue;
        }
        // ---- output: d = psi^-1/2 (Eqs. 8-9), row sorted by column (C9)
        const double d = 1.0 / sqrt(psi);
        int32_t *oc = a.scol + orow * a.stride;
        double *ov = a.sval + orow * a.stride;
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) {
            const int q = lane + 32 * tt;
            if (q < m) {
                const int32_t pj = w.P[q];
                int rank = 0;
                for (int q2 = 0; q2 < m; ++q2) rank += (w.P[q2] < pj);
                oc[rank] = pj;
                ov[rank] = w.g[q] * d;
            }
        }
        if (lane == 0) {
            oc[m] = i;
            ov[m] = d;
            a.nnz_row[orow] = m + 1;
            a.steps[orow] = steps;
            a.reason[orow] = reason;
            c_steps += steps;
            c_r0 += (reason == 0);
            c_r1 += (reason == 1);
            c_r2 += (reason == 2);
            c_r3 += (reason == 3);
            c_univ = max(c_univ, (unsigned long long)w.misc[0]);
        }
        __syncwarp();
        PHASE(6)
    }
#undef PHASE
    // ---- statistics (one atomic per warp and counter)
    unsigned long long g1 = c_gfma, g2 = c_gent;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        g1 += __shfl_xor_sync(kFull, g1, o);
        g2 += __shfl_xor_sync(kFull, g2, o);
    }
    if (lane == 0) {
        atomicAdd(&a.counters[0], c_steps);
        atomicAdd(&a.counters[1], c_border);
        atomicAdd(&a.counters[2], c_back);
        atomicAdd(&a.counters[3], g1);
        atomicAdd(&a.counters[4], g2);
        atomicAdd(&a.counters[5], c_r0);
        atomicAdd(&a.counters[6], c_r1);
        atomicAdd(&a.counters[7], c_r2);
        atomicAdd(&a.counters[8], c_r3);
#pragma unroll
        for (int k = 0; k < 7; ++k) atomicAdd(&a.counters[9 + k], (unsigned long long)ph[k]);
        atomicMax(&a.counters[16], c_univ);
    }
}

// ---- host-side launcher: picks the template instance
template <int NT, int GS>
static cudaError_t launch_inst(const SetupKArgs &a, int grid, int block, size_t smem, cudaStream_t st) {
    auto kern = afsai_setup_rows_kernel<NT, GS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, block, smem, st>>>(a);
    return cudaGetLastError();
}

template <int NT>
static cudaError_t launch_nt(const SetupKArgs &a, int gs, int grid, int block, size_t smem, cudaStream_t st) {
    switch (gs) {
        case 1: return launch_inst<NT, 1>(a, grid, block, smem, st);
        case 2: return launch_inst<NT, 2>(a, grid, block, smem, st);
        case 3: return launch_inst<NT, 3>(a, grid, block, smem, st);
        default: return launch_inst<NT, 4>(a, grid, block, smem, st);
    }
}

int64_t setup_warp_bytes(int H, int mmax, int s) { return warp_state_bytes(H, mmax, s); }

cudaError_t launch_setup_rows(const SetupKArgs &a, int warps_per_cta, int grid, cudaStream_t st) {
    const int nt = (a.mmax + 31) / 32 < 1 ? 1 : (a.mmax + 31) / 32;
    const int gs = a.s < kMaxGroup ? a.s : kMaxGroup;
    const size_t smem = (size_t)a.warp_smem * warps_per_cta;
    const int block = 32 * warps_per_cta;
    switch (nt) {
        case 1: return launch_nt<1>(a, gs, grid, block, smem, st);
        case 2: return launch_nt<2>(a, gs, grid, block, smem, st);
        case 3: return launch_nt<3>(a, gs, grid, block, smem, st);
        default: return launch_nt<4>(a, gs, grid, block, smem, st);
    }
}

int setup_occupancy(int mmax, int s, int warps_per_cta, size_t smem) {
    const int nt = (mmax + 31) / 32 < 1 ? 1 : (mmax + 31) / 32;
    const int gs = s < kMaxGroup ? s : kMaxGroup;
    int blocks = 0;
    const void *f = nullptr;
#define AFSAI_F(NT_, GS_) if (nt == NT_ && gs == GS_) f = (const void *)afsai_setup_rows_kernel<NT_, GS_>;
    AFSAI_F(1, 1) AFSAI_F(1, 2) AFSAI_F(1, 3) AFSAI_F(1, 4)
    AFSAI_F(2, 1) AFSAI_F(2, 2) AFSAI_F(2, 3) AFSAI_F(2, 4)
    AFSAI_F(3, 1) AFSAI_F(3, 2) AFSAI_F(3, 3) AFSAI_F(3, 4)
    AFSAI_F(4, 1) AFSAI_F(4, 2) AFSAI_F(4, 3) AFSAI_F(4, 4)
#undef AFSAI_F
    if (!f) return 0;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, f, 32 * warps_per_cta, smem);
    return blocks;
}

}  // namespace afsai
