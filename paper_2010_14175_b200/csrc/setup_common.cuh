// setup_common.cuh -- device code shared by the two per-row set-up kernels
// (setup_scan.cu: general rows; setup_hits.cu: short rows with hit lists).
#pragma once
#ifndef AFSAI_FMAD_OFF
#error "set-up device code must be compiled with -fmad=false -DAFSAI_FMAD_OFF (arithmetic contract, DESIGN.md 3.1)"
#endif
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "afsai_internal.h"
#include "setup_kernel.h"

// Precision of the set-up arithmetic.  Every set-up translation unit is compiled
// twice (build.py): as afsai::dp (fp64, `real` = double; the default set-up) and,
// with -DAFSAI_SETUP_FP32, as afsai::sp (`real` = float: the single-precision
// set-up of PAPER.md §4.3, on A_s = single(A)).  The contract C1-C12
// is the same in both; the fp32 oracle (oracle/ built with -DOR_FP32) pins sp.
// Comparisons against the double constants 1e-30 and eps widen the float operand
// exactly (as the oracle does); the output scratch is fp64: G = double(G_s).
#ifdef AFSAI_SETUP_FP32
#define AFSAI_PNS sp
#else
#define AFSAI_PNS dp
#endif

namespace afsai {
namespace AFSAI_PNS {

#ifdef AFSAI_SETUP_FP32
typedef float real;
#else
typedef double real;
#endif

// A's values in the set-up's precision (A_s for the fp32 set-up)
__device__ __forceinline__ const real *aval(const SetupKArgs &a) {
#ifdef AFSAI_SETUP_FP32
    return a.val32;
#else
    return a.val;
#endif
}

// bytes of n values, padded so what follows stays 16-byte aligned
__host__ __device__ inline int64_t real_bytes(int64_t n) { return (n * (int64_t)sizeof(real) + 15) & ~int64_t(15); }

constexpr int32_t kEmpty = -1;
constexpr int8_t kCand = -2;
constexpr int kGradChunk = 8;  // row entries loaded per batch in the gradient

// lanes [base, base+LPR) of a warp working on one row
template <int LPR>
struct Group {
    int gl;         // lane within the group
    unsigned mask;  // the group's lanes
    __device__ explicit Group(int lane)
        : gl(lane & (LPR - 1)),
          mask(LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (lane & ~(LPR - 1)))) {}
    template <class T>
    __device__ __forceinline__ T bcast(T v, int src) const { return __shfl_sync(mask, v, src, LPR); }
    template <class T>
    __device__ __forceinline__ T xorv(T v, int o) const { return __shfl_xor_sync(mask, v, o, LPR); }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
    __device__ __forceinline__ int sum(int v) const {
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) v += xorv(v, o);
        return v;
    }
    __device__ __forceinline__ unsigned long long sum(unsigned long long v) const {
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) v += xorv(v, o);
        return v;
    }
};

__device__ __forceinline__ uint32_t hslot(int32_t key, int log2H) {
    return ((uint32_t)key * 2654435761u) >> (32 - log2H);
}

__device__ __forceinline__ int hfind(const int32_t *hkey, int H, int log2H, int32_t key) {
    uint32_t msk = (uint32_t)H - 1u, sl = hslot(key, log2H);
    for (int pr = 0; pr < H; ++pr) {
        const int32_t k = hkey[sl];
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
        const int32_t k = hkey[sl];
        if (k == key) { *ins = false; return (int)sl; }
        if (k == kEmpty) {
            const int32_t old = atomicCAS(&hkey[sl], kEmpty, key);
            if (old == kEmpty) { *ins = true; return (int)sl; }
            if (old == key) { *ins = false; return (int)sl; }
        }
        sl = (sl + 1u) & msk;
    }
    *ins = false;
    return -1;
}

// packed row-major L: L[q][c], c < q, at q(q+1)/2 + c (the diagonal slot is
// unused: with this offset any 16 consecutive rows start in distinct banks, so
// a column read by 16 lanes is conflict free; q(q-1)/2 collides rows 0 and 1)
__device__ __forceinline__ int tri(int q) { return (q * (q + 1)) >> 1; }

// (|a|, ja) better than (|b|, jb)?  |acc| descending, then column ascending.
// The magnitudes are |acc| >= 0 or the sentinel -1: for non-negative IEEE values
// the order of the bit patterns (as signed integers) is the numeric order, and the
// sentinel's sign bit makes it smaller than all of them, so the comparison runs on
// the integer pipe (same result as the floating-point compare).
__device__ __forceinline__ bool better(double aa, int32_t ja, double ab, int32_t jb) {
    const long long ia = __double_as_longlong(aa), ib = __double_as_longlong(ab);
    return (ia > ib) || (ia == ib && ja < jb);
}
__device__ __forceinline__ bool better(float aa, int32_t ja, float ab, int32_t jb) {
    const int ia = __float_as_int(aa), ib = __float_as_int(ab);
    return (ia > ib) || (ia == ib && ja < jb);
}

// Insert (ca, cj, ct) into the sorted top-GS list (ba, bj, bt) under better(),
// dropping the last entry.  All GS comparisons are against the list as it was
// (the list is sorted, so the outcomes are monotone in q) and the new list is
// selected from them: two dependent steps per candidate instead of a GS-long
// compare-and-swap chain, with the same result as the sequential insertion.
template <int GS>
__device__ __forceinline__ void topk_insert(real (&ba)[GS], int32_t (&bj)[GS], int32_t (&bt)[GS], real ca, int32_t cj,
                                            int32_t ct) {
    bool b[GS];
#pragma unroll
    for (int q = 0; q < GS; ++q) b[q] = better(ca, cj, ba[q], bj[q]);
#pragma unroll
    for (int q = GS - 1; q >= 1; --q) {
        ba[q] = b[q] ? (b[q - 1] ? ba[q - 1] : ca) : ba[q];
        bj[q] = b[q] ? (b[q - 1] ? bj[q - 1] : cj) : bj[q];
        bt[q] = b[q] ? (b[q - 1] ? bt[q - 1] : ct) : bt[q];
    }
    ba[0] = b[0] ? ca : ba[0];
    bj[0] = b[0] ? cj : bj[0];
    bt[0] = b[0] ? ct : bt[0];
}

__device__ __forceinline__ int64_t rp_of(const SetupKArgs &a, int64_t r) {
#ifdef AFSAI_BOUNDS_CHECK
    if (r < a.a_lo || r > a.a_hi) {
        printf("afsai bounds: row pointer of row %lld outside [%lld, %lld] (block %d thread %d)\n", (long long)r,
               (long long)a.a_lo, (long long)a.a_hi, (int)blockIdx.x, (int)threadIdx.x);
        return 0;  // report and continue (a trap can lose the printf buffer)
    }
    const int64_t v = a.rowptr[r - a.a_lo] - a.base;
    if (v < 0 || v > a.nnz) {
        printf("afsai bounds: row %lld starts at entry %lld outside [0, %lld]\n", (long long)r, (long long)v,
               (long long)a.nnz);
        return 0;
    }
    return v;
#else
    return a.rowptr[r - a.a_lo] - a.base;
#endif
}

// Bordered Cholesky of the group of new rows q = qf .. qf+gs-1 (gathered rows in
// arow/brow slots ug .. ug+gs-1), forward solve and psi update.
//  - old columns c < qf: right-looking column sweep.  At stage k the owner lane
//    of column k turns its accumulator into L[q][k] = t * inv[k] and broadcasts
//    it; every lane folds fma(-L[q][k], L[c][k], t_c) into its own columns.  The
//    owner multiplies by its column's inverse diagonal, held in a register, and
//    the stage's shared-memory operands are loaded first (they arrive during the
//    DMUL -> SHFL), so no software pipelining is needed.  Accumulators of
//    finalized columns are dead: folded unpredicated (loads of any in-bounds row).
//  - new columns (the diagonal of each new row and the couplings between new
//    rows) are few: every lane keeps them redundantly, no broadcast needed.
// One copy of the stage per column chunk, not unrolled (the set-up kernels are
// instruction-cache sensitive).  Every accumulator folds in k-ascending order,
// exactly DESIGN.md C5.  Returns false on a pivot !(> 1e-30).
//  kSmemBcast: the owner lane alone stores L[q][k] and every lane reads it back
//  (shared-memory broadcast) instead of the 64-bit shuffles.
template <int LPR, int NT, int GS, bool kSmemBcast = false, class State>
__device__ bool border_group(const State &w, const Group<LPR> &G, int qf, int gs, int ug, real &psi) {
    const int M = w.M, gl = G.gl;
    real t[GS][NT], dg[GS], ty[GS], cp[GS][GS], ivc[NT];
    real *Lnew[GS];
    const real *Lr[NT];
#pragma unroll
    for (int u = 0; u < GS; ++u) {
        const real *ar = w.arow + (ug + u) * M;
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) {
            const int c = gl + LPR * tt;
            t[u][tt] = (u < gs && c < qf) ? ar[c] : real(0);
        }
        dg[u] = (u < gs) ? ar[qf + u] : real(0);
#pragma unroll
        for (int v = 0; v < GS; ++v) cp[u][v] = (v < u && u < gs) ? ar[qf + v] : real(0);
        ty[u] = (u < gs) ? -w.brow[ug + u] : real(0);
        Lnew[u] = w.L + tri(qf + u < M ? qf + u : 0);
    }
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        const int c = gl + LPR * tt;
        Lr[tt] = (c < qf) ? w.L + tri(c) : w.L;  // dead columns: any in-bounds row
        ivc[tt] = (c < qf) ? w.inv[c] : real(0);
    }
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        int lnend = qf - LPR * tt;
        if (lnend > LPR) lnend = LPR;
#pragma unroll 1
        for (int ln = 0; ln < lnend; ++ln) {
            const int k = LPR * tt + ln;
            const real y_k = w.y[k];
            real lsm[NT];
#pragma unroll
            for (int t2 = tt; t2 < NT; ++t2) lsm[t2] = Lr[t2][k];
            real l[GS];
            if constexpr (kSmemBcast) {
#pragma unroll
                for (int u = 0; u < GS; ++u)
                    if (gl == ln && u < gs) Lnew[u][k] = t[u][tt] * ivc[tt];
                G.sync();
                // rows u >= gs read any in-bounds value into their dead state
#pragma unroll
                for (int u = 0; u < GS; ++u) l[u] = Lnew[u][k];
            } else {
#pragma unroll
                for (int u = 0; u < GS; ++u) l[u] = G.bcast(t[u][tt] * ivc[tt], ln);
                // broadcast values: every lane stores the same bits (no divergent
                // branch before the next stage's shuffles)
#pragma unroll
                for (int u = 0; u < GS; ++u)
                    if (u < gs) Lnew[u][k] = l[u];
            }
#pragma unroll
            for (int t2 = tt; t2 < NT; ++t2)
#pragma unroll
                for (int u = 0; u < GS; ++u) t[u][t2] = fma(-l[u], lsm[t2], t[u][t2]);
#pragma unroll
            for (int u = 0; u < GS; ++u) {
                dg[u] = fma(-l[u], l[u], dg[u]);
                ty[u] = fma(-l[u], y_k, ty[u]);
#pragma unroll
                for (int v = 0; v < GS; ++v)
                    if (v < u) cp[u][v] = fma(-l[u], l[v], cp[u][v]);
            }
        }
    }
    // ---- the group's own columns k = qf + uf: finalize row uf, fold it into the
    //      later group rows (all values redundant in every lane)
#pragma unroll
    for (int uf = 0; uf < GS; ++uf) {
        if (uf >= gs) break;
        const int k = qf + uf;
        const real piv = dg[uf];
        if (!(piv > 1e-30)) return false;
        const real dq = sqrt(piv);  // C5.2: two correctly rounded operations
        const real inv_k = real(1) / dq;
        const real y_k = ty[uf] * inv_k;
        psi = fma(-y_k, y_k, psi);     // C6
        w.inv[k] = inv_k;  // redundant values: every lane stores the same bits
        w.y[k] = y_k;
        real lu[GS];
#pragma unroll
        for (int u = 0; u < GS; ++u) {
            lu[u] = real(0);
            if (u > uf && u < gs) {
                lu[u] = cp[u][uf] * inv_k;
                Lnew[u][k] = lu[u];
            }
        }
#pragma unroll
        for (int u = 0; u < GS; ++u) {
            if (u > uf && u < gs) {
                dg[u] = fma(-lu[u], lu[u], dg[u]);
                ty[u] = fma(-lu[u], y_k, ty[u]);
#pragma unroll
                for (int v = 0; v < GS; ++v)
                    if (v > uf && v < u) cp[u][v] = fma(-lu[u], lu[v], cp[u][v]);
            }
        }
    }
    G.sync();
    return true;
}

// Back-substitution g~ = L^-T y (C7): descending column sweep; lane c
// folds fma(-L[k][c], g[k], t_c) for k = m-1 down to c+1.  Row k of L is read
// contiguously by the lanes through a running pointer (tri(k-1) = tri(k) - k);
// reads past the row's live columns stay inside the row's shared-memory region
// (every state layout puts arow and more after L) and feed dead accumulators
// (c >= k: final), so the fold is unpredicated.  The owner multiplies by its
// column's inverse diagonal, held in a register.
template <int LPR, int NT, bool kSmemBcast = false, class State>
__device__ void back_substitute(const State &w, const Group<LPR> &G, int m) {
    const int gl = G.gl;
    real tb[NT], ivc[NT];
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        const int c = gl + LPR * tt;
        tb[tt] = (c < m) ? w.y[c] : real(0);
        ivc[tt] = (c < m) ? w.inv[c] : real(0);
    }
    const real *pk = w.L + tri(m > 0 ? m - 1 : 0) + gl;
#pragma unroll
    for (int tt = NT - 1; tt >= 0; --tt) {
        int ln0 = m - 1 - LPR * tt;
        if (ln0 > LPR - 1) ln0 = LPR - 1;
#pragma unroll 1
        for (int ln = ln0; ln >= 0; --ln) {
            const int k = LPR * tt + ln;
            real lk[NT];
#pragma unroll
            for (int t2 = 0; t2 <= tt; ++t2) lk[t2] = pk[LPR * t2];
            pk -= k;
            real gk;
            if constexpr (kSmemBcast) {
                if (gl == ln) w.g[k] = tb[tt] * ivc[tt];  // owner stores, every lane reads
                G.sync();
                gk = w.g[k];
            } else {
                gk = G.bcast(tb[tt] * ivc[tt], ln);
                w.g[k] = gk;  // broadcast value, stored by every lane
            }
#pragma unroll
            for (int t2 = 0; t2 <= tt; ++t2) tb[t2] = fma(-lk[t2], gk, tb[t2]);
        }
    }
    G.sync();
}

}  // namespace AFSAI_PNS
}  // namespace afsai
