// setup_kernel.cu -- the per-row adaptive FSAI set-up on sm_100a.
//
// A GROUP of LPR lanes (8, 16 or 32) owns one row i of G at a time; a warp
// holds 32/LPR rows (persistent grid, atomic row queue).  For its row a group
// runs the whole k_max loop of PAPER.md P:383-396 with all state on chip:
//   phase G  Kaporin gradient (Eq. 15): for every candidate j,
//            acc_j = sum_{r in P U {i}} a_jr g~_r read from row j of A in storage
//            order (C3); one lane per candidate, the next candidate's
//            row prefetched while the current one is folded;
//   phase S  top-s selection with the (|acc| desc, j asc) total order (P:383-387,
//            DESIGN.md R5): per-lane register top-s lists merged by shuffles;
//   phase A  gather of the new rows of A[P,P] and A[P,i] (Eq. 7),
//            which also extends the candidate universe (R7);
//   phase B  bordered (incremental) Cholesky + forward solve + psi (Eq. 9
//            denominator) for the new rows only: a right-looking column sweep
//            over the old columns (every lane folds its own columns, ascending k,
//            DESIGN.md C5-C6), the few new columns kept redundantly in every lane;
//   phase U  back-substitution g~ = L^-T y as a descending column sweep (C7);
//   exit     Eq. 16 (C8); output scaled by psi^-1/2 (Eqs. 8-9, C9).
// Compiled with -fmad=false: the only fused multiply-adds are the explicit fma()
// of the contract.  Several rows per warp turn the otherwise idle lanes of a
// short triangular sweep into instruction-level parallelism.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "setup_common.cuh"

namespace afsai {
namespace AFSAI_PNS {

// On-chip state of one row (one group), carved from dynamic shared memory.
struct RowState {
    real *inv, *y, *g, *L, *arow, *brow, *dscr, *hacc;
    int64_t *gstart;
    int32_t *hkey, *P, *sel, *selt, *glen, *misc, *coff;
    int16_t *clist, *clen;
    int8_t *hval;
    int M, CL;
};

__host__ __device__ inline int cand_cap(int H) { return (3 * H) / 4 + 8; }

__host__ __device__ inline int64_t row_state_bytes(int H, int M, int S, bool hacc) {
    const int CL = cand_cap(H);
    int64_t dbl = 3 * (int64_t)M + (M * (M + 1)) / 2 + 1 + (int64_t)S * M + S + 2 + (hacc ? H : 0);
    int64_t i64 = S;
    int64_t i32 = (int64_t)H + M + 3 * S + 4 + CL;
    int64_t i16 = 2 * (int64_t)CL;
    int64_t i8 = H;
    int64_t b = real_bytes(dbl) + i64 * 8 + i32 * 4 + i16 * 2 + i8;
    return (b + 15) & ~int64_t(15);
}

__device__ __forceinline__ RowState carve(char *base, const SetupKArgs &a, bool hacc) {
    RowState w;
    const int H = a.H, M = a.mmax, S = a.s;
    w.M = M;
    w.CL = cand_cap(H);
    real *d = reinterpret_cast<real *>(base);
    w.inv = d; d += M;
    w.y = d; d += M;
    w.g = d; d += M;
    w.L = d; d += (M * (M + 1)) / 2 + 1;
    w.arow = d; d += S * M;
    w.brow = d; d += S;
    w.dscr = d; d += 2;
    w.hacc = nullptr;
    if (hacc) { w.hacc = d; d += H; }
    int64_t *l8 = reinterpret_cast<int64_t *>(base + real_bytes(d - reinterpret_cast<real *>(base)));
    w.gstart = l8; l8 += S;
    int32_t *ip = reinterpret_cast<int32_t *>(l8);
    w.hkey = ip; ip += H;
    w.P = ip; ip += M;
    w.sel = ip; ip += S;
    w.selt = ip; ip += S;
    w.glen = ip; ip += S;
    w.misc = ip; ip += 4;
    w.coff = ip; ip += w.CL;
    int16_t *sp = reinterpret_cast<int16_t *>(ip);
    w.clist = sp; sp += w.CL;
    w.clen = sp; sp += w.CL;
    w.hval = reinterpret_cast<int8_t *>(sp);
    return w;
}

// Insert column c (< i) into the row's universe; a new key is appended to the
// candidate list together with its row extent (offset from row i, length).
// Returns the slot of an already present key, else -1.
__device__ __forceinline__ int universe_insert(const RowState &w, const SetupKArgs &a, int H, int log2H, int32_t c,
                                               int64_t e0i) {
    bool ins;
    const int sl = hinsert(w.hkey, H, log2H, c, &ins);
    if (sl < 0) {
        w.misc[1] = 1;
        return -1;
    }
    if (!ins) return sl;
    const int p = atomicAdd(&w.misc[2], 1);
    atomicAdd(&w.misc[0], 1);
    if (p >= w.CL) {
        w.misc[1] = 1;
        return -1;
    }
    // Columns below the exact halo (a_lo) are kmax+1 hops from i: they enter the
    // universe only at the last step's gather and are never evaluated, so they get
    // an empty extent instead of a rowptr read outside the halo.
    const bool inside = c >= a.a_lo;
    const int64_t e0 = inside ? rp_of(a, c) : e0i, e1 = inside ? rp_of(a, (int64_t)c + 1) : e0i;
    w.clist[p] = (int16_t)sl;
    w.coff[p] = (int32_t)(e0 - e0i);
    w.clen[p] = (int16_t)(e1 - e0);
    return -1;
}

// Kaporin-gradient fold of one chunk of row j (C3): storage order, pattern hits only
__device__ __forceinline__ void grad_fold(const RowState &w, int H, int log2H, int32_t i, const int32_t (&cc)[kGradChunk],
                                          const real (&vv)[kGradChunk], real &acc, unsigned long long &nfma,
                                          unsigned long long &nent) {
    real gv[kGradChunk];
    bool hit[kGradChunk];
#pragma unroll
    for (int u = 0; u < kGradChunk; ++u) {
        const int32_t r = cc[u];
        hit[u] = false;
        gv[u] = real(1);
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
            ++nfma;
        }
        nent += (cc[u] <= i);
    }
}

__device__ __forceinline__ void load_chunk(const SetupKArgs &a, int64_t eb, int cnt, int32_t (&cc)[kGradChunk],
                                           real (&vv)[kGradChunk]) {
#pragma unroll
    for (int u = 0; u < kGradChunk; ++u) {
        const bool in = u < cnt;
        cc[u] = in ? __ldg(a.col + eb + u) : 0x7fffffff;
        vv[u] = in ? __ldg(aval(a) + eb + u) : real(0);
    }
}

template <int LPR, int NT, int GS>
__global__ void __launch_bounds__(256, (LPR == 32 ? 2 : 1)) afsai_setup_rows_kernel(SetupKArgs a) {
    extern __shared__ __align__(16) char smem[];
    const int lane = threadIdx.x & 31;
    const Group<LPR> G(lane);
    const int gl = G.gl;
    const bool use_hacc = a.s > GS;
    RowState w = carve(smem + (size_t)(threadIdx.x / LPR) * a.warp_smem, a, use_hacc);
    const int H = a.H, log2H = a.log2H;
    unsigned long long c_steps = 0, c_border = 0, c_back = 0, c_gfma = 0, c_gent = 0;
    unsigned long long c_r0 = 0, c_r1 = 0, c_r2 = 0, c_r3 = 0, c_univ = 0;
    // per-phase SM cycles (group leader): prologue, gradient, select, gather, border, backsub, output
    long long ph[7] = {0, 0, 0, 0, 0, 0, 0};
    G.sync();
    long long tph = clock64();
#define PHASE(idx)                       \
    {                                    \
        const long long t1_ = clock64(); \
        ph[idx] += t1_ - tph;            \
        tph = t1_;                       \
    }

    for (;;) {
        unsigned long long t_idx = 0;
        if (gl == 0) t_idx = atomicAdd(a.work, 1ull);
        t_idx = G.bcast(t_idx, 0);
        if ((int64_t)t_idx >= a.nrows) break;
        const int64_t i64 = a.rows ? a.rows[t_idx] : a.row_lo + (int64_t)t_idx;
        const int32_t i = (int32_t)i64;
        const int64_t orow = i64 - a.out_base;
        const int64_t e0i = rp_of(a, i64), e1i = rp_of(a, i64 + 1);

        tph = clock64();
        // ---- prologue: empty table, universe = columns j < i of row i, a_ii
        for (int sl = gl; sl < H; sl += LPR) {
            w.hkey[sl] = kEmpty;
            w.hval[sl] = kCand;  // every key starts as a candidate
        }
        if (gl == 0) {
            w.misc[0] = 0;  // keys inserted
            w.misc[1] = 0;  // overflow
            w.misc[2] = 0;  // candidate list length
            w.dscr[0] = real(0);
        }
        G.sync();
        for (int64_t e = e0i + gl; e < e1i; e += LPR) {
            const int32_t c = a.col[e];
            if (c == i) w.dscr[0] = aval(a)[e];
            else if (c < i) universe_insert(w, a, H, log2H, c, e0i);
        }
        G.sync();
        const real a_ii = w.dscr[0];
        const real psi0 = a_ii;
        real psi = psi0;
        int m = 0, steps = 0, reason = AFSAI_STOP_KMAX;
        bool fail = false, overflow = (w.misc[1] != 0);
        int fail_code = 0, fail_step = 0;
        PHASE(0)

        for (int k = 1; k <= a.nsteps && !overflow; ++k) {
            int room = a.s;
            if (a.cap - 1 - m < room) room = a.cap - 1 - m;
            if (room <= 0) { reason = AFSAI_STOP_CAP; break; }

            // ---- phase G: gradient (C3), one lane per candidate, next row prefetched
            const int ncl = w.misc[2];
            int nc = 0;
            real ba[GS];
            int32_t bj[GS], bt[GS];
#pragma unroll
            for (int q = 0; q < GS; ++q) { ba[q] = -real(1); bj[q] = 0x7fffffff; bt[q] = -1; }
            {
                int t = gl;
                int32_t ncc[kGradChunk];
                real nvv[kGradChunk];
                int64_t neb = 0;
                int nlen = 0;
                if (t < ncl) {
                    neb = e0i + w.coff[t];
                    nlen = w.clen[t];
                    load_chunk(a, neb, nlen, ncc, nvv);
                }
                while (t < ncl) {
                    int32_t cc[kGradChunk];
                    real vv[kGradChunk];
#pragma unroll
                    for (int u = 0; u < kGradChunk; ++u) { cc[u] = ncc[u]; vv[u] = nvv[u]; }
                    const int64_t eb = neb;
                    const int len = nlen;
                    const int tc = t;
                    t += LPR;
                    if (t < ncl) {  // prefetch the next candidate's first chunk
                        neb = e0i + w.coff[t];
                        nlen = w.clen[t];
                        load_chunk(a, neb, nlen, ncc, nvv);
                    }
                    real acc = real(0);
                    grad_fold(w, H, log2H, i, cc, vv, acc, c_gfma, c_gent);
                    for (int off = kGradChunk; off < len && cc[kGradChunk - 1] < i; off += kGradChunk) {
                        load_chunk(a, eb + off, len - off, cc, vv);
                        grad_fold(w, H, log2H, i, cc, vv, acc, c_gfma, c_gent);
                    }
                    const int sl = w.clist[tc];
                    if (use_hacc) w.hacc[sl] = acc;
                    if (acc != real(0)) {
                        ++nc;
                        if (!use_hacc) {
                            real ca = fabs(acc);
                            int32_t cj = w.hkey[sl];
                            int32_t ct = tc;
#pragma unroll
                            for (int q = 0; q < GS; ++q) {
                                if (better(ca, cj, ba[q], bj[q])) {
                                    const real ta = ba[q];
                                    const int32_t tj = bj[q], t2 = bt[q];
                                    ba[q] = ca; bj[q] = cj; bt[q] = ct;
                                    ca = ta; cj = tj; ct = t2;
                                }
                            }
                        }
                    }
                }
            }
            nc = G.sum(nc);
            PHASE(1)
            if (nc == 0) { reason = AFSAI_STOP_NOCAND; break; }
            const int nsel = nc < room ? nc : room;

            // ---- phase S: top-nsel under the total order (|acc| desc, j asc)
            if (!use_hacc) {
                for (int u = 0; u < nsel; ++u) {
                    real wa = ba[0];
                    int32_t wj = bj[0];
#pragma unroll
                    for (int o = LPR / 2; o > 0; o >>= 1) {
                        const real oa = G.xorv(wa, o);
                        const int32_t oj = G.xorv(wj, o);
                        if (better(oa, oj, wa, wj)) { wa = oa; wj = oj; }
                    }
                    if (bj[0] == wj) {  // column indices are unique: exactly one lane
                        w.sel[u] = wj;
                        w.selt[u] = bt[0];
#pragma unroll
                        for (int q = 0; q + 1 < GS; ++q) { ba[q] = ba[q + 1]; bj[q] = bj[q + 1]; bt[q] = bt[q + 1]; }
                        ba[GS - 1] = -real(1); bj[GS - 1] = 0x7fffffff; bt[GS - 1] = -1;
                    }
                }
            } else {
                // s > GS: nsel rounds of group argmax over the candidate list
                for (int u = 0; u < nsel; ++u) {
                    real xa = -real(1);
                    int32_t xj = 0x7fffffff, xt = -1;
                    for (int t = gl; t < ncl; t += LPR) {
                        const int sl = w.clist[t];
                        if (w.hval[sl] != kCand) continue;
                        const real aa = fabs(w.hacc[sl]);
                        if (aa == real(0)) continue;
                        const int32_t j = w.hkey[sl];
                        if (better(aa, j, xa, xj)) { xa = aa; xj = j; xt = t; }
                    }
#pragma unroll
                    for (int o = LPR / 2; o > 0; o >>= 1) {
                        const real oa = G.xorv(xa, o);
                        const int32_t oj = G.xorv(xj, o);
                        const int32_t ot = G.xorv(xt, o);
                        if (better(oa, oj, xa, xj)) { xa = oa; xj = oj; xt = ot; }
                    }
                    if (gl == 0) {
                        w.sel[u] = xj;
                        w.selt[u] = xt;
                        w.hval[w.clist[xt]] = -3;  // taken
                    }
                    G.sync();
                }
            }
            G.sync();
            // append in ascending column order (R9); extents of the rows to gather
            if (gl < nsel) {
                const int32_t j = w.sel[gl];
                int rank = 0;
                for (int u = 0; u < nsel; ++u) rank += (w.sel[u] < j);
                const int tsel = w.selt[gl];
                w.P[m + rank] = j;
                w.hval[w.clist[tsel]] = (int8_t)(m + rank);
                w.gstart[rank] = e0i + w.coff[tsel];
                w.glen[rank] = w.clen[tsel];
            }
            G.sync();
            // drop the selected slots from the candidate list (in-group compaction)
            {
                int wr = 0;
                for (int base = 0; base < ncl; base += LPR) {
                    const int t = base + gl;
                    int sl = 0, of = 0, ln_ = 0;
                    if (t < ncl) { sl = w.clist[t]; of = w.coff[t]; ln_ = w.clen[t]; }
                    const bool keep = t < ncl && w.hval[sl] == kCand;
                    const unsigned bal = __ballot_sync(G.mask, keep) >> (lane & ~(LPR - 1));
                    G.sync();
                    if (keep) {
                        const int p = wr + __popc(bal & ((1u << gl) - 1u));
                        w.clist[p] = (int16_t)sl;
                        w.coff[p] = of;
                        w.clen[p] = (int16_t)ln_;
                    }
                    wr += __popc(bal);
                    G.sync();
                }
                if (gl == 0) w.misc[2] = wr;
            }
            // zero the gathered rows
            for (int x = gl; x < nsel * w.M; x += LPR) w.arow[x] = real(0);
            if (gl < nsel) w.brow[gl] = real(0);
            G.sync();
            PHASE(2)

            // ---- phase A: gather rows P_q (q = m..m+nsel-1) of A, all rows at once;
            //      extend the universe with their columns (R7)
            {
                int total = 0;
                for (int u = 0; u < nsel; ++u) total += w.glen[u];
                for (int t = gl; t < total; t += LPR) {
                    int u = 0, off = t;
                    while (off >= w.glen[u]) { off -= w.glen[u]; ++u; }
                    const int64_t e = w.gstart[u] + off;
                    const int32_t c = __ldg(a.col + e);
                    if (c == i) w.brow[u] = __ldg(aval(a) + e);
                    else if (c < i) {
                        const int sl = universe_insert(w, a, H, log2H, c, e0i);
                        if (sl >= 0) {
                            const int st = w.hval[sl];
                            if (st >= 0 && st <= m + u) w.arow[u * w.M + st] = __ldg(aval(a) + e);
                        }
                    }
                }
            }
            G.sync();
            PHASE(3)
            if (w.misc[1] != 0 || w.misc[0] * 4 > H * 3) { overflow = true; break; }

            // ---- phase B: bordered Cholesky of the new rows, in lockstep groups of GS
            for (int ug = 0; ug < nsel && !fail; ug += GS) {
                const int gs = (nsel - ug) < GS ? (nsel - ug) : GS;
                if (!border_group<LPR, NT, GS>(w, G, m + ug, gs, ug, psi)) {
                    fail = true;
                    fail_code = AFSAI_ENOTSPD;
                    fail_step = k;
                }
            }
            if (fail) break;
            for (int u = 0; u < nsel; ++u) {
                const long q = m + u;
                c_border += (unsigned long long)(q * (q - 1) / 2 + 2 * q + 1);
            }
            m += nsel;
            if (!(psi > real(0))) { fail = true; fail_code = AFSAI_ENOTSPD; fail_step = k; break; }
            PHASE(4)

            // ---- phase U: back-substitution
            back_substitute<LPR, NT>(w, G, m);
            c_back += (unsigned long long)(m * (m - 1) / 2);
            steps = k;
            PHASE(5)
            // ---- Eq. 16 exit test (C8)
            if (psi / psi0 <= a.eps) { reason = AFSAI_STOP_TOL; break; }
        }

        if (overflow) {
            if (gl == 0) {
                const int p = atomicAdd(a.retry_count, 1);
                a.retry_rows[p] = i64;
            }
            G.sync();
            continue;
        }
        if (fail) {
            if (gl == 0) {
                const unsigned long long code = ((unsigned long long)i64 << 24) |
                                                ((unsigned long long)(fail_step & 0xfffff) << 4) |
                                                (unsigned long long)fail_code;
                atomicMin(a.err, code);
                a.nnz_row[orow] = 0;
            }
            G.sync();
            continue;
        }
        // ---- output: d = psi^-1/2 (Eqs. 8-9), row sorted by column (C9)
        const real d = real(1) / sqrt(psi);
        int32_t *oc = a.scol + orow * a.stride;
        double *ov = a.sval + orow * a.stride;
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) {
            const int q = gl + LPR * tt;
            if (q < m) {
                const int32_t pj = w.P[q];
                int rank = 0;
                for (int q2 = 0; q2 < m; ++q2) rank += (w.P[q2] < pj);
                oc[rank] = pj;
                ov[rank] = w.g[q] * d;
            }
        }
        if (gl == 0) {
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
        G.sync();
        PHASE(6)
    }
#undef PHASE
    // ---- statistics (one atomic per group and counter)
    const unsigned long long g1 = G.sum(c_gfma), g2 = G.sum(c_gent);
    if (gl == 0) {
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

}  // namespace AFSAI_PNS
}  // namespace afsai

namespace afsai {
namespace AFSAI_PNS {
// ---------------------------------------------------------------- host side
template <int LPR, int NT>
static SetupKernFn scan_gs(int gs) {
    switch (gs) {
        case 1: return afsai_setup_rows_kernel<LPR, NT, 1>;
        case 2: return afsai_setup_rows_kernel<LPR, NT, 2>;
        case 3: return afsai_setup_rows_kernel<LPR, NT, 3>;
        default: return afsai_setup_rows_kernel<LPR, NT, 4>;
    }
}

template <int LPR>
static SetupKernFn scan_nt(int nt, int gs) {
    switch (nt) {
        case 1: return scan_gs<LPR, 1>(gs);
        case 2: return scan_gs<LPR, 2>(gs);
        case 3: return scan_gs<LPR, 3>(gs);
        case 4: return scan_gs<LPR, 4>(gs);
        case 5: return scan_gs<LPR, 5>(gs);
        default: return scan_gs<LPR, 6>(gs);
    }
}

SetupKernFn scan_kernel_for(int lpr, int mmax, int s) {
    const int m = mmax < 1 ? 1 : mmax;
    const int nt = (m + lpr - 1) / lpr;
    const int gs = s < kMaxGroup ? s : kMaxGroup;
    if (lpr == 16) return scan_nt<16>(nt, gs);
    return nt <= 4 ? scan_nt<32>(nt, gs) : nullptr;
}

int64_t scan_row_bytes(int H, int mmax, int s) {
    const int gs = s < kMaxGroup ? s : kMaxGroup;
    return row_state_bytes(H, mmax, s, s > gs);
}
}  // namespace AFSAI_PNS
}  // namespace afsai
