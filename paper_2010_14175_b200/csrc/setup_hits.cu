// setup_hits.cu -- hit-list variant of the per-row set-up kernel (short rows).
#include "setup_hits.cuh"

namespace afsai {
namespace AFSAI_PNS {

// ======================================================================
// Hit-list variant for matrices with short rows (max row length - 1 <= HC).
//
// Every candidate j keeps the list of its "hits" -- the pairs (r, a_jr) with r in
// P U {i} -- sorted by r.  A hit is recorded when its pattern row r is gathered
// (a_jr is read from row r at column j; A is bitwise symmetric, C1),
// so the gradient of every step (C3) is a short shared-memory fold per
// candidate: no loads of candidate rows, no hash look-ups.  The fold visits the
// hits in ascending r, exactly as the scan of row j in storage order does.
// ======================================================================
// One pass over the entries of one row of A (row r, pattern position q; q = -1
// for row i itself): extend the universe, record hits, and (q >= 0) gather the
// row of the local system.  Rows are short (<= LPR entries): lane t holds entry
// t (c, v), loaded by the caller.  Keys are unique within a row, so the lanes
// never touch the same slot concurrently.  New candidates get active slots
// through a group-aggregated allocation (free stack first, then high-water).
template <int LPR, int HC>
__device__ void scan_row_hits(const HitState &w, const Group<LPR> &G, int H, int log2H, int32_t i, bool valid,
                              int32_t c, real v, int32_t e, int q, real *arow_u, real *brow_u) {
    const int CA = w.CA;
    const int32_t r = q < 0 ? i : w.P[q];
    bool need = false;
    int sl = -1;
    if (valid) {
        if (c == i) {
            if (q >= 0) *brow_u = v;
            else w.dscr[0] = v;
        } else if (c < i) {
            bool ins;
            sl = hinsert(w.hkey, H, log2H, c, &ins);
            if (sl < 0) w.misc[1] = 1;
            else if (ins) need = true;
            else {
                const int st = w.hval[sl];
                if (st >= 0) {
                    if (q >= 0 && st <= q) arow_u[st] = v;  // gather A[P_q, P_st]
                } else if (st <= -2) {
                    hit_insert<HC>(w, -2 - st, q, r, AFSAI_HIT(v, e));  // existing candidate: new hit
                }                                            // st == -1: dropped (row overflowed)
            }
        }
    }
    // group-aggregated allocation of active slots for the new candidates
    const unsigned bal = __ballot_sync(G.mask, need) >> (threadIdx.x & 31 & ~(LPR - 1));
    if (bal) {
        const int nf = w.misc[3], hw = w.misc[2];
        G.sync();
        if (need) {
            const int rk = __popc(bal & ((1u << G.gl) - 1u));
            const int aa = rk < nf ? w.afree[nf - 1 - rk] : hw + (rk - nf);
            if (aa >= CA) {
                w.misc[1] = 1;          // the row is retried with larger tables;
                w.hval[sl] = (int8_t)-1;  // the key must not decode as an active slot
            } else {
                w.hval[sl] = (int8_t)(-2 - aa);
                w.akey[aa] = c;
                w.ahs[aa] = (int16_t)sl;
                w.ahn[aa] = 1;
                w.ahq[aa] = (int8_t)q;
                w.hv[aa] = AFSAI_HIT(v, e);
            }
            atomicAdd(&w.misc[0], 1);
        }
        const int k = __popc(bal);
        if (G.gl == 0) {
            const int take = k < nf ? k : nf;
            w.misc[3] = nf - take;
            w.misc[2] = hw + (k - take);
        }
    }
    G.sync();
}

template <int LPR, int NT, int GS, int HC>
__global__ void __launch_bounds__(256, (LPR == 32 ? 2 : 1)) afsai_setup_rows_hits_kernel(SetupKArgs a) {
    extern __shared__ __align__(16) char smem[];
    const int lane = threadIdx.x & 31;
    const Group<LPR> G(lane);
    const int gl = G.gl;
    const bool use_acc = a.s > GS;
    HitState w = carve_hits<HC>(smem + (size_t)(threadIdx.x / LPR) * a.warp_smem, a, use_acc);
    const int H = a.H, log2H = a.log2H, CA = w.CA;
    unsigned long long c_steps = 0, c_border = 0, c_back = 0, c_gfma = 0;
    unsigned long long c_r0 = 0, c_r1 = 0, c_r2 = 0, c_r3 = 0, c_univ = 0;
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
        for (int sl = gl; sl < H; sl += LPR) {
            w.hkey[sl] = kEmpty;
            w.hval[sl] = (int8_t)-1;  // no stale shared memory is ever decoded
        }
        for (int x = gl; x < CA; x += LPR) w.ahn[x] = 0;
        if (gl == 0) {
            w.misc[0] = 0;
            w.misc[1] = 0;
            w.misc[2] = 0;
            w.misc[3] = 0;
            w.dscr[0] = real(0);
        }
        G.sync();
        // universe = columns j < i of row i, each with its hit (i, a_ji)
        {
            const bool vi = gl < (int)(e1i - e0i);
            const int32_t ci = vi ? __ldg(a.col + e0i + gl) : 0;
            const real xi = vi ? __ldg(aval(a) + e0i + gl) : real(0);
            scan_row_hits<LPR, HC>(w, G, H, log2H, i, vi, ci, xi, G.gl, -1, nullptr, nullptr);
        }
        const real a_ii = w.dscr[0];
        const real psi0 = a_ii;
        real psi = psi0;
        int m = 0, steps = 0, reason = AFSAI_STOP_KMAX;
        bool fail = false, overflow = (w.misc[1] != 0);
        int fail_step = 0;
        PHASE(0)
        for (int k = 1; k <= a.nsteps && !overflow; ++k) {
            int room = a.s;
            if (a.cap - 1 - m < room) room = a.cap - 1 - m;
            if (room <= 0) { reason = AFSAI_STOP_CAP; break; }
            // ---- phase G: gradient = fold of each active candidate's hits (C3)
            const int hw = w.misc[2];
            int nc = 0;
            real ba[GS];
            int32_t bj[GS], bt[GS];
#pragma unroll
            for (int q = 0; q < GS; ++q) { ba[q] = -real(1); bj[q] = 0x7fffffff; bt[q] = -1; }
            for (int aa = gl; aa < hw; aa += LPR) {
                const int n = w.ahn[aa];
                if (n == 0) continue;  // free slot
                real acc = real(0);
#pragma unroll
                for (int h = 0; h < HC; ++h) {
                    if (h < n) {
                        const int q = w.ahq[h * CA + aa];
                        const real gv = q < 0 ? real(1) : w.g[q];
                        acc = fma(__ldg(aval(a) + (q < 0 ? e0i : (int64_t)w.prs[q]) + w.hv[h * CA + aa]), gv, acc);
                    }
                }
                c_gfma += n;
                if (use_acc) w.acc[aa] = acc;
                if (acc != real(0)) {
                    ++nc;
                    if (!use_acc) {
                        real ca = fabs(acc);
                        int32_t cj = w.akey[aa];
                        int32_t ct = aa;
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
            nc = G.sum(nc);
            PHASE(1)
            if (nc == 0) { reason = AFSAI_STOP_NOCAND; break; }
            const int nsel = nc < room ? nc : room;
            // ---- phase S: top-nsel under (|acc| desc, j asc)
            if (!use_acc) {
                for (int u = 0; u < nsel; ++u) {
                    real wa = ba[0];
                    int32_t wj = bj[0];
#pragma unroll
                    for (int o = LPR / 2; o > 0; o >>= 1) {
                        const real oa = G.xorv(wa, o);
                        const int32_t oj = G.xorv(wj, o);
                        if (better(oa, oj, wa, wj)) { wa = oa; wj = oj; }
                    }
                    if (bj[0] == wj) {
                        w.sel[u] = wj;
                        w.sela[u] = bt[0];
#pragma unroll
                        for (int q = 0; q + 1 < GS; ++q) { ba[q] = ba[q + 1]; bj[q] = bj[q + 1]; bt[q] = bt[q + 1]; }
                        ba[GS - 1] = -real(1); bj[GS - 1] = 0x7fffffff; bt[GS - 1] = -1;
                    }
                }
            } else {
                for (int u = 0; u < nsel; ++u) {
                    real xa = -real(1);
                    int32_t xj = 0x7fffffff, xt = -1;
                    for (int aa = gl; aa < hw; aa += LPR) {
                        if (w.ahn[aa] <= 0) continue;
                        const real av = fabs(w.acc[aa]);
                        if (av == real(0)) continue;
                        const int32_t j = w.akey[aa];
                        if (better(av, j, xa, xj)) { xa = av; xj = j; xt = aa; }
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
                        w.sela[u] = xt;
                        w.ahn[xt] = -1;  // taken (excluded from later rounds)
                    }
                    G.sync();
                }
            }
            G.sync();
            // positions in ascending column order (R9); free the selected slots
            if (gl < nsel) {
                const int32_t j = w.sel[gl];
                int rank = 0;
                for (int u = 0; u < nsel; ++u) rank += (w.sel[u] < j);
                const int aa = w.sela[gl];
                w.P[m + rank] = j;
                w.hval[w.ahs[aa]] = (int8_t)(m + rank);
                const int64_t g0 = rp_of(a, j), g1 = rp_of(a, (int64_t)j + 1);
                w.gstart[rank] = g0;
                w.prs[m + rank] = (int32_t)g0;
                w.glen[rank] = (int32_t)(g1 - g0);
                w.ahn[aa] = 0;
                w.afree[w.misc[3] + gl] = (int16_t)aa;
            }
            for (int x = gl; x < nsel * w.M; x += LPR) w.arow[x] = real(0);
            if (gl < nsel) w.brow[gl] = real(0);
            G.sync();
            if (gl == 0) w.misc[3] += nsel;
            G.sync();
            PHASE(2)
            // ---- phase A: gather the new rows (one row per pass), record hits
            for (int ug = 0; ug < nsel; ug += GS) {
                int32_t pc[GS], pe[GS];
                real pv[GS];
                bool pvld[GS];
#pragma unroll
                for (int u = 0; u < GS; ++u) {  // every row's entries in flight at once
                    pvld[u] = (ug + u < nsel) && gl < w.glen[ug + u];
                    pe[u] = gl;   // the entry's position within its row
                    pc[u] = pvld[u] ? __ldg(a.col + w.gstart[ug + u] + gl) : 0;
                    pv[u] = pvld[u] ? __ldg(aval(a) + w.gstart[ug + u] + gl) : real(0);
                }
#pragma unroll
                for (int u = 0; u < GS; ++u)
                    if (ug + u < nsel)
                        scan_row_hits<LPR, HC>(w, G, H, log2H, i, pvld[u], pc[u], pv[u], pe[u], m + ug + u,
                                               w.arow + (ug + u) * w.M, w.brow + ug + u);
            }
            PHASE(3)
            if (w.misc[1] != 0 || w.misc[0] * 4 > H * 3) { overflow = true; break; }
            // ---- phase B / U: bordered Cholesky, back-substitution
            for (int ug = 0; ug < nsel && !fail; ug += GS) {
                const int gs = (nsel - ug) < GS ? (nsel - ug) : GS;
                if (!border_group<LPR, NT, GS>(w, G, m + ug, gs, ug, psi)) {
                    fail = true;
                    fail_step = k;
                }
            }
            if (fail) break;
            for (int u = 0; u < nsel; ++u) {
                const long q = m + u;
                c_border += (unsigned long long)(q * (q - 1) / 2 + 2 * q + 1);
            }
            m += nsel;
            if (!(psi > real(0))) { fail = true; fail_step = k; break; }
            PHASE(4)
            back_substitute<LPR, NT>(w, G, m);
            c_back += (unsigned long long)(m * (m - 1) / 2);
            steps = k;
            PHASE(5)
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
                                                (unsigned long long)AFSAI_ENOTSPD;
                atomicMin(a.err, code);
                a.nnz_row[orow] = 0;
            }
            G.sync();
            continue;
        }
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
    const unsigned long long g1 = G.sum(c_gfma);
    if (gl == 0) {
        atomicAdd(&a.counters[0], c_steps);
        atomicAdd(&a.counters[1], c_border);
        atomicAdd(&a.counters[2], c_back);
        atomicAdd(&a.counters[3], g1);
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
template <int LPR, int NT, int HC>
static SetupKernFn hits_gs(int gs) {
    switch (gs) {
        case 1: return afsai_setup_rows_hits_kernel<LPR, NT, 1, HC>;
        case 2: return afsai_setup_rows_hits_kernel<LPR, NT, 2, HC>;
        case 3: return afsai_setup_rows_hits_kernel<LPR, NT, 3, HC>;
        default: return afsai_setup_rows_hits_kernel<LPR, NT, 4, HC>;
    }
}

template <int LPR, int HC>
static SetupKernFn hits_nt(int nt, int gs) {
    switch (nt) {
        case 1: return hits_gs<LPR, 1, HC>(gs);
        case 2: return hits_gs<LPR, 2, HC>(gs);
        case 3: return hits_gs<LPR, 3, HC>(gs);
        case 4: return hits_gs<LPR, 4, HC>(gs);
        case 5: return hits_gs<LPR, 5, HC>(gs);
        default: return hits_gs<LPR, 6, HC>(gs);
    }
}

SetupKernFn hits_kernel_for(int lpr, int mmax, int s, int hc) {
    const int m = mmax < 1 ? 1 : mmax;
    const int nt = (m + lpr - 1) / lpr;
    const int gs = s < kMaxGroup ? s : kMaxGroup;
    if (lpr == 16) return hc <= 6 ? hits_nt<16, 6>(nt, gs) : hits_nt<16, 8>(nt, gs);
    if (nt > 4) return nullptr;
    return hc <= 6 ? hits_nt<32, 6>(nt, gs) : hits_nt<32, 8>(nt, gs);
}

int64_t hits_row_bytes(int H, int mmax, int s, int cact, int hc) {
    const int gs = s < kMaxGroup ? s : kMaxGroup;
    return hc <= 6 ? hit_state_bytes<6>(H, mmax, s, cact, s > gs) : hit_state_bytes<8>(H, mmax, s, cact, s > gs);
}
}  // namespace AFSAI_PNS
}  // namespace afsai
