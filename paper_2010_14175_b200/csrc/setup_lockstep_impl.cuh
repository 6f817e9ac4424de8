// setup_lockstep_impl.cuh -- hit-list set-up kernel, several rows per warp in LOCKSTEP.
//
// Same algorithm and arithmetic as setup_hits.cu (C1-C12), but the
// 32/LPR rows of a warp advance together: every loop that contains a shuffle
// or a warp barrier runs to the warp-uniform maximum of its trip count and
// each row's updates are predicated (by selects, so the arithmetic of a live
// row is exactly the unpredicated one).  Two things follow:
//  - shuffles use the full warp mask (no per-shuffle convergence checks), and
//  - every stage of the triangular sweeps does the work of all the warp's rows
//    at once: with 8 lanes per row each lane folds up to 6 columns per stage,
//    so the fixed per-stage cost (operand loads, the broadcast, the owner's
//    store, the loop) is shared by four rows.
// Used for short rows (<= LPR entries, stencils) and s <= 4.
#pragma once
#include "setup_hits.cuh"

namespace afsai {
namespace AFSAI_PNS {

constexpr unsigned kAll = 0xffffffffu;

template <int LPR>
struct LGroup {
    int gl;
    __device__ explicit LGroup(int lane) : gl(lane & (LPR - 1)) {}
    template <class T>
    __device__ __forceinline__ T bcast(T v, int src) const { return __shfl_sync(kAll, v, src, LPR); }
    template <class T>
    __device__ __forceinline__ T xorv(T v, int o) const { return __shfl_xor_sync(kAll, v, o, LPR); }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
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
    // this group's bits of a full-warp ballot
    __device__ __forceinline__ unsigned ballot(bool p) const {
        const unsigned b = __ballot_sync(kAll, p) >> ((threadIdx.x & 31) & ~(LPR - 1));
        return LPR == 32 ? b : (b & ((1u << LPR) - 1u));
    }
};

__device__ __forceinline__ int warp_max(int v) { return (int)__reduce_max_sync(kAll, (unsigned)(v < 0 ? 0 : v)); }

// Per-row bookkeeping of the hit-list tables, held in registers with identical
// values in every lane of the row's group (updated from ballots; no shared-memory
// round trips, atomics or barriers): keys in the table, active-slot high-water
// mark, size of the free-slot stack; ovf = this lane saw a table overflow.
struct RowBook {
    int nkeys, hw, nf;
    bool ovf;
    unsigned why;  // overflow reasons: 1 hash table, 2 active candidate slots, 4 hit list
};

// hit_insert of setup_hits.cuh; returns false when the list is full
template <int HC>
__device__ __forceinline__ bool hit_insert_ls(const HitState &w, int aa, int q, int32_t r, hit_t v) {
    const int CA = w.CA;
    const int n = w.ahn[aa];
    if (n >= HC) return false;
    int pos = n;
    while (pos > 0) {
        const int qp = w.ahq[(pos - 1) * CA + aa];
        const int32_t rp = qp < 0 ? 0x7fffffff : w.P[qp];
        if (rp <= r) break;
        w.ahq[pos * CA + aa] = (int8_t)qp;
        w.hv[pos * CA + aa] = w.hv[(pos - 1) * CA + aa];
        --pos;
    }
    w.ahq[pos * CA + aa] = (int8_t)q;
    w.hv[pos * CA + aa] = v;
    w.ahn[aa] = (int8_t)(n + 1);
    return true;
}

// scan_row_hits of setup_hits.cu with the slot allocation made warp-uniform: the
// entry (c, v) of row P_q (q = -1: row i itself) of every lane joins the row's
// universe: a pattern column is gathered into the local system, an existing
// candidate gets the hit (r = P_q, v), a new column becomes a candidate.  All
// lanes of the warp call it (ballot); one barrier at the end publishes the
// tables to the next call.
template <int LPR, int HC>
__device__ void scan_row_hits_ls(const HitState &w, const LGroup<LPR> &G, int H, int log2H, int32_t i, bool valid,
                                 int32_t c, real v, int32_t e, int q, real *arow_u, real *brow_u, RowBook &b) {
    const int CA = w.CA;
    bool need = false;
    int sl = -1;
    if (valid) {
        if (c == i) {
            if (q >= 0) *brow_u = v;
            else w.dscr[0] = v;
        } else if (c < i) {
            bool ins;
            sl = hinsert(w.hkey, H, log2H, c, &ins);
            if (sl < 0) { b.ovf = true; b.why |= 1u; }
            else if (ins) need = true;
            else {
                const int st = w.hval[sl];
                if (st >= 0) {
                    if (q >= 0 && st <= q) arow_u[st] = v;  // gather A[P_q, P_st]
                } else if (st <= -2) {                      // existing candidate: new hit
                    const int32_t r = q < 0 ? i : w.P[q < w.M ? q : 0];
                    if (!hit_insert_ls<HC>(w, -2 - st, q, r, AFSAI_HIT(v, e))) { b.ovf = true; b.why |= 4u; }
                }                                            // st == -1: dropped (row overflowed)
            }
        }
    }
    const unsigned bal = G.ballot(need);
    if (need) {
        const int rk = __popc(bal & ((1u << G.gl) - 1u));
        const int aa = rk < b.nf ? w.afree[b.nf - 1 - rk] : b.hw + (rk - b.nf);
        if (aa >= CA) {
            b.ovf = true;             // the row is retried with larger tables;
            b.why |= 2u;
            w.hval[sl] = (int8_t)-1;  // the key must not decode as an active slot
        } else {
            w.hval[sl] = (int8_t)(-2 - aa);
            w.ahs[aa] = (int16_t)sl;
            w.ahn[aa] = 1;
            w.ahq[aa] = (int8_t)q;
            w.hv[aa] = AFSAI_HIT(v, e);
        }
    }
    const int k = __popc(bal);
    const int take = k < b.nf ? k : b.nf;
    b.nf -= take;
    b.hw += k - take;
    b.nkeys += k;
    G.sync();
}

// predicated fma: if (p) d = fma(a, b, d), as one predicated DFMA / FFMA (no selects,
// no temporaries; a plain `if` around fma() compiles to DFMA + two moves)
__device__ __forceinline__ void fma_if(bool p, double a, double b, double &d) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q fma.rn.f64 %0, %1, %2, %0;\n\t}"
        : "+d"(d)
        : "d"(a), "d"(b), "r"((int)p));
}
__device__ __forceinline__ void fma_if(bool p, float a, float b, float &d) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q fma.rn.f32 %0, %1, %2, %0;\n\t}"
        : "+f"(d)
        : "f"(a), "f"(b), "r"((int)p));
}

// Bordered Cholesky of the new rows q = qf .. qf+gs-1 (gathered into their L rows), forward
// solve and psi update, in lockstep: the old-column stages run to the warp maximum
// qf_max; a row's updates happen only while live (active && k < qf).
//  - right-looking column sweep: at stage k the owner lane of column k turns its
//    accumulator into L[q][k] = t * inv[k] and broadcasts it; every lane folds
//    fma(-L[q][k], L[c][k], t_c) into its columns.  The owner multiplies by the
//    inverse diagonal of its own column, held in a register (no per-stage load on
//    the broadcast's critical path); the stage's shared-memory operands are
//    loaded first and arrive during the DMUL -> SHFL.
//  - finalized accumulators are dead: folded unpredicated (their loads read any
//    in-bounds row of L).
//  - the group's own columns (diagonal of each new row, couplings among the new
//    rows) are kept redundantly in every lane.
// Every accumulator folds in k-ascending order, exactly DESIGN.md C5.  One copy of
// the stage per column chunk and no unrolling: the kernel is instruction-cache bound
// when its code grows.  Returns false on a pivot !(> 1e-30).
template <int LPR, int NT, int GS>
__device__ bool border_group_ls(const HitState &w, const LGroup<LPR> &G, bool active, int qf, int gs, int ug,
                                int qf_max, real &psi) {
    const int M = w.M, gl = G.gl;
    real t[GS][NT], dg[GS], ty[GS], cp[GS][GS], ivc[NT];
    real *Lnew[GS];
    const real *Lr[NT];
    bool st[GS];
#pragma unroll
    for (int u = 0; u < GS; ++u) {
        const real *ar = w.L + tri(qf + u < M ? qf + u : 0);  // the gathered row, in place (compact state)
        const bool ur = active && u < gs;
        st[u] = ur;
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) {
            const int c = gl + LPR * tt;
            t[u][tt] = (ur && c < qf) ? ar[c] : real(0);
        }
        dg[u] = ur ? ar[qf + u] : real(0);
#pragma unroll
        for (int v = 0; v < GS; ++v) cp[u][v] = (v < u && ur) ? ar[qf + v] : real(0);
        ty[u] = ur ? -w.brow[ug + u] : real(0);
        Lnew[u] = w.L + tri(qf + u < M ? qf + u : 0);
    }
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        const int c = gl + LPR * tt;
        const bool old = active && c < qf;
        Lr[tt] = old ? w.L + tri(c) : w.L;  // dead columns: any in-bounds row
        ivc[tt] = old ? w.L[tri(c) + c] : real(0);  // 1/L[c][c] in the diagonal slot
    }
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        int lnend = qf_max - LPR * tt;
        if (lnend > LPR) lnend = LPR;
#pragma unroll 1
        for (int ln = 0; ln < lnend; ++ln) {
            const int k = LPR * tt + ln;
            const bool live = active && k < qf;
            const real y_k = w.y[k];
            real lsm[NT];
#pragma unroll
            for (int t2 = tt; t2 < NT; ++t2) lsm[t2] = Lr[t2][k];
            real l[GS];
            // the owner stores L[q][k] (a predicated store, no divergence) and every
            // lane reads it back: a shared-memory broadcast instead of 64-bit shuffles
#pragma unroll
            for (int u = 0; u < GS; ++u)
                if (gl == ln && live && st[u]) Lnew[u][k] = t[u][tt] * ivc[tt];
            G.sync();
#pragma unroll
            for (int u = 0; u < GS; ++u) l[u] = Lnew[u][k];  // dead rows: any value, folded into dead state
#pragma unroll
            for (int t2 = tt; t2 < NT; ++t2)
#pragma unroll
                for (int u = 0; u < GS; ++u) t[u][t2] = fma(-l[u], lsm[t2], t[u][t2]);
#pragma unroll
            for (int u = 0; u < GS; ++u) {
                fma_if(live, -l[u], l[u], dg[u]);
                fma_if(live, -l[u], y_k, ty[u]);
#pragma unroll
                for (int v = 0; v < GS; ++v)
                    if (v < u) fma_if(live, -l[u], l[v], cp[u][v]);
            }
        }
    }
    // the group's own columns (no shuffles: per row, divergence allowed)
    bool ok = true;
    if (active) {
#pragma unroll
        for (int uf = 0; uf < GS; ++uf) {
            if (uf >= gs) break;
            const int k = qf + uf;
            const real piv = dg[uf];
            if (!(piv > 1e-30)) {
                ok = false;
                break;
            }
            const real dq = sqrt(piv);  // C5.2
            const real inv_k = real(1) / dq;
            const real y_k = ty[uf] * inv_k;
            psi = fma(-y_k, y_k, psi);     // C6
            w.L[tri(k) + k] = inv_k;  // 1/L[k][k] (diagonal slot); every lane stores the same bits
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
    }
    G.sync();
    return ok;
}

// Back-substitution g~ = L^-T y (C7) in lockstep (stages to the warp
// maximum m_max): descending column sweep; lane c folds fma(-L[k][c], g[k], t_c) for
// k = m-1 down to c+1.  Row k of L is read contiguously by the lanes (a running
// pointer: tri(k-1) = tri(k) - k); reads past the row's live columns land inside the
// row's shared-memory region (carve_hits: brow, dscr and the integer arrays follow
// L) and feed dead
// accumulators; a row's folds are predicated on its live stages (k < m).
template <int LPR, int NT>
__device__ void back_substitute_ls(const HitState &w, const LGroup<LPR> &G, bool active, int m, int m_max) {
    const int gl = G.gl;
    real tb[NT], ivc[NT];
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
        const int c = gl + LPR * tt;
        const bool in = active && c < m;
        tb[tt] = in ? w.y[c] : real(0);
        ivc[tt] = in ? w.L[tri(c) + c] : real(0);
    }
    const real *pk = w.L + tri(m_max > 0 ? m_max - 1 : 0) + gl;  // row k, this lane's first column
#pragma unroll
    for (int tt = NT - 1; tt >= 0; --tt) {
        int ln0 = m_max - 1 - LPR * tt;
        if (ln0 > LPR - 1) ln0 = LPR - 1;
#pragma unroll 1
        for (int ln = ln0; ln >= 0; --ln) {
            const int k = LPR * tt + ln;
            const bool live = active && k < m;
            real lk[NT];
#pragma unroll
            for (int t2 = 0; t2 <= tt; ++t2) lk[t2] = pk[LPR * t2];  // L[k][c]; c >= k: dead
            pk -= k;
            if (gl == ln && live) w.g[k] = tb[tt] * ivc[tt];
            G.sync();
            const real gk = w.g[k];
#pragma unroll
            for (int t2 = 0; t2 <= tt; ++t2) fma_if(live, -lk[t2], gk, tb[t2]);
        }
    }
    G.sync();
}


template <int LPR, int NT, int GS, int HC>
// 16 lanes per row: <= 170 registers (three warps per SMSP register file) and CTAs
// of up to three warps (six rows: the per-CTA shared-memory reserve then fits 18
// rows per SM)
__global__ void __launch_bounds__(LPR == 16 ? 96 : 256, LPR == 16 ? 4 : 1) afsai_setup_rows_lockstep_kernel(SetupKArgs a) {
    extern __shared__ __align__(16) char smem[];
    constexpr int RPW = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const LGroup<LPR> G(lane);
    const int gl = G.gl;
    HitState w = carve_hits<HC>(smem + (size_t)(threadIdx.x / LPR) * a.warp_smem, a, false, true);
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
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.work, (unsigned long long)RPW);
        base = __shfl_sync(kAll, base, 0);
        if ((int64_t)base >= a.nrows) break;  // warp-uniform
        const int64_t tix = (int64_t)base + (lane / LPR);
        const bool has = tix < a.nrows;
        const int64_t i64 = has ? (a.rows ? a.rows[tix] : a.row_lo + tix) : 0;
        const int32_t i = (int32_t)i64;
        const int64_t orow = i64 - a.out_base;
        const int64_t e0i = has ? rp_of(a, i64) : 0, e1i = has ? rp_of(a, i64 + 1) : 0;
        tph = clock64();
        for (int sl = gl; sl < H; sl += LPR) {
            w.hkey[sl] = kEmpty;
            w.hval[sl] = (int8_t)-1;  // no stale shared memory is ever decoded
        }
        for (int x = gl; x < CA; x += LPR) w.ahn[x] = 0;
        if (gl == 0) w.dscr[0] = real(0);
        RowBook bk{0, 0, 0, false, 0u};
        G.sync();
        {
            const bool vi = has && gl < (int)(e1i - e0i);
            const int32_t ci = vi ? __ldg(a.col + e0i + gl) : 0;
            const real xi = vi ? __ldg(aval(a) + e0i + gl) : real(0);
            scan_row_hits_ls<LPR, HC>(w, G, H, log2H, i, vi, ci, xi, gl, -1, nullptr, nullptr, bk);
        }
        const real a_ii = w.dscr[0];
        const real psi0 = a_ii;
        real psi = psi0;
        int m = 0, steps = 0, reason = AFSAI_STOP_KMAX, fail_step = 0;
        const bool ovf0 = G.ballot(bk.ovf) != 0;  // full-warp ballot: every lane, before any && short-circuit
        bool fail = false, overflow = has && ovf0;
        bool running = has && !overflow;
        PHASE(0)
        for (int k = 1; k <= a.nsteps; ++k) {
            if (!__any_sync(kAll, running)) break;
            int room = a.s;
            if (a.cap - 1 - m < room) room = a.cap - 1 - m;
            if (running && room <= 0) {
                reason = AFSAI_STOP_CAP;
                running = false;
            }
            // ---- gradient: fold of each active candidate's hits (C3); no shuffles inside
            int nc = 0;
            real ba[GS];
            int32_t bj[GS], bt[GS];
#pragma unroll
            for (int q = 0; q < GS; ++q) { ba[q] = -real(1); bj[q] = 0x7fffffff; bt[q] = -1; }
            if (running) {
                const int hw = bk.hw;
                // two candidate slots per iteration: the hit values of both are
                // loaded before either fold (one L2 wait per two slots) and the two
                // folds interleave; each slot's fold keeps its own hit order (C3).
                // M3 rows kernel 495.6 -> 472.1 ms (a generic k-slot form with the
                // folds one after the other: 508.5 ms at k = 2, 570.5 at k = 3)
                for (int aa = gl; aa < hw; aa += 2 * LPR) {
                    const int ab = aa + LPR;
                    const int n0 = w.ahn[aa], n1 = ab < hw ? w.ahn[ab] : 0;  // 0: a freed slot
                    real v0[HC], v1[HC], u0[HC], u1[HC];
#pragma unroll
                    for (int h = 0; h < HC; ++h) {
                        const bool i0 = h < n0, i1 = h < n1;
                        const int q0 = i0 ? w.ahq[h * CA + aa] : -1;
                        const int q1 = i1 ? w.ahq[h * CA + ab] : -1;
                        u0[h] = q0 < 0 ? real(1) : w.g[q0];
                        u1[h] = q1 < 0 ? real(1) : w.g[q1];
                        const int64_t r0 = q0 < 0 ? e0i : (int64_t)w.prs[q0];
                        const int64_t r1 = q1 < 0 ? e0i : (int64_t)w.prs[q1];
                        v0[h] = i0 ? __ldg(aval(a) + r0 + w.hv[h * CA + aa]) : real(0);
                        v1[h] = i1 ? __ldg(aval(a) + r1 + w.hv[h * CA + ab]) : real(0);
                    }
                    real acc0 = real(0), acc1 = real(0);
#pragma unroll
                    for (int h = 0; h < HC; ++h) {
                        acc0 = h < n0 ? fma(v0[h], u0[h], acc0) : acc0;
                        acc1 = h < n1 ? fma(v1[h], u1[h], acc1) : acc1;
                    }
                    c_gfma += n0 + n1;
                    const bool cand0 = acc0 != real(0), cand1 = acc1 != real(0);
                    nc += cand0 + cand1;
                    topk_insert<GS>(ba, bj, bt, cand0 ? fabs(acc0) : -real(1), cand0 ? w.hkey[w.ahs[aa]] : 0x7fffffff, aa);
                    topk_insert<GS>(ba, bj, bt, cand1 ? fabs(acc1) : -real(1), cand1 ? w.hkey[w.ahs[ab]] : 0x7fffffff, ab);
                }
            }
            // row extents of the lane's local top-GS candidates, loaded now: they
            // arrive during the group argmax, and the winners' are stored by their
            // lanes (one L2 round trip per step less on the row's critical path)
            int64_t rs[GS], re[GS];
#pragma unroll
            for (int q = 0; q < GS; ++q) {
                const bool ok = bt[q] >= 0;
                rs[q] = ok ? rp_of(a, bj[q]) : 0;
                re[q] = ok ? rp_of(a, (int64_t)bj[q] + 1) : 0;
            }
            nc = G.sum(nc);
            PHASE(1)
            if (running && nc == 0) {
                reason = AFSAI_STOP_NOCAND;
                running = false;
            }
            const int nsel = running ? (nc < room ? nc : room) : 0;
            const int nsel_max = warp_max(nsel);
            if (nsel_max == 0) continue;
            // ---- selection: nsel_max (<= GS) rounds of group argmax over the list
            //      heads; every lane keeps the winners (selj) and their ranks in
            //      registers, the winner's lane stores its slot and row extent
            int32_t selj[GS];
            int32_t pc[GS], pe[GS];
            int64_t g0s[GS];
            real pv[GS];
            bool pvld[GS];
#pragma unroll
            for (int u = 0; u < GS; ++u) {
                selj[u] = 0x7fffffff;
                pvld[u] = false;
                pc[u] = 0;
                pv[u] = real(0);
                if (u < nsel_max) {
                    real wa = ba[0];
                    int32_t wj = bj[0];
#pragma unroll
                    for (int o = LPR / 2; o > 0; o >>= 1) {
                        const real oa = G.xorv(wa, o);
                        const int32_t oj = G.xorv(wj, o);
                        if (better(oa, oj, wa, wj)) { wa = oa; wj = oj; }
                    }
                    if (u < nsel) selj[u] = wj;
                    // the winner's row entries are loaded right away (one per lane):
                    // they arrive during the next round and the bookkeeping below
                    const bool won = u < nsel && bj[0] == wj;
                    const unsigned wb = G.ballot(won);
                    const int wl = wb ? __ffs(wb) - 1 : 0;
                    const int64_t g0 = G.bcast(rs[0], wl);
                    const int gn = G.bcast((int)(re[0] - rs[0]), wl);
                    pvld[u] = (u < nsel) && gl < gn;
                    pc[u] = pvld[u] ? __ldg(a.col + g0 + gl) : 0;
                    pe[u] = gl;   // the entry's position within its row
                    g0s[u] = g0;
                    pv[u] = pvld[u] ? __ldg(aval(a) + g0 + gl) : real(0);
                    if (won) {
                        w.sela[u] = bt[0];
#pragma unroll
                        for (int q = 0; q + 1 < GS; ++q) {
                            ba[q] = ba[q + 1]; bj[q] = bj[q + 1]; bt[q] = bt[q + 1];
                            rs[q] = rs[q + 1]; re[q] = re[q + 1];
                        }
                        ba[GS - 1] = -real(1); bj[GS - 1] = 0x7fffffff; bt[GS - 1] = -1;
                    }
                }
            }
            // new columns join P in ascending order: winner u goes to position m + rk[u]
            int rk[GS];
#pragma unroll
            for (int u = 0; u < GS; ++u) {
                rk[u] = 0;
#pragma unroll
                for (int v = 0; v < GS; ++v) rk[u] += (selj[v] < selj[u]);
            }
            // what border reads: the new rows q = m .. m+nsel-1 of L (the gather
            // writes A[P_q, P] there), zeroed by fixed per-lane column tiles
#pragma unroll
            for (int u = 0; u < GS; ++u)
#pragma unroll
                for (int tt = 0; tt < NT; ++tt)
                    if (u < nsel && gl + LPR * tt <= m + u) w.L[tri(m + u) + gl + LPR * tt] = real(0);
            if (gl < nsel) w.brow[gl] = real(0);
            G.sync();
            if (gl < nsel) {
                int32_t j = selj[0];
                int r = rk[0];
                int64_t g0 = g0s[0];
#pragma unroll
                for (int u = 1; u < GS; ++u)
                    if (gl == u) { j = selj[u]; r = rk[u]; g0 = g0s[u]; }
                const int aa = w.sela[gl];
                w.P[m + r] = j;
                w.prs[m + r] = (int32_t)g0;
                w.hval[w.ahs[aa]] = (int8_t)(m + r);
                w.ahn[aa] = 0;
                w.afree[bk.nf + gl] = (int16_t)aa;
            }
            bk.nf += nsel;
            G.sync();
            PHASE(2)
            // ---- gather: new rows (one entry per lane, loaded during the selection)
            for (int ug = 0; ug < nsel_max; ug += GS) {  // nsel_max <= GS: one pass
#pragma unroll
                for (int u = 0; u < GS; ++u)
                    if (ug + u < nsel_max) {  // winner u (selection order) is pattern position m + rk[u]
                        const int r = rk[u] < GS ? rk[u] : 0;
                        scan_row_hits_ls<LPR, HC>(w, G, H, log2H, i, pvld[u], pc[u], pv[u], pe[u], m + r,
                                                  w.L + tri(m + r), w.brow + r, bk);
                    }
            }
            PHASE(3)
            const bool ovf_any = G.ballot(bk.ovf) != 0;
            if (running && (ovf_any || bk.nkeys * 4 > H * 3)) {
                if (bk.nkeys * 4 > H * 3) bk.why |= 1u;
                overflow = true;
                running = false;
            }
            // ---- bordered Cholesky of the new rows, groups of GS rows
            for (int ug = 0; ug < nsel_max; ug += GS) {
                int gs = running ? nsel - ug : 0;
                gs = gs < 0 ? 0 : (gs > GS ? GS : gs);
                const bool act = gs > 0;
                const int qf_max = warp_max(act ? m + ug : 0);
                if (!border_group_ls<LPR, NT, GS>(w, G, act, m + ug, gs, ug, qf_max, psi)) {
                    fail = true;
                    fail_step = k;
                    running = false;
                }
            }
            if (running) {
                for (int u = 0; u < nsel; ++u) {
                    const long q = m + u;
                    c_border += (unsigned long long)(q * (q - 1) / 2 + 2 * q + 1);
                }
                m += nsel;
                if (!(psi > real(0))) {
                    fail = true;
                    fail_step = k;
                    running = false;
                }
            }
            PHASE(4)
            // ---- back-substitution
            const int m_max = warp_max(running ? m : 0);
            back_substitute_ls<LPR, NT>(w, G, running, m, m_max);
            if (running) {
                c_back += (unsigned long long)(m * (m - 1) / 2);
                steps = k;
                if (psi / psi0 <= a.eps) {
                    reason = AFSAI_STOP_TOL;
                    running = false;
                }
            }
            PHASE(5)
        }
        // ---- per-row outcome (no shuffles below until the final sync)
        const unsigned whyw = __reduce_or_sync(kAll, overflow ? bk.why : 0u);  // both rows' reasons
        if (has) {
            if (overflow) {
                if (gl == 0) {
                    atomicOr(&a.counters[20], (unsigned long long)whyw);  // the host's table sizing
                    const int p = atomicAdd(a.retry_count, 1);
                    a.retry_rows[p] = i64;
                }
            } else if (fail) {
                if (gl == 0) {
                    const unsigned long long code = ((unsigned long long)i64 << 24) |
                                                    ((unsigned long long)(fail_step & 0xfffff) << 4) |
                                                    (unsigned long long)AFSAI_ENOTSPD;
                    atomicMin(a.err, code);
                    a.nnz_row[orow] = 0;
                }
            } else {
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
                    c_univ = max(c_univ, (unsigned long long)bk.nkeys);
                }
            }
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

// kernel instance with GS new rows per bordering group (one translation unit per
// GS: setup_lockstep_g{1..4}.cu)
template <int GS>
SetupKernFn ls_instance(int lpr, int nt, int hc) {
#define AFSAI_LS_NT(L, H)                                                 \
    switch (nt) {                                                         \
        case 1: return afsai_setup_rows_lockstep_kernel<L, 1, GS, H>;     \
        case 2: return afsai_setup_rows_lockstep_kernel<L, 2, GS, H>;     \
        case 3: return afsai_setup_rows_lockstep_kernel<L, 3, GS, H>;     \
        case 4: return afsai_setup_rows_lockstep_kernel<L, 4, GS, H>;     \
        case 5: return afsai_setup_rows_lockstep_kernel<L, 5, GS, H>;     \
        default: return afsai_setup_rows_lockstep_kernel<L, 6, GS, H>;    \
    }
    if (lpr == 8) {
        if (hc <= 6) { AFSAI_LS_NT(8, 6) } else { AFSAI_LS_NT(8, 8) }
    }
    if (hc <= 6) { AFSAI_LS_NT(16, 6) } else { AFSAI_LS_NT(16, 8) }
#undef AFSAI_LS_NT
}

}  // namespace AFSAI_PNS
}  // namespace afsai
