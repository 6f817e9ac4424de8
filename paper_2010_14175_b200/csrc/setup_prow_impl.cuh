// setup_prow_impl.cuh -- kernel body of the pattern-row set-up (see
// setup_prow.cuh), instantiated per group size by setup_prow_g*.cu so the
// instances compile in parallel.  Compiled with -fmad=false (C12).
#pragma once
#include <climits>

#include "setup_prow.cuh"

namespace afsai {
namespace AFSAI_PNS {

#ifndef AFSAI_PROW_BATCH
#define AFSAI_PROW_BATCH 10
#endif
// pattern rows fetched per batch in the gradient.  The value and slot loads come
// from L2 (~1.5k cycles under load, two dies); every load in flight shares one
// scoreboard, so the loads of a batch are issued together and waited on once
// (a rolling prefetch, 6-12 rows deep, waited for its newest load at every row:
// M4 2.04 s; batches of 10: 1.75 s; two alternating batches of 6: 2.01 s;
// DESIGN.md §4.1).  Registers cap the batch (11 per row; 12 rows: 254).
constexpr int kProwBatch = AFSAI_PROW_BATCH;
constexpr int kProwGather = 8;  // entries per lane loaded per gather batch
// L[q][k] broadcast through shared memory in the bordering sweep (owner store,
// __syncwarp, every lane loads) instead of 64-bit shuffles: M4 border phase
// 351 -> 325 ms.  (The same for g~[k] in the back-substitution: 154 -> 180 ms, so
// that one keeps the shuffle.)
#ifdef AFSAI_PROW_BCAST_SHFL
constexpr bool kProwSmemBcast = false;
#else
constexpr bool kProwSmemBcast = true;
#endif

// Insert-if-absent of one key per lane (lanes with !valid idle).  The probe loop
// is controlled by a warp vote and its body is structured, so the warp leaves it
// converged: divergent exits here would leave the warp split for the rest of the
// row and send every later shuffle through its divergent slow path.
// Returns the slot (-1: table full); *ins = newly inserted.
__device__ __forceinline__ int hinsert_warp(int32_t *hkey, int H, int log2H, bool valid, int32_t key, bool *ins) {
    const uint32_t msk = (uint32_t)H - 1u;
    uint32_t sl = hslot(key, log2H);
    int res = -1, pr = 0;
    bool done = !valid, fresh = false;
    while (__any_sync(0xffffffffu, !done)) {
        if (!done) {
            const int32_t k = hkey[sl];
            bool hit = k == key, taken = false;
            if (k == kEmpty) {
                const int32_t old = atomicCAS(&hkey[sl], kEmpty, key);
                taken = old == kEmpty;
                hit = old == key;
            }
            if (hit || taken) {
                res = (int)sl;
                fresh = taken;
                done = true;
            } else {
                sl = (sl + 1u) & msk;
                done = ++pr >= H;
            }
        }
    }
    *ins = fresh;
    return res;
}

// append the slots this call inserted (ins) to ulist, in lane order; ucnt is
// group-uniform
__device__ __forceinline__ void ulist_append(const PRowState &w, int gl, bool ins, int sl, int &ucnt) {
    const unsigned bal = __ballot_sync(0xffffffffu, ins);
    if (ins) w.ulist[ucnt + __popc(bal & ((1u << gl) - 1u))] = (int16_t)sl;
    ucnt += __popc(bal);
}

// registers of one fetched pattern row: its entries x = gl + LPR*v below
// column i (slot, value) and g~ of the row
template <int NV>
struct PRowFetch {
    real v[NV];
    int s[NV];  // acc slot (H: the spare slot)
    real gq;
};

// One pattern row from its descriptor pd[idx] = {first entry - e0i, list offset,
// (count << 16) | position q, column}; the rows are kept in ascending column
// order with row i (position M, g~_i = g[M] = 1) last.
// Branch-free: rows past m read row m's descriptor with no entries.  Lanes
// without an entry fold 0 into the spare slot acc[H].
template <int LPR, int NV>
__device__ __forceinline__ void prow_fetch(const PRowState &w, const real *vrow, int spare, int idx, int m,
                                           int gl, PRowFetch<NV> &f) {
    const bool live = idx <= m;
    const int4 d = w.pd[live ? idx : m];
    const int q = d.z & 0xffff, n = live ? (d.z >> 16) : 0;
    f.gq = w.g[q];
    const real *vb = vrow + d.x;
    const int16_t *lb = w.lu + d.y;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int x = gl + LPR * v;
        const bool in = x < n;
        f.s[v] = in ? (int)lb[x] : spare;
        f.v[v] = in ? __ldg(vb + x) : real(0);
    }
}

// fold one fetched pattern row into acc: lanes without an entry fold 0 into the
// spare slot.  A lane's slots within one row are distinct columns: all loads,
// then all fmas, then all stores (one LDS -> DFMA -> STS chain per row).
template <int NV>
__device__ __forceinline__ void prow_fold(const PRowState &w, const PRowFetch<NV> &f) {
    real av[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) av[v] = w.acc[f.s[v]];
#pragma unroll
    for (int v = 0; v < NV; ++v) av[v] = fma(f.v[v], f.gq, av[v]);
#pragma unroll
    for (int v = 0; v < NV; ++v) w.acc[f.s[v]] = av[v];
}

template <int LPR, int NT, int GS, int NV>
__global__ void __launch_bounds__(128) afsai_setup_rows_prow_kernel(SetupKArgs a) {
    extern __shared__ __align__(16) char smem[];
    const int lane = threadIdx.x & 31;
    const Group<LPR> G(lane);
    const int gl = G.gl;
    PRowState w = carve_prow(smem + (size_t)(threadIdx.x / LPR) * a.warp_smem, a);
    const int H = a.H, log2H = a.log2H, M = w.M;
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
        // ---- prologue: empty table; universe = columns j < i of row i (its slots
        //      form the list of row i, slot M); a_ii
        for (int sl = gl; sl < H; sl += LPR) {
            w.hkey[sl] = kEmpty;
            w.hval[sl] = kCand;
        }
        if (gl == 0) {
            w.misc[0] = 0;  // keys inserted
            w.misc[1] = 0;  // overflow
            w.g[M] = real(1);   // g~_i
        }
        G.sync();
        int ucnt = 0;  // occupied slots = length of ulist (group-uniform)
        {
            bool full = false;
            for (int64_t e0 = e0i; e0 < e1i; e0 += LPR) {  // warp-uniform trip count
                const int64_t e = e0 + gl;
                const bool in = e < e1i;
                const int32_t c = in ? __ldg(a.col + e) : INT_MAX;
                const real v = in ? __ldg(aval(a) + e) : real(0);
                if (c == i) {
                    w.dscr[0] = v;
                    // row i's descriptor: entries below the diagonal
                    w.pd[0] = make_int4(0, 0, ((int)(e - e0i) << 16) | M, i);
                }
                bool ins;
                const int sl = hinsert_warp(w.hkey, H, log2H, c < i, c, &ins);
                if (c < i && sl >= 0) w.lu[e - e0i] = (int16_t)sl;
                ulist_append(w, gl, ins, sl, ucnt);
                full |= __any_sync(0xffffffffu, c < i && sl < 0);
            }
            if (gl == 0) {
                w.misc[0] = ucnt;
                w.misc[1] = full ? 1 : 0;
            }
        }
        G.sync();
        const real a_ii = w.dscr[0];
        const real psi0 = a_ii;
        real psi = psi0;
        int m = 0, steps = 0, reason = AFSAI_STOP_KMAX;
        bool fail = false, overflow = (w.misc[1] != 0) || w.misc[0] * 4 > H * 3;
        int fail_code = 0, fail_step = 0;
        int lused = w.pd[0].z >> 16;  // list entries in use (group-uniform)
        int gsum = lused;             // gradient fmas per step: entries below i of P's rows and row i
        PHASE(0)

        for (int k = 1; k <= a.nsteps && !overflow; ++k) {
            int room = a.s;
            if (a.cap - 1 - m < room) room = a.cap - 1 - m;
            if (room <= 0) { reason = AFSAI_STOP_CAP; break; }

            // ---- phase G: gradient (C3) over the pattern rows in ascending column
            //      order, then row i; every acc[slot] sees the fma sequence of the
            //      storage order of its own row (bitwise symmetry, C1)
            for (int x = gl; x < ucnt; x += LPR) w.acc[w.ulist[x]] = real(0);
            G.sync();
            {
                // batches of kProwBatch pattern rows: all their loads are issued
                // together and waited on once (the load scoreboard is shared by
                // every load in flight, so a rolling prefetch would wait for the
                // newest load at every row)
                const real *vrow = aval(a) + e0i;
                const int spare = H;
                for (int base = 0; base <= m; base += kProwBatch) {
                    PRowFetch<NV> pf[kProwBatch];
#pragma unroll
                    for (int d = 0; d < kProwBatch; ++d) prow_fetch<LPR, NV>(w, vrow, spare, base + d, m, gl, pf[d]);
#pragma unroll
                    for (int d = 0; d < kProwBatch; ++d) {
                        if (base + d <= m) {
                            prow_fold<NV>(w, pf[d]);
                            G.sync();
                        }
                    }
                }
            }
            c_gfma += (unsigned long long)gsum;
#ifdef AFSAI_PROW_DIAG
            PHASE(0)  // diagnostics build: the fold goes to slot 0, the candidate scan stays in slot 1
#endif
            // candidates: keys not in P with acc != 0; per-lane top-GS lists
            int nc = 0;
            real ba[GS];
            int32_t bj[GS], bt[GS];
#pragma unroll
            for (int q = 0; q < GS; ++q) { ba[q] = -real(1); bj[q] = INT_MAX; bt[q] = -1; }
            // over the occupied slots only (ulist: about half of the table)
            for (int x0 = 0; x0 < ucnt; x0 += LPR) {
                const bool in = x0 + gl < ucnt;
                const int sl = in ? w.ulist[x0 + gl] : 0;
                const int32_t key = w.hkey[sl];
                const real acc = w.acc[sl];
                const bool cand = in && w.hval[sl] == kCand && acc != real(0);
                nc += cand;
                real ca = cand ? fabs(acc) : -real(1);
                int32_t cj = cand ? key : INT_MAX, ct = sl;
                topk_insert<GS>(ba, bj, bt, ca, cj, ct);
            }
            // row extents of the lane's local top-GS candidates, loaded now: they
            // arrive during the group argmax; the winners' are stored by their lanes
            int64_t rs[GS], re[GS];
#pragma unroll
            for (int q = 0; q < GS; ++q) {
                const bool ok = bt[q] >= 0;
                rs[q] = ok ? rp_of(a, bj[q]) : 0;
                re[q] = ok ? rp_of(a, (int64_t)bj[q] + 1) : 0;
            }
            nc = G.sum(nc);
            PHASE(1)
            if (nc == 0) { reason = AFSAI_STOP_NOCAND; break; }
            const int nsel = nc < room ? nc : room;

            // ---- phase S: top-nsel under (|acc| desc, j asc)
            for (int u = 0; u < nsel; ++u) {
                real wa = ba[0];
                int32_t wj = bj[0];
#pragma unroll
                for (int o = LPR / 2; o > 0; o >>= 1) {
                    const real oa = G.xorv(wa, o);
                    const int32_t oj = G.xorv(wj, o);
                    if (better(oa, oj, wa, wj)) { wa = oa; wj = oj; }
                }
                const bool me = bj[0] == wj;  // unique column: exactly one lane
                if (me) {
                    w.sel[u] = wj;
                    w.selt[u] = bt[0];
                    w.srs[u] = rs[0];
                    w.sre[u] = re[0];
                }
#pragma unroll
                for (int q = 0; q + 1 < GS; ++q) {
                    ba[q] = me ? ba[q + 1] : ba[q];
                    bj[q] = me ? bj[q + 1] : bj[q];
                    bt[q] = me ? bt[q + 1] : bt[q];
                    rs[q] = me ? rs[q + 1] : rs[q];
                    re[q] = me ? re[q + 1] : re[q];
                }
                ba[GS - 1] = me ? -real(1) : ba[GS - 1];
                bj[GS - 1] = me ? INT_MAX : bj[GS - 1];
                bt[GS - 1] = me ? -1 : bt[GS - 1];
            }
            G.sync();
            // append in ascending column order (R9); merge the new positions into
            // ord (pattern positions by ascending column)
            int newpos = -1, newq = -1;
            {
                const bool mine = gl < nsel;
                const int32_t j = w.sel[mine ? gl : 0];
                int rank = 0;
                for (int u = 0; u < nsel; ++u) rank += (w.sel[u] < j);
                const int q = m + rank;
                const int64_t rs = w.srs[mine ? gl : 0], re = w.sre[mine ? gl : 0];
                if (mine) {
                    w.P[q] = j;
                    w.hval[w.selt[gl]] = (int8_t)q;
                    w.rstart[q] = rs;
                    w.rend[rank] = re;
                }
                // old columns below j: binary search with a fixed trip count (m < 2^8)
                int lo = 0, hi = m;
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int mid = (lo + hi) >> 1;
                    const bool go = lo < hi;
                    const bool lt = go && w.pd[go ? mid : 0].w < j;
                    lo = lt ? mid + 1 : lo;
                    hi = (go && !lt) ? mid : hi;
                }
                newpos = mine ? lo + rank : -1;
                newq = q;
            }
            // old descriptors (and row i's, at m) move up by the new columns below them
            int4 oval[NT + 1];
            int opos[NT + 1];
#pragma unroll
            for (int tt = 0; tt <= NT; ++tt) {
                const int x = gl + LPR * tt;
                opos[tt] = -1;
                oval[tt] = make_int4(0, 0, 0, 0);
                if (x <= m) {
                    const int4 d = w.pd[x];
                    int sh = 0;
                    for (int u = 0; u < nsel; ++u) sh += (w.sel[u] < d.w);
                    oval[tt] = d;
                    opos[tt] = x + sh;
                }
            }
            G.sync();
#pragma unroll
            for (int tt = 0; tt <= NT; ++tt)
                if (opos[tt] >= 0) w.pd[opos[tt]] = oval[tt];
            for (int x = gl; x < nsel * M; x += LPR) w.arow[x] = real(0);
            if (gl < nsel) w.brow[gl] = real(0);
            G.sync();
            // list offsets of the new rows (full row lengths reserved)
            int total = 0;
            for (int u = 0; u < nsel; ++u) {
                const int len = (int)(w.rend[u] - w.rstart[m + u]);
                if (gl == 0) w.lofs[m + u] = lused + total;
                total += len;
            }
            if (lused + total > a.lcap) { overflow = true; break; }
            lused += total;
            G.sync();
            PHASE(2)

            // ---- phase A: gather the new rows P_q of A (Eq. 7):
            //      A[P,P] row entries, A[P,i], their list slots; universe grows (R7)
            {
                // row u of entry t: t in [pre[u], pre[u+1]) (nsel <= GS <= 4 rows)
                int pre[4];
                int64_t rb[4];
                int lo4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool in = u < nsel;
                    rb[u] = in ? w.rstart[m + u] : 0;
                    lo4[u] = in ? w.lofs[m + u] : 0;
                }
                {
                    int acc_ = 0;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        acc_ += u < nsel ? (int)(w.rend[u] - rb[u]) : 0;
                        pre[u] = acc_;  // end of row u
                    }
                }
                int nlow[4] = {0, 0, 0, 0};
                bool full = false;
                for (int t0 = 0; t0 < total; t0 += LPR * kProwGather) {
                    int32_t cc[kProwGather];
                    real vv[kProwGather];
                    int uu[kProwGather], oo[kProwGather];
#pragma unroll
                    for (int b = 0; b < kProwGather; ++b) {
                        const int t = t0 + gl + LPR * b;
                        const bool in = t < total;
                        const int u = (t >= pre[0]) + (t >= pre[1]) + (t >= pre[2]);
                        const int st = u == 0 ? 0 : (u == 1 ? pre[0] : (u == 2 ? pre[1] : pre[2]));
                        const int64_t rbu = u == 0 ? rb[0] : (u == 1 ? rb[1] : (u == 2 ? rb[2] : rb[3]));
                        const int off = t - st;
                        const int64_t e = rbu + off;
                        cc[b] = in ? __ldg(a.col + e) : INT_MAX;
                        vv[b] = in ? __ldg(aval(a) + e) : real(0);
                        uu[b] = in ? u : 0;
                        oo[b] = off;
                    }
#pragma unroll
                    for (int b = 0; b < kProwGather; ++b) {
                        const int32_t c = cc[b];
                        const int u = uu[b];
                        if (c == i) w.brow[u] = vv[b];
                        const bool low = c < i;
                        bool ins;
                        const int sl = hinsert_warp(w.hkey, H, log2H, low, c, &ins);
                        const bool ok = low && sl >= 0;
                        const int lo_u = u == 0 ? lo4[0] : (u == 1 ? lo4[1] : (u == 2 ? lo4[2] : lo4[3]));
                        if (ok) w.lu[lo_u + oo[b]] = (int16_t)sl;
                        const int st = ok ? (int)w.hval[sl] : -1;
                        if (st >= 0 && st <= m + u) w.arow[u * M + st] = vv[b];
                        ulist_append(w, gl, ins, sl, ucnt);
                        // lane-local counts, reduced once after the gather
                        full |= low && sl < 0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) nlow[q] += (ok && u == q);
                    }
                }
                full = __any_sync(0xffffffffu, full);
#pragma unroll
                for (int q = 0; q < 4; ++q) nlow[q] = q < nsel ? G.sum(nlow[q]) : 0;
                gsum += nlow[0] + nlow[1] + nlow[2] + nlow[3];
                if (gl == 0) {
                    w.misc[0] = ucnt;
                    if (full) w.misc[1] = 1;
                }
                // descriptors of the new rows at their sorted positions
                if (newpos >= 0) {
                    const int u = newq - m;
                    const int cu = u == 0 ? nlow[0] : (u == 1 ? nlow[1] : (u == 2 ? nlow[2] : nlow[3]));
                    const int lu_ = u == 0 ? lo4[0] : (u == 1 ? lo4[1] : (u == 2 ? lo4[2] : lo4[3]));
                    const int64_t rbu = u == 0 ? rb[0] : (u == 1 ? rb[1] : (u == 2 ? rb[2] : rb[3]));
                    w.pd[newpos] = make_int4((int)(rbu - e0i), lu_, (cu << 16) | newq, w.P[newq]);
                }
            }
            G.sync();
            PHASE(3)
            if (w.misc[1] != 0 || w.misc[0] * 4 > H * 3) { overflow = true; break; }

            // ---- phase B: bordered Cholesky of the new rows (C5-C6)
            for (int ug = 0; ug < nsel && !fail; ug += GS) {
                const int gs = (nsel - ug) < GS ? (nsel - ug) : GS;
                if (!border_group<LPR, NT, GS, kProwSmemBcast>(w, G, m + ug, gs, ug, psi)) {
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

            // ---- phase U: back-substitution (C7)
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
        // ---- output: d = psi^-1/2 (Eqs. 8-9); the row sorted by column (C9) is
        //      the ord permutation
        const real d = real(1) / sqrt(psi);
        int32_t *oc = a.scol + orow * a.stride;
        double *ov = a.sval + orow * a.stride;
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) {
            const int x = gl + LPR * tt;
            if (x < m) {
                const int4 pdx = w.pd[x];
                oc[x] = pdx.w;
                ov[x] = w.g[pdx.z & 0xffff] * d;
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
    const unsigned long long g1 = c_gfma;  // group-uniform; added once by lane 0
    if (gl == 0) {
        atomicAdd(&a.counters[0], c_steps);
        atomicAdd(&a.counters[1], c_border);
        atomicAdd(&a.counters[2], c_back);
        atomicAdd(&a.counters[3], g1);
        atomicAdd(&a.counters[4], g1);
        atomicAdd(&a.counters[5], c_r0);
        atomicAdd(&a.counters[6], c_r1);
        atomicAdd(&a.counters[7], c_r2);
        atomicAdd(&a.counters[8], c_r3);
#pragma unroll
        for (int k = 0; k < 7; ++k) atomicAdd(&a.counters[9 + k], (unsigned long long)ph[k]);
        atomicMax(&a.counters[16], c_univ);
    }
}

template <int GS>
SetupKernFn prow_instance(int nt, int nv) {
#define AFSAI_PROW_NV(NT_)                                               \
    switch (nv) {                                                        \
        case 1: return afsai_setup_rows_prow_kernel<32, NT_, GS, 1>;     \
        case 2: return afsai_setup_rows_prow_kernel<32, NT_, GS, 2>;     \
        case 3: return afsai_setup_rows_prow_kernel<32, NT_, GS, 3>;     \
        default: return afsai_setup_rows_prow_kernel<32, NT_, GS, 4>;    \
    }
    switch (nt) {
        case 1: AFSAI_PROW_NV(1)
        case 2: AFSAI_PROW_NV(2)
        case 3: AFSAI_PROW_NV(3)
        default: AFSAI_PROW_NV(4)
    }
#undef AFSAI_PROW_NV
}

}  // namespace AFSAI_PNS
}  // namespace afsai
