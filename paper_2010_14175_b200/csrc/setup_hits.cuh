// setup_hits.cuh -- per-row state of the hit-list set-up kernels (setup_hits.cu,
// setup_lockstep.cu).
#pragma once
#include "setup_common.cuh"

namespace afsai {
namespace AFSAI_PNS {

// A recorded hit (candidate j, pattern row r = P_q) is the position of the entry
// (r, j) within row r (rows of the hit-list plans hold <= 16 entries: one int8),
// not the value a_jr: with the start of each pattern row kept once per position
// (prs[q], int32; row i's start is a register) the gradient re-reads the value
// (an L1/L2 hit, the same bits) -- 1 byte per hit instead of 8, so more rows fit
// in shared memory.  Needs nnz(A_ext) < 2^31 (run_rows).
typedef int8_t hit_t;
#define AFSAI_HIT(v, off) ((int8_t)(off))

struct HitState {
    real *inv, *y, *g, *L, *arow, *brow, *dscr, *acc;
    hit_t *hv;
    int64_t *gstart;
    int32_t *hkey, *P, *sel, *sela, *glen, *misc, *akey, *prs;
    int16_t *ahs, *afree;
    int8_t *hval, *ahn, *ahq;
    int M, CA;
};

// compact (the lockstep kernel): no inv[] (1/L[k][k] lives in L's unused diagonal
// slot), no akey[] (a candidate's column is hkey[ahs[a]]) and no arow[] (a new
// row's gathered A[P, P_q] is written straight into its own, still empty, row q of
// L, the diagonal a_qq into the diagonal slot): (2 + S) M doubles and CA ints less
// per row
template <int HC>
__host__ __device__ inline int64_t hit_state_bytes(int H, int M, int S, int CA, bool acc, bool compact = false) {
    int64_t dbl = (compact ? 2 : 3) * (int64_t)M + (M * (M + 1)) / 2 + 1 + (compact ? 0 : (int64_t)S * M) + S + 2 +
                  (acc ? CA : 0);
    int64_t i64 = S;
    int64_t i32 = (int64_t)H + M + 3 * S + 8 + (compact ? 0 : (int64_t)CA) + M;  // ... akey, prs
    int64_t i16 = 2 * (int64_t)CA;
    int64_t i8 = (int64_t)H + CA + 2 * (int64_t)CA * HC;  // hval, ahn, ahq, hv
    int64_t b = real_bytes(dbl) + i64 * 8 + i32 * 4 + i16 * 2 + i8;
    return (b + 15) & ~int64_t(15);
}

template <int HC>
__device__ __forceinline__ HitState carve_hits(char *base, const SetupKArgs &a, bool acc, bool compact = false) {
    HitState w;
    const int H = a.H, M = a.mmax, S = a.s, CA = a.cact;
    w.M = M;
    w.CA = CA;
    real *d = reinterpret_cast<real *>(base);
    // g first: the lockstep fast paths prefetch inv[-1] / y[-1] (unused values) and
    // read up to 31 doubles past the end of L (into arow), all inside the row's region
    w.g = d; d += M;
    w.inv = nullptr;
    if (!compact) { w.inv = d; d += M; }
    w.y = d; d += M;
    w.L = d; d += (M * (M + 1)) / 2 + 1;
    w.arow = nullptr;
    if (!compact) { w.arow = d; d += S * M; }
    w.brow = d; d += S;
    w.dscr = d; d += 2;
    w.acc = nullptr;
    if (acc) { w.acc = d; d += CA; }
    int64_t *l8 = reinterpret_cast<int64_t *>(base + real_bytes(d - reinterpret_cast<real *>(base)));
    w.gstart = l8; l8 += S;
    int32_t *ip = reinterpret_cast<int32_t *>(l8);
    w.hkey = ip; ip += H;
    w.P = ip; ip += M;
    w.sel = ip; ip += S;
    w.sela = ip; ip += S;
    w.glen = ip; ip += S;
    w.misc = ip; ip += 8;
    w.akey = nullptr;
    if (!compact) { w.akey = ip; ip += CA; }
    w.prs = ip; ip += M;
    int16_t *sp = reinterpret_cast<int16_t *>(ip);
    w.ahs = sp; sp += CA;
    w.afree = sp; sp += CA;
    int8_t *bp = reinterpret_cast<int8_t *>(sp);
    w.hval = bp; bp += H;
    w.ahn = bp; bp += CA;
    w.ahq = bp; bp += CA * HC;  // [h][a]
    w.hv = bp;                  // [h][a]
    return w;
}

// misc: [0] keys inserted  [1] overflow  [2] active high-water  [3] free-stack size

// Insert the hit (column r at pattern position q, value v) into active slot aa,
// keeping the list sorted by r; q = -1 stands for r = i (always last).
template <int HC>
__device__ __forceinline__ void hit_insert(const HitState &w, int aa, int q, int32_t r, hit_t v) {
    const int CA = w.CA;
    int n = w.ahn[aa];
    if (n >= HC) {
        w.misc[1] = 1;
        return;
    }
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
}

}  // namespace AFSAI_PNS
}  // namespace afsai
