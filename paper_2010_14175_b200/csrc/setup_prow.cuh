// setup_prow.cuh -- the per-row set-up for long rows of A (FE matrices):
// the Kaporin gradient is folded over the PATTERN rows instead of the
// candidate rows.
//
// Eq. 15 needs, for every candidate j, the fold over
// r in P U {i} of a_jr g~_r in the storage order of row j (ascending r,
// DESIGN.md C3).  Rows of A are bitwise symmetric (C1), so a_jr has the same
// bits as a_rj, the entry of pattern row r at column j.  Visiting the pattern
// rows in ascending column order and folding each of their entries j < i into
// acc[j] therefore applies exactly the same fma sequence to every acc[j] as the
// candidate-row scan, while touching only |P|+1 rows of A per step instead of
// one row per candidate (FE: ~45 pattern rows vs ~500 candidates).
//
// Per row (one group of LPR lanes), in shared memory:
//   hash table hkey[H] (column -> slot), hval[H] (kCand or pattern position),
//   acc[H] indexed by slot, ulist (the occupied slots, in insertion order), L;
// in a per-warp region of global memory: for each pattern row (and row i) the
//   slots of its entries below column i (lu, filled once when the row joins P),
//   so the gradient needs no hash lookups; the values themselves are re-read from
//   L2, fetched into registers in batches of pattern rows (setup_prow_impl.cuh).
#pragma once
#include "setup_common.cuh"

namespace afsai {
namespace AFSAI_PNS {

struct PRowState {
    real *inv, *y, *g, *L, *arow, *brow, *dscr, *acc;
    int4 *pd;         // [M+1] row descriptors in ascending column order (prow_fetch)
    int64_t *rstart;  // [M] first entry of pattern row q, relative to A's base
    int64_t *rend;    // [S] end entry of the rows selected this step
    int64_t *srs, *sre;  // [S] row extents of the winners, by selection round
    int32_t *hkey, *P, *sel, *selt, *misc, *lofs;  // lofs [M]
    int16_t *lu;      // [LC]: slot of each entry below column i of the pattern rows (global memory)
    int16_t *ulist;   // [H]: the occupied table slots in insertion order (the universe)
    int8_t *hval;
    int M;
};

__host__ __device__ inline int64_t prow_state_bytes(int H, int M, int S, int LC) {
    int64_t dbl = 3 * (int64_t)M + 1 + (int64_t)(M * (M + 1)) / 2 + 1 + (int64_t)S * M + S + 2 + H + 1;
    int64_t i128 = M + 1;
    int64_t i64 = M + 3 * S;
    int64_t i32 = (int64_t)H + M + 2 * S + 4 + M;
    // the lu lists live in global memory (one region per warp, L1/L2-resident; their
    // loads ride with the batched value loads): 67 -> 52 KB per FE row, 4 rows per SM
    int64_t i16 = H;  // ulist
    (void)LC;
    int64_t i8 = H;
    int64_t b = real_bytes(dbl) + 8 /* int4 alignment */ + i128 * 16 + i64 * 8 + i32 * 4 + i16 * 2 + i8;
    return (b + 15) & ~int64_t(15);
}

__device__ __forceinline__ PRowState carve_prow(char *base, const SetupKArgs &a) {
    PRowState w;
    const int H = a.H, M = a.mmax, S = a.s;
    w.M = M;
    real *d = reinterpret_cast<real *>(base);
    w.inv = d; d += M;
    w.y = d; d += M;
    w.g = d; d += M + 1;  // g[M] = 1: row i in the gradient
    w.L = d; d += (M * (M + 1)) / 2 + 1;
    w.arow = d; d += S * M;
    w.brow = d; d += S;
    w.dscr = d; d += 2;
    w.acc = d; d += H + 1;  // slot H: spare target of the branch-free gradient fold
    w.pd = reinterpret_cast<int4 *>(base + (((reinterpret_cast<char *>(d) - base) + 15) & ~15));
    int64_t *l8 = reinterpret_cast<int64_t *>(w.pd + M + 1);
    w.rstart = l8; l8 += M;
    w.rend = l8; l8 += S;
    w.srs = l8; l8 += S;
    w.sre = l8; l8 += S;
    int32_t *ip = reinterpret_cast<int32_t *>(l8);
    w.hkey = ip; ip += H;
    w.P = ip; ip += M;
    w.sel = ip; ip += S;
    w.selt = ip; ip += S;
    w.misc = ip; ip += 4;
    w.lofs = ip; ip += M;
    int16_t *sp = reinterpret_cast<int16_t *>(ip);
    w.lu = a.lu_global + (int64_t)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * a.lcap;
    w.ulist = sp; sp += H;
    w.hval = reinterpret_cast<int8_t *>(sp);
    return w;
}

}  // namespace AFSAI_PNS
}  // namespace afsai
