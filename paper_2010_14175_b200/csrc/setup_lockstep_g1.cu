// setup_lockstep_g1.cu -- lockstep hit-list kernel instances with one new row per
// bordering group, and the dispatcher over all instances (setup_lockstep_g*.cu).
#include "setup_lockstep_impl.cuh"

namespace afsai {
namespace AFSAI_PNS {
template SetupKernFn ls_instance<1>(int lpr, int nt, int hc);
extern template SetupKernFn ls_instance<2>(int lpr, int nt, int hc);
extern template SetupKernFn ls_instance<3>(int lpr, int nt, int hc);
extern template SetupKernFn ls_instance<4>(int lpr, int nt, int hc);

// lpr (8 or 16) lanes per row, 32/lpr rows per warp; rows <= lpr entries,
// s <= 4, mmax <= 6 * lpr
SetupKernFn lockstep_kernel_for(int lpr, int mmax, int s, int hc) {
    if (s > kMaxGroup || s < 1 || mmax > 6 * lpr) return nullptr;
    const int m = mmax < 1 ? 1 : mmax;
    const int nt = (m + lpr - 1) / lpr;
    lpr = lpr == 8 ? 8 : 16;
    switch (s) {
        case 1: return ls_instance<1>(lpr, nt, hc);
        case 2: return ls_instance<2>(lpr, nt, hc);
        case 3: return ls_instance<3>(lpr, nt, hc);
        default: return ls_instance<4>(lpr, nt, hc);
    }
}

int64_t lockstep_row_bytes(int H, int mmax, int s, int cact, int hc) {
    return hc <= 6 ? hit_state_bytes<6>(H, mmax, s, cact, false, true) : hit_state_bytes<8>(H, mmax, s, cact, false, true);
}
}  // namespace AFSAI_PNS
}  // namespace afsai
