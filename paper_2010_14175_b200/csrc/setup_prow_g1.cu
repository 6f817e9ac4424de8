// setup_prow_g1.cu -- pattern-row set-up kernel instances with one new column
// per step, and the dispatcher over all instances (setup_prow_g*.cu).
#include "setup_prow_impl.cuh"

namespace afsai {
namespace AFSAI_PNS {
template SetupKernFn prow_instance<1>(int nt, int nv);
extern template SetupKernFn prow_instance<2>(int nt, int nv);
extern template SetupKernFn prow_instance<3>(int nt, int nv);
extern template SetupKernFn prow_instance<4>(int nt, int nv);

SetupKernFn prow_kernel_for(int mmax, int s, int64_t max_row_len) {
    const int nt = (mmax < 1 ? 1 : mmax + 31) / 32;
    const int nv = (int)((max_row_len + 31) / 32);
    if (nt > 4 || nv > 4 || s < 1 || s > 4) return nullptr;
    switch (s) {
        case 1: return prow_instance<1>(nt, nv < 1 ? 1 : nv);
        case 2: return prow_instance<2>(nt, nv < 1 ? 1 : nv);
        case 3: return prow_instance<3>(nt, nv < 1 ? 1 : nv);
        default: return prow_instance<4>(nt, nv < 1 ? 1 : nv);
    }
}

int64_t prow_row_bytes(int H, int mmax, int s, int lcap) { return prow_state_bytes(H, mmax, s, lcap); }
}  // namespace AFSAI_PNS
}  // namespace afsai
