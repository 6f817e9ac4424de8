// setup_prow_g4.cu -- pattern-row set-up kernel instances with 4 new columns bordered in lockstep.
#include "setup_prow_impl.cuh"

namespace afsai {
namespace AFSAI_PNS {
template SetupKernFn prow_instance<4>(int nt, int nv);
}  // namespace AFSAI_PNS
}  // namespace afsai
