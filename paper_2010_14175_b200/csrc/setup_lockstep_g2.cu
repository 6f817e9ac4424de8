// setup_lockstep_g2.cu -- lockstep hit-list kernel instances with 2 new rows per bordering group.
#include "setup_lockstep_impl.cuh"

namespace afsai {
namespace AFSAI_PNS {
template SetupKernFn ls_instance<2>(int lpr, int nt, int hc);
}  // namespace AFSAI_PNS
}  // namespace afsai
