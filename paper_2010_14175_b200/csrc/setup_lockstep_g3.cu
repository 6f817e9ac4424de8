// setup_lockstep_g3.cu -- lockstep hit-list kernel instances with 3 new rows per bordering group.
#include "setup_lockstep_impl.cuh"

namespace afsai {
namespace AFSAI_PNS {
template SetupKernFn ls_instance<3>(int lpr, int nt, int hc);
}  // namespace AFSAI_PNS
}  // namespace afsai
