// dist.cu -- multi-GPU set-up halo, G^T exchange and PCG halos.
#include "dist.h"

namespace afsai {
int dist_setup(afsai_ctx_t, const afsai_csr_t *, const afsai_params_t *, afsai_factor_t *, afsai_status_t *status) {
    return set_status(status, AFSAI_ELIMIT, "multi-GPU set-up not built yet");
}
int dist_apply(afsai_ctx_t, afsai_factor_t, const double *, double *, afsai_status_t *status) {
    return set_status(status, AFSAI_ELIMIT, "multi-GPU apply not built yet");
}
int dist_pcg(afsai_ctx_t, const afsai_csr_t *, afsai_factor_t, const double *, double *, double, int32_t,
             afsai_pcg_report_t *, afsai_status_t *status) {
    return set_status(status, AFSAI_ELIMIT, "multi-GPU PCG not built yet");
}
void dist_free(afsai_factor_t) {}
}  // namespace afsai
