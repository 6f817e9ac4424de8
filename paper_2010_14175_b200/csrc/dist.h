// Multi-GPU (one process per GPU, NCCL over NVLink) entry points: dist.cu.
#pragma once
#include "afsai_internal.h"

namespace afsai {
int dist_setup(afsai_ctx_t ctx, const afsai_csr_t *A_local, const afsai_params_t *p, afsai_factor_t *out,
               afsai_status_t *status);
int dist_apply(afsai_ctx_t ctx, afsai_factor_t F, const double *r, double *z, afsai_status_t *status);
int dist_pcg(afsai_ctx_t ctx, const afsai_csr_t *A_local, afsai_factor_t F, const double *b, double *x, double tol,
             int32_t max_iters, afsai_pcg_report_t *rep, afsai_status_t *status);
void dist_free(afsai_factor_t F);
int plan_ranges(int32_t me, int32_t nranks, const int64_t *bounds, const int64_t *lo, const int64_t *hi,
                int64_t *out, int32_t max_out);
}  // namespace afsai
