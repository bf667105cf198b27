// dist.cu -- multi-GPU hooks (placeholder until the NCCL exchange lands).
#include "ctx.cuh"

void diter_dist_free(di_ctx *) {}
double diter_dist_max(di_ctx *, double v) { return v; }
double diter_dist_sum(di_ctx *, double v) { return v; }
di_status diter_dist_reset(di_ctx *) { return DI_OK; }
di_status diter_dist_run(di_ctx *ctx, double) {
  diter_set_err(ctx, "distributed run not built");
  return DI_ERR_UNSUPPORTED;
}
extern "C" di_status di_create_dist(di_ctx **out, int32_t, int32_t, const void *, const int64_t *, int64_t,
                                    const int64_t *, const int32_t *, const double *, const double *, double,
                                    const di_options *) {
  if (out) *out = nullptr;
  diter_set_err(nullptr, "di_create_dist: not built");
  return DI_ERR_UNSUPPORTED;
}
extern "C" di_status di_get_unique_id(void *) {
  diter_set_err(nullptr, "di_get_unique_id: not built");
  return DI_ERR_UNSUPPORTED;
}
