// Inner operator seam: the reference's private batch functions as device
// operators (fixed schedule).  Stubs until the op kernels land.
#include <string>

#include "../../include/nswrank_b200.h"

extern "C" {

nsw_status nsw_sinkhorn_batch_f64(const double*, const double*, int32_t, int32_t, int32_t, int32_t, double*,
                                  double*, double*, double*, void*) {
  return NSW_ERR_UNSUPPORTED;
}
nsw_status nsw_sinkhorn_batch_f32(const float*, const float*, int32_t, int32_t, int32_t, int32_t, float*, float*,
                                  float*, float*, void*) {
  return NSW_ERR_UNSUPPORTED;
}
nsw_status nsw_sinkhorn_backward_batch_f64(const double*, const double*, const double*, const double*,
                                           const double*, const double*, int32_t, int32_t, int32_t, int32_t,
                                           double*, void*) {
  return NSW_ERR_UNSUPPORTED;
}
nsw_status nsw_sinkhorn_backward_batch_f32(const float*, const float*, const float*, const float*, const float*,
                                           const float*, int32_t, int32_t, int32_t, int32_t, float*, void*) {
  return NSW_ERR_UNSUPPORTED;
}

}  // extern "C"
