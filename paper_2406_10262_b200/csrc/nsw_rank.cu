// Top-m ranking of a stochastic ranking tensor X [U][n][m] (m = positions +
// dummy): out[u][k] = argmax_i X[u][i][k] for every real position k < m-1,
// lowest index on ties (numpy argmax semantics).
//
// The reference defines no ranking extraction; this is the definition
// SURVEY.md 8(a) names for the north star's "top-m ranking bit-exact" check
// (the oracle's top_positions).  One CTA per user, one warp per position:
// lanes stride the items in increasing order (a lane keeps the first of its
// ties), then a warp arg-max that prefers the lower index on equal values.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/nswrank_b200.h"

namespace nsw {
namespace {

constexpr int kRankThreads = 128;

template <typename S>
__global__ void __launch_bounds__(kRankThreads) top_positions_kernel(const S* __restrict__ X, int n, int m,
                                                                     int32_t* __restrict__ out) {
  const int u = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const S* xu = X + size_t(u) * n * m;
  for (int k = warp; k < m - 1; k += kRankThreads / 32) {
    S best = S(0);
    int idx = n;   // sentinel: no item seen
    for (int i = lane; i < n; i += 32) {
      const S v = __ldg(xu + size_t(i) * m + k);
      if (idx == n || v > best) {
        best = v;
        idx = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const S ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      const bool take = oi != n && (idx == n || ob > best || (ob == best && oi < idx));
      if (take) {
        best = ob;
        idx = oi;
      }
    }
    if (lane == 0) out[size_t(u) * (m - 1) + k] = idx;
  }
}

template <typename S>
nsw_status launch_top_positions(const void* X, int32_t U, int32_t n, int32_t m, int32_t* out, void* stream) {
  if (!X || !out) return NSW_ERR_ARG;
  if (U <= 0 || n <= 0 || m < 2) return NSW_ERR_SHAPE;
  top_positions_kernel<S><<<U, kRankThreads, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const S*>(X), n, m,
                                                                                       out);
  return cudaGetLastError() == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}

}  // namespace
}  // namespace nsw

extern "C" {

nsw_status nsw_top_positions_f32(const float* X, int32_t U, int32_t n, int32_t m, int32_t* out, void* stream) {
  return nsw::launch_top_positions<float>(X, U, n, m, out, stream);
}

nsw_status nsw_top_positions_f64(const double* X, int32_t U, int32_t n, int32_t m, int32_t* out, void* stream) {
  return nsw::launch_top_positions<double>(X, U, n, m, out, stream);
}

}  // extern "C"
