// On-device generation of the BASELINE synthetic relevance (SURVEY.md 8(d),
// 8(f) rank 4), so configs 3 / 4 (50k x 2000, 100k x 4000) need no host
// generation or host-to-device copy of a multi-GB matrix.
//
// Counter-based: every random value is a pure function of (seed, stream,
// index) through Philox4x32-10, so any user slice is generated independently
// and identically (a rank generates exactly its shard), and a host port
// (oracle/datagen_port.py, test infrastructure) reproduces the values.
//   latent    r_ui = sigmoid(<p_u, q_i> + b_i), p, q ~ N(0, I_d / d),
//             b ~ N(0, s) or b = L - mean(L), L ~ LogNormal(0, s)  (configs 1, 2, 4)
//   sparse    per user `per_user` distinct items drawn with P(i) ~ rank_i^-s
//             (Gumbel-top-k: the top keys log p_i + Gumbel are a sample
//             without replacement), r ~ Beta(2, 5) as G2 / (G2 + G5) with
//             integer-shape gammas from uniforms; every other entry `floor`
//             (config 3)
// Streams: 1 user factors, 2 item factors, 3 item bias, 4 Zipf ranks,
// 5 Gumbel keys, 6 Beta values.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/nswrank_b200.h"
#include "nsw_device.cuh"
#include "nsw_pool.h"

namespace nsw {
namespace {

struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ inline void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
  const uint64_t p = uint64_t(a) * b;
  hi = uint32_t(p >> 32);
  lo = uint32_t(p);
}

// Philox4x32-10 (Salmon et al., SC'11)
__device__ inline U4 philox(uint64_t index, uint32_t stream, uint64_t seed) {
  uint32_t c0 = uint32_t(index), c1 = uint32_t(index >> 32), c2 = stream, c3 = 0;
  uint32_t k0 = uint32_t(seed), k1 = uint32_t(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2511F53u, c0, hi0, lo0);
    mulhilo(0xCD9E8D57u, c2, hi1, lo1);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return U4{c0, c1, c2, c3};
}

// 53-bit uniform in the open interval (0, 1): log(u) and log(-log(u)) finite
__device__ inline double u53(uint32_t a, uint32_t b) {
  const uint64_t v = (uint64_t(a >> 5) << 26) | uint64_t(b >> 6);
  return (double(v) + 0.5) * (1.0 / 9007199254740992.0);
}

__device__ inline double normal01(uint64_t index, uint32_t stream, uint64_t seed) {
  const U4 x = philox(index, stream, seed);
  const double u1 = u53(x.x, x.y), u2 = u53(x.z, x.w);
  return __dmul_rn(sqrt(-2.0 * log(u1)), cos(6.283185307179586 * u2));
}

// out[r][c] = scale * N(0,1) of element index (row0 + r) * cols + c
__global__ void normal_matrix_kernel(double* __restrict__ out, int rows, int cols, long long row0, double scale,
                                     uint32_t stream, uint64_t seed) {
  const size_t total = size_t(rows) * cols;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x)
    out[e] = __dmul_rn(normal01(uint64_t(row0) * cols + e, stream, seed), scale);
}

// item bias: kind 0 none, 1 normal(0, s), 2 lognormal(0, s) centred; one CTA,
// fixed-order mean (deterministic)
__global__ void bias_kernel(double* __restrict__ b, int n, int kind, double s, uint64_t seed) {
  __shared__ double part[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) {
    double v = 0.0;
    if (kind == 1) v = __dmul_rn(normal01(uint64_t(i), 3, seed), s);
    if (kind == 2) v = exp(__dmul_rn(normal01(uint64_t(i), 3, seed), s));
    b[i] = v;
    acc += v;
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  if (kind == 2) {
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int t = 0; t < 256; ++t) tot += part[t];
      part[0] = tot / n;
    }
    __syncthreads();
    const double mean = part[0];
    for (int i = threadIdx.x; i < n; i += 256) b[i] = b[i] - mean;
  }
}

// r = clamp(sigmoid(<P_u, Q_i> + b_i)), the dot in index order with separate
// multiply and add roundings; 32 users x 32 items per CTA, factors in smem
template <typename S>
__global__ void latent_kernel(const double* __restrict__ P, const double* __restrict__ Q,
                              const double* __restrict__ b, int U, int n, int d, double floor_v,
                              S* __restrict__ out) {
  extern __shared__ double sm[];   // [32][d + 1] P rows, [32][d + 1] Q rows
  double* sP = sm;
  double* sQ = sm + 32 * (d + 1);
  const int u0 = blockIdx.y * 32, i0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * d; e += blockDim.x) {
    const int r = e / d, c = e - r * d;
    sP[r * (d + 1) + c] = u0 + r < U ? P[size_t(u0 + r) * d + c] : 0.0;
    sQ[r * (d + 1) + c] = i0 + r < n ? Q[size_t(i0 + r) * d + c] : 0.0;
  }
  __syncthreads();
  const int ti = threadIdx.x & 31;
  for (int ru = threadIdx.x >> 5; ru < 32; ru += blockDim.x >> 5) {
    const int u = u0 + ru, i = i0 + ti;
    if (u >= U || i >= n) continue;
    double z = 0.0;
    for (int c = 0; c < d; ++c) z = __dadd_rn(z, __dmul_rn(sP[ru * (d + 1) + c], sQ[ti * (d + 1) + c]));
    z = __dadd_rn(z, b[i]);
    double r = 1.0 / (1.0 + exp(-z));
    r = fmin(fmax(r, 1e-6), 1.0);
    if constexpr (sizeof(S) == 4) r = fmin(fmax(double(float(r)), 1e-6), 1.0);
    out[size_t(u) * n + i] = S(r);
  }
}

// Zipf ranks: rank_i = 1 + #{j : key_j < key_i} with 64-bit keys from stream 4
// (a uniformly random permutation); logp_i = -s log(rank_i)
__global__ void zipf_logp_kernel(double* __restrict__ logp, int n, double s, uint64_t seed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  auto key = [&](int j) {
    const U4 x = philox(uint64_t(j), 4, seed);
    return (uint64_t(x.x) << 32) | x.y;
  };
  const uint64_t ki = key(i);
  int rank = 1;
  for (int j = 0; j < n; ++j) {
    const uint64_t kj = key(j);
    rank += (kj < ki) || (kj == ki && j < i);
  }
  logp[i] = -s * log(double(rank));
}

// One CTA per user: Gumbel keys in shared memory, `per_user` rounds of a
// block arg-max (largest key, lowest index on ties), Beta(2, 5) values in
// selection order
template <typename S>
__global__ void __launch_bounds__(256) sparse_kernel(const double* __restrict__ logp, int U0, int n, int per_user,
                                                     double floor_v, uint64_t seed, S* __restrict__ out) {
  extern __shared__ double keys[];   // [n]
  __shared__ double bv[8];
  __shared__ int bi[8];
  const int ul = blockIdx.x;
  const uint64_t u = uint64_t(U0) + ul;
  S* row = out + size_t(ul) * n;
  for (int i = threadIdx.x; i < n; i += 256) {
    const U4 x = philox(u * uint64_t(n) + i, 5, seed);
    keys[i] = logp[i] - log(-log(u53(x.x, x.y)));
    row[i] = S(floor_v);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = 0; j < per_user; ++j) {
    double best = -INFINITY;
    int bidx = n;
    for (int i = threadIdx.x; i < n; i += 256)
      if (keys[i] > best) {
        best = keys[i];
        bidx = i;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) {
        best = ov;
        bidx = oi;
      }
    }
    if (lane == 0) {
      bv[warp] = best;
      bi[warp] = bidx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b0 = bv[0];
      int i0 = bi[0];
      for (int w = 1; w < 8; ++w)
        if (bv[w] > b0 || (bv[w] == b0 && bi[w] < i0)) {
          b0 = bv[w];
          i0 = bi[w];
        }
      // Beta(2, 5) = G2 / (G2 + G5), G_k = -sum of k log-uniforms; the 7
      // uniforms of draw (u, j) come from Philox indices 4 (u per_user + j) + 0..3
      const uint64_t base = (u * uint64_t(per_user) + j) * 4;
      double l[8];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const U4 x = philox(base + c, 6, seed);
        l[2 * c] = log(u53(x.x, x.y));
        l[2 * c + 1] = log(u53(x.z, x.w));
      }
      const double g2 = -(l[0] + l[1]);
      const double g5 = -((((l[2] + l[3]) + l[4]) + l[5]) + l[6]);
      double r = g2 / (g2 + g5);
      r = fmin(fmax(r, 1e-6), 1.0);
      if constexpr (sizeof(S) == 4) r = fmin(fmax(double(float(r)), 1e-6), 1.0);
      row[i0] = S(r);
      keys[i0] = -INFINITY;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace nsw

using namespace nsw;

extern "C" {

nsw_status nsw_datagen_latent(int64_t user0, int32_t users, int32_t n, int32_t d, int32_t bias_kind,
                              double bias_scale, uint64_t seed, int32_t dtype, void* out, void* stream) {
  if (!out || users <= 0 || n <= 0 || d <= 0 || user0 < 0) return NSW_ERR_ARG;
  if (dtype != NSW_F32 && dtype != NSW_F64) return NSW_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* buf = nullptr;   // P [users][d] | Q [n][d] | b [n]
  if (private_malloc((void**)&buf, (size_t(users) * d + size_t(n) * d + n) * sizeof(double), st) != cudaSuccess)
    return NSW_ERR_CUDA;
  double* P = buf;
  double* Q = P + size_t(users) * d;
  double* b = Q + size_t(n) * d;
  const double sc = 1.0 / sqrt(double(d));
  normal_matrix_kernel<<<sm_count() * 4, 256, 0, st>>>(P, users, d, user0, sc, 1, seed);
  normal_matrix_kernel<<<sm_count() * 4, 256, 0, st>>>(Q, n, d, 0, sc, 2, seed);
  bias_kernel<<<1, 256, 0, st>>>(b, n, bias_kind, bias_scale, seed);
  const dim3 grid((n + 31) / 32, (users + 31) / 32);
  const size_t smem = size_t(64) * (d + 1) * sizeof(double);
  if (dtype == NSW_F32) {
    allow_smem((const void*)latent_kernel<float>, size_t(smem));
    latent_kernel<float><<<grid, 256, smem, st>>>(P, Q, b, users, n, d, 1e-6, static_cast<float*>(out));
  } else {
    allow_smem((const void*)latent_kernel<double>, size_t(smem));
    latent_kernel<double><<<grid, 256, smem, st>>>(P, Q, b, users, n, d, 1e-6, static_cast<double*>(out));
  }
  const cudaError_t e = cudaGetLastError();
  cudaFreeAsync(buf, st);
  return e == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}

nsw_status nsw_datagen_sparse(int64_t user0, int32_t users, int32_t n, int32_t per_user, double zipf_s,
                              double floor_value, uint64_t seed, int32_t dtype, void* out, void* stream) {
  if (!out || users <= 0 || n <= 0 || per_user <= 0 || per_user > n || user0 < 0) return NSW_ERR_ARG;
  if (dtype != NSW_F32 && dtype != NSW_F64) return NSW_ERR_ARG;
  if (size_t(n) * sizeof(double) > 200 * 1024) return NSW_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* logp = nullptr;
  if (private_malloc((void**)&logp, size_t(n) * sizeof(double), st) != cudaSuccess) return NSW_ERR_CUDA;
  zipf_logp_kernel<<<(n + 127) / 128, 128, 0, st>>>(logp, n, zipf_s, seed);
  const size_t smem = size_t(n) * sizeof(double);
  if (dtype == NSW_F32) {
    allow_smem((const void*)sparse_kernel<float>, size_t(smem));
    sparse_kernel<float><<<users, 256, smem, st>>>(logp, int(user0), n, per_user, floor_value, seed,
                                                   static_cast<float*>(out));
  } else {
    allow_smem((const void*)sparse_kernel<double>, size_t(smem));
    sparse_kernel<double><<<users, 256, smem, st>>>(logp, int(user0), n, per_user, floor_value, seed,
                                                    static_cast<double*>(out));
  }
  const cudaError_t e = cudaGetLastError();
  cudaFreeAsync(logp, st);
  return e == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}

}  // extern "C"
