// Cost of one cluster-wide column-total exchange (config-4 cluster tile shape:
// 9 CTAs x 256 threads, 13 float4 column groups per CTA), three mechanisms:
//   0: push with st.async to every CTA's slot, completion on the receiver's
//      mbarrier (expect_tx) -- the product's exchange
//   1: push with plain remote stores + release-add on the receiver's counter,
//      receivers poll their own counter with acquire loads
//   2: local write, cluster barrier (arrive.release / wait.acquire), pull the
//      other CTAs' totals with remote loads
//   3: flagged 8-byte pushes (value + sequence tag in one b64 remote store, the
//      "LL" idea): no mbarrier, no fence; receivers poll their own slots until
//      every tag carries this exchange's sequence number
// Each iteration: the exchange, a fixed-order sum, two CTA barriers (as in
// the kernel).  Prints cycles per exchange (max over CTAs).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_exchange cluster_exchange.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

constexpr int CL = 9, NT = 256, NG = 13, ITERS = 2000;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) {
  unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}

template <int MODE>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT, 1) xk(long long* cyc, float* out) {
  __shared__ __align__(16) float slots[2][CL][NG * 4];
  __shared__ __align__(16) float own[NG * 4];
  __shared__ __align__(8) unsigned long long mb[2];
  __shared__ unsigned cnt[2];
  __shared__ float vec[NG * 4];
  __shared__ __align__(8) unsigned long long ll[2][CL][NG * 4];
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x;
  const unsigned rank = cluster.block_rank();
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mb[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mb[1])));
    cnt[0] = cnt[1] = 0;
  }
  if (MODE >= 3) {
    for (int q = tid; q < 2 * CL * NG * 4; q += NT) (&ll[0][0][0])[q] = 0ull;
  }
  if (tid == 0) {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < NG * 4) vec[tid] = 1.f + rank;
  cluster.sync();
  float acc = 0.f;
  unsigned ph = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    const int par = it & 1;
    if (MODE <= 2 && tid < NG) {
      float4 v = make_float4(vec[4 * tid] + it, vec[4 * tid + 1], vec[4 * tid + 2], vec[4 * tid + 3]);
      if (MODE == 2) {
        reinterpret_cast<float4*>(own)[tid] = v;
      } else {
        const unsigned slot = smem_u32(&slots[par][rank][4 * tid]);
        for (int q = 0; q < CL; ++q) {
          const unsigned ra = mapa(slot, q);
          if (MODE == 0) {
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                         ::"r"(ra), "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                           "r"(__float_as_uint(v.w)), "r"(mapa(smem_u32(&mb[par]), q)) : "memory");
          } else {
            asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "f"(v.x), "f"(v.y), "f"(v.z),
                         "f"(v.w) : "memory");
            asm volatile("red.release.cluster.shared::cluster.add.u32 [%0], 1;" ::"r"(mapa(smem_u32(&cnt[par]), q)) : "memory");
          }
        }
      }
    }
    if (MODE >= 3 && tid < NG * 4) {
      const float v = vec[tid] + (tid % 4 == 0 ? float(it) : 0.f);
      const unsigned long long pk = (unsigned long long)__float_as_uint(v) | ((unsigned long long)(unsigned(it) + 1u) << 32);
      const unsigned slot = smem_u32(&ll[par][rank][tid]);
      for (int q = 0; q < CL; ++q) {
        if (MODE == 3) asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(mapa(slot, q)), "l"(pk) : "memory");
        if (MODE == 4) asm volatile("st.volatile.shared::cluster.b64 [%0], %1;" ::"r"(mapa(slot, q)), "l"(pk) : "memory");
        if (MODE == 5) asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(mapa(slot, q)), "l"(pk) : "memory");
        if (MODE == 9) asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(mapa(slot, q)), "l"(pk) : "memory");
        if (MODE >= 6 && MODE <= 8) asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                                    ::"r"(mapa(slot, q)), "l"(pk), "r"(mapa(smem_u32(&mb[par]), q)) : "memory");
      }
    }
    if (MODE >= 6 && MODE <= 8 && tid == 0)   // keep the sink mbarrier's tx-count centred; nobody waits on it
      asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mb[par])), "r"(CL * NG * 4 * 8) : "memory");
    if (MODE == 0 && tid == 0) {
      asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(&mb[par])),
                   "r"(CL * NG * 16) : "memory");
    }
    if (MODE == 2) {
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (tid < NG * 4) {
      if (MODE == 0) {
        unsigned done = 0;
        while (!done)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(done) : "r"(smem_u32(&mb[par])), "r"((ph >> par) & 1u) : "memory");
      } else if (MODE == 1) {
        const unsigned want = unsigned(CL * NG) * unsigned(it / 2 + 1);
        unsigned c = 0;
        do {
          asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(c) : "r"(smem_u32(&cnt[par])) : "memory");
        } while (c < want);
      }
      float s = 0.f;
      if (MODE >= 3) {
        unsigned long long x[CL];
        bool all;
        do {
          all = true;
          for (int q = 0; q < CL; ++q) {
            if (MODE == 3) asm volatile("ld.relaxed.cluster.shared::cta.b64 %0, [%1];" : "=l"(x[q]) : "r"(smem_u32(&ll[par][q][tid])) : "memory");
            else if (MODE >= 8) asm volatile("ld.volatile.shared::cluster.b64 %0, [%1];" : "=l"(x[q]) : "r"(mapa(smem_u32(&ll[par][q][tid]), rank)) : "memory");
            else asm volatile("ld.volatile.shared::cta.b64 %0, [%1];" : "=l"(x[q]) : "r"(smem_u32(&ll[par][q][tid])) : "memory");
            all = all && unsigned(x[q] >> 32) == unsigned(it) + 1u;
          }
          if (MODE == 7 && !all) __nanosleep(40);
        } while (!all);
        for (int q = 0; q < CL; ++q) s += __uint_as_float(unsigned(x[q]));
      } else
      for (int q = 0; q < CL; ++q) {
        if (MODE == 2) {
          float x;
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x) : "r"(mapa(smem_u32(&own[tid]), q)) : "memory");
          s += x;
        } else {
          s += slots[par][q][tid];
        }
      }
      acc += s;
      vec[tid] = s * 1e-9f;
    }
    ph ^= 1u << par;
    __syncthreads();
    if (MODE == 2) {   // nobody overwrites `own` before every CTA has read it
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  if (tid < NG * 4) out[blockIdx.x * NG * 4 + tid] = acc;
  cluster.sync();
}

template <int MODE>
void run(const char* name) {
  const int grid = CL * 15;
  long long* cyc; float* out;
  cudaFuncSetAttribute(xk<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaMalloc(&cyc, grid * sizeof(long long));
  cudaMemset(cyc, 0, grid * sizeof(long long));
  cudaMalloc(&out, grid * NG * 4 * sizeof(float));
  xk<MODE><<<grid, NT>>>(cyc, out);
  xk<MODE><<<grid, NT>>>(cyc, out);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[grid];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-40s %s: %.0f cycles per exchange (max over CTAs)\n", name, cudaGetErrorString(e), double(mx) / ITERS);
  cudaFree(cyc); cudaFree(out);
}

int main() {
  run<0>("st.async + mbarrier (product)");
  run<1>("remote st + release-add counter");
  run<2>("cluster barrier + remote loads");
  run<3>("flagged b64 pushes, relaxed.cluster st/ld");
  run<4>("flagged b64 pushes, volatile st/ld");
  run<5>("flagged b64 pushes, weak st, volatile ld");
  run<6>("flagged b64 st.async (sink mbarrier), polled");
  run<7>("flagged b64 st.async, polled with nanosleep(40)");
  run<8>("flagged b64 st.async, polled via shared::cluster");
  run<9>("flagged b64 weak st, polled via shared::cluster");
  return 0;
}
