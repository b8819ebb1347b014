// FP32-pipe issue-rate microbenchmark (B200): scalar FFMA (3 registers),
// FFMA with an immediate, and packed FFMA2 (fma.rn.f32x2).  Prints FMA
// operations per clock per SM for each form.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_rate fma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;   // independent chains per thread

__global__ void k_ffma(float* out, float x0, float y0) {
  float acc[CH], x[CH], y[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) { acc[j] = threadIdx.x * 1e-9f + j; x[j] = x0 + j * 1e-7f; y[j] = y0 - j * 1e-7f; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[j]) : "f"(x[j]), "f"(y[(j + 1) % CH]));
  }
  float s = 0; for (int j = 0; j < CH; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma_imm(float* out, float x0, float y0) {
  float acc[CH], x[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) { acc[j] = threadIdx.x * 1e-9f + j; x[j] = x0 + j * 1e-7f; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j) asm volatile("fma.rn.f32 %0, %1, 0f3F7FFFFE, %0;" : "+f"(acc[j]) : "f"(x[j]));
  }
  float s = 0; for (int j = 0; j < CH; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float x0, float y0) {
  unsigned long long acc[CH], x[CH], y[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    float2 a = make_float2(threadIdx.x * 1e-9f + j, j), b = make_float2(x0 + j * 1e-7f, x0), c = make_float2(y0 - j * 1e-7f, y0);
    acc[j] = *reinterpret_cast<unsigned long long*>(&a); x[j] = *reinterpret_cast<unsigned long long*>(&b);
    y[j] = *reinterpret_cast<unsigned long long*>(&c);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j]) : "l"(x[j]), "l"(y[(j + 1) % CH]));
  }
  float s = 0;
  for (int j = 0; j < CH; ++j) { float2 a = *reinterpret_cast<float2*>(&acc[j]); s += a.x + a.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// rdot-like: acc = fma(x_k, y_k, acc) with x_k, y_k streaming through registers
__global__ void k_ffma_dot(float* out, float x0, float y0) {
  float acc[4], x[16], y[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) { x[j] = x0 + j * 1e-7f; y[j] = y0 - j * 1e-7f; }
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = threadIdx.x * 1e-9f + j;
  for (int it = 0; it < ITERS / 2; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[k & 3]) : "f"(x[k]), "f"(y[(k * 5) & 15]));
  }
  float s = acc[0] + acc[1] + acc[2] + acc[3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// dependent-chain latency (one warp): cycles per FFMA / FFMA2 in a chain
__global__ void k_lat(float* out, long long* cyc, float x0) {
  float a = x0 + threadIdx.x, b = x0 * 0.5f;
  unsigned long long a2, b2;
  { float2 t = make_float2(a, a + 1), u = make_float2(b, b); a2 = *reinterpret_cast<unsigned long long*>(&t);
    b2 = *reinterpret_cast<unsigned long long*>(&u); }
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < 256; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(a) : "f"(b));
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < 256; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a2) : "l"(b2));
  long long t2 = clock64();
  out[threadIdx.x] = a + __uint_as_float(unsigned(a2));
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}

template <typename K>
void run(const char* name, K kern, float* d, int blocks, int threads, double flops_per_inst, int clk_khz, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  kern<<<blocks, threads>>>(d, 1.0f, 0.5f);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(d, 1.0f, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double insts = 5.0 * blocks * threads * double(ITERS) * CH;  // thread-level FMA instructions
  const double fma_ops = insts * flops_per_inst;
  const double per_s = fma_ops / (ms * 1e-3);
  printf("%-10s blocks=%d threads=%d  %.3f ms  %.2f T fma-ops/s  (%.1f per clk per SM at %d MHz max)\n", name, blocks,
         threads, ms / 5, per_s * 1e-12, per_s / (sms * clk_khz * 1e3), clk_khz / 1000);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* d; cudaMalloc(&d, 1 << 26);
  long long* cyc; cudaMallocManaged(&cyc, 16);
  k_lat<<<1, 32>>>(d, cyc, 1.0f); cudaDeviceSynchronize();
  k_lat<<<1, 32>>>(d, cyc, 1.0f); cudaDeviceSynchronize();
  printf("dependent chain: FFMA %.2f cycles, FFMA2 %.2f cycles\n", cyc[0] / 256.0, cyc[1] / 256.0);
  for (int t : {128, 256, 512}) {
    int blocks = p.multiProcessorCount * (1024 / t);
    run("ffma", k_ffma, d, blocks, t, 1.0, clk, p.multiProcessorCount);
    run("ffma_imm", k_ffma_imm, d, blocks, t, 1.0, clk, p.multiProcessorCount);
    run("ffma2", k_ffma2, d, blocks, t, 2.0, clk, p.multiProcessorCount);
    run("ffma_dot", k_ffma_dot, d, blocks, t, 1.0, clk, p.multiProcessorCount);
  }
  return 0;
}
