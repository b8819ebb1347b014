// Private stream-ordered device memory pool of the library (one per device,
// created on first use; keeps its memory between calls so repeated solves and
// metrics passes allocate without OS calls).  The device's default pool --
// shared with torch and every other cudaMallocAsync user -- is never touched.
// nsw_release_cached() trims it.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

namespace nsw {

struct PoolTable {
  std::mutex mu;
  cudaMemPool_t pool[64] = {};
};

// Raises a kernel's dynamic shared-memory cap (per device), never lowers it:
// solvers of different shapes in one process -- in different host threads --
// share the kernels, and a cap lowered by one between another's setup and its
// launch would fail that launch.  The cap is a permission, not a request: a
// launch's carve-out follows the bytes it asks for.
inline cudaError_t allow_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cap;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = cap[{dev, fn}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e == cudaSuccess) cur = bytes;
  return e;
}

inline PoolTable& pool_table() {
  static PoolTable t;
  return t;
}

inline cudaMemPool_t private_pool(int device) {
  if (device < 0 || device >= 64) return nullptr;
  PoolTable& t = pool_table();
  std::lock_guard<std::mutex> lk(t.mu);
  if (!t.pool[device]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
    uint64_t keep = ~uint64_t(0);
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    t.pool[device] = p;
  }
  return t.pool[device];
}

// stream-ordered allocation on the current device from the private pool
inline cudaError_t private_malloc(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool = private_pool(dev);
  if (!pool) return cudaErrorMemoryAllocation;
  return cudaMallocFromPoolAsync(p, bytes < 16 ? 16 : bytes, pool, st);
}

}  // namespace nsw
