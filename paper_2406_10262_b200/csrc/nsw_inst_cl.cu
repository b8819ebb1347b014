// Cluster-tile instantiations (m up to 52, n up to CL * rows-per-CTA):
// compiled with -DNSW_F64=0|1.
#include "nsw_registry.h"
#include "nsw_step_cluster.cuh"

#if NSW_F64
#define NSW_S double
#define NSW_DT 1
#define NSW_R 2
#else
#define NSW_S float
#define NSW_DT 0
#define NSW_R 8
#endif

namespace nsw {
namespace {

template <int CL>
size_t cl_smem_of(int T) {
  return cl_smem_bytes<NSW_S, 13, 4, NSW_R, 256, CL>(T);
}

#define NSW_CAT2(a, b) a##b
#define NSW_CAT(a, b) NSW_CAT2(a, b)
#define NSW_REG_CL(CLS)                                                                                        \
  Registrar NSW_CAT(regcl_, __LINE__)(Variant{NSW_DT, 52, NSW_R, 256,                                          \
                                              (const void*)&step_kernel_cl<NSW_S, 13, 4, NSW_R, 256, CLS>,     \
                                              &cl_smem_of<CLS>, CLS, ClTile<NSW_S, 13, 4, NSW_R, 256, CLS>::NR});

NSW_REG_CL(1)
NSW_REG_CL(2)
NSW_REG_CL(4)
NSW_REG_CL(8)
NSW_REG_CL(16)   // non-portable cluster size (B200 GPCs hold 16 SMs): n up to 8192 (fp32) / 2048 (fp64)

}  // namespace
}  // namespace nsw
