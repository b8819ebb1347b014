// One translation unit per (scalar type, M): compiled with
//   -DNSW_F64=0|1 -DNSW_M=<columns>
// and registers the (rows/thread, threads/CTA, min CTAs/SM) tile shapes for
// that pair.  MINB caps registers at 64K / (NT * MINB) per thread.
#include "nsw_registry.h"
#include "nsw_step_kernel.cuh"

#ifndef NSW_EXP_TILES
#define NSW_EXP_TILES 0
#endif
#ifndef NSW_M
#error "NSW_M must be defined"
#endif
// tensor-core adjoint variants (tcgen05 + TMEM), fp32 only; registered with
// dtype 2 so the default chooser skips them until selected explicitly
#define NSW_REG_TC(R, NT, MINB)                                                                        \
  Registrar NSW_CAT(regtc_, __LINE__)(Variant{2, NSW_M, R, NT,                                         \
                                              (const void*)&step_kernel<NSW_S, NSW_M, R, NT, MINB, true>, \
                                              &smem_tc_of<R, NT, MINB>, 1, 0, MINB});

#if NSW_F64
#define NSW_S double
#define NSW_DT 1
#else
#define NSW_S float
#define NSW_DT 0
#endif

namespace nsw {
namespace {

template <int R, int NT, int MINB>
size_t smem_of(int T) {
  return step_smem_bytes<NSW_S, NSW_M, R, NT, MINB>(T);
}
template <int R, int NT, int MINB>
size_t smem_tc_of(int T) {
  return step_smem_bytes<NSW_S, NSW_M, R, NT, MINB, true>(T);
}

#define NSW_CAT2(a, b) a##b
#define NSW_CAT(a, b) NSW_CAT2(a, b)
#define NSW_REG(R, NT, MINB)                                                                        \
  Registrar NSW_CAT(reg_, __LINE__)(Variant{NSW_DT, NSW_M, R, NT,                                   \
                                            (const void*)&step_kernel<NSW_S, NSW_M, R, NT, MINB>, \
                                            &smem_of<R, NT, MINB>, 1, 0, MINB});

#if NSW_F64
// parity instantiation: shapes up to 2048 (M <= 16) / 1024 (M <= 32) items
#if NSW_M <= 16
NSW_REG(1, 64, 1)
NSW_REG(1, 128, 1)
NSW_REG(1, 256, 1)
NSW_REG(2, 256, 1)
NSW_REG(2, 512, 1)
NSW_REG(4, 512, 1)
#else
NSW_REG(1, 64, 1)
NSW_REG(1, 128, 1)
NSW_REG(1, 256, 1)
NSW_REG(1, 512, 1)
NSW_REG(2, 512, 1)
#endif
#else
#if NSW_M <= 11
NSW_REG_TC(4, 128, 4)
NSW_REG(16, 32, 7)   // one-warp tile, 7 per SM: 1036 users per wave (config 1 in one wave)
NSW_REG(1, 64, 1)
NSW_REG(2, 64, 1)
NSW_REG(4, 64, 6)
NSW_REG(8, 64, 6)
NSW_REG(8, 64, 7)   // 7 per SM (register-lean, no input staging): 1036 users per wave
NSW_REG(4, 128, 3)
NSW_REG(4, 128, 4)   // 4 per SM: one wave of up to 592 users (strong-scaling shards)
NSW_REG(8, 128, 3)
// (tail tile capped at 128 / 80 registers to start beside draining main CTAs:
// 0.4 / 1.2 % slower, profiles/r01/r01g_tail_registers.txt)
NSW_REG(8, 256, 1)   // (4, 512, 1): 16 warps, 11 % slower on config 3 (profiles/r01/r01d_row_tiles_cfg2_cfg3.txt)
NSW_REG(2, 256, 1)
NSW_REG(1, 512, 1)
#if NSW_EXP_TILES   // A/B builds only: 9-13-warp row tiles for config 3
NSW_REG(6, 352, 1)
NSW_REG(7, 288, 1)
NSW_REG(5, 416, 1)
#endif
#elif NSW_M <= 16
NSW_REG(1, 64, 1)
NSW_REG(2, 64, 1)
NSW_REG(4, 64, 4)
NSW_REG(8, 64, 4)
NSW_REG(4, 128, 2)
NSW_REG(8, 128, 2)
NSW_REG(8, 256, 1)
NSW_REG(2, 256, 1)
NSW_REG(1, 512, 1)
#elif NSW_M <= 24
NSW_REG_TC(4, 256, 1)   // config 2 tile with the tensor-core adjoint
NSW_REG(1, 64, 1)
NSW_REG(2, 64, 1)
NSW_REG(4, 64, 4)
NSW_REG(4, 128, 1)
NSW_REG(4, 256, 1)
NSW_REG(2, 256, 1)
NSW_REG(2, 512, 1)
#if NSW_EXP_TILES   // A/B builds only: 7-12-warp row tiles for config 2
NSW_REG(3, 384, 1)
NSW_REG(4, 288, 1)
NSW_REG(5, 224, 1)
#endif
#else
NSW_REG(1, 64, 1)
NSW_REG(2, 64, 1)
NSW_REG(2, 128, 1)
NSW_REG(2, 256, 1)
NSW_REG(4, 256, 1)   // (2, 512) at M = 32 crashes ptxas 12.9
#endif
#endif

}  // namespace
}  // namespace nsw
