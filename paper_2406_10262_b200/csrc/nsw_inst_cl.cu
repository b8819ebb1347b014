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

template <int MC, int CG, int R, int NT, int CL>
size_t cl_smem_of(int T) {
  return cl_smem_bytes<NSW_S, MC, CG, R, NT, CL>(T);
}

#define NSW_CAT2(a, b) a##b
#define NSW_CAT(a, b) NSW_CAT2(a, b)
// (MC columns x CG lanes per row group, R rows per thread, NT threads, CL CTAs
// per user, MINB CTAs per SM)
#define NSW_REG_CLT(MC, CG, R, NT, CLS, MINB)                                                              \
  Registrar NSW_CAT(regcl_, __LINE__)(Variant{NSW_DT, MC * CG, R, NT,                                     \
                                              (const void*)&step_kernel_cl<NSW_S, MC, CG, R, NT, CLS, MINB>, \
                                              &cl_smem_of<MC, CG, R, NT, CLS>, CLS,                        \
                                              ClTile<NSW_S, MC, CG, R, NT, CLS>::NR, MINB});
#define NSW_REG_CL(CLS) NSW_REG_CLT(13, 4, NSW_R, 256, CLS, 1)

NSW_REG_CL(1)
NSW_REG_CL(2)
NSW_REG_CL(4)
NSW_REG_CL(8)
NSW_REG_CL(16)   // non-portable cluster size (B200 GPCs hold 16 SMs): n up to 8192 (fp32) / 2048 (fp64)
#if !NSW_F64 && defined(NSW_EXP_TILES) && NSW_EXP_TILES
// A/B builds only: config 2 (1000 x 21) split over 2-CTA clusters so two
// users share an SM (MINB 2)
NSW_REG_CLT(21, 1, 2, 256, 2, 2)
NSW_REG_CLT(11, 2, 4, 256, 2, 2)
NSW_REG_CLT(21, 1, 4, 128, 2, 2)
#endif
#if !NSW_F64
// 9-CTA clusters of 448 items (n <= 4032, config 4): B200's GPCs hold 15
// resident 8- or 9-CTA clusters, so 9 x 15 = 135 SMs work instead of 120
NSW_REG_CLT(13, 4, 7, 256, 9, 1)
// (two CTAs per SM on 16-CTA clusters -- (13,4,8,128), (7,8,8,256), (13,4,4,256)
// -- and a 14-warp (13,4,4,448) 9-CTA tile ran 3-19 % slower than the
// 1-CTA/SM tiles: profiles/r01/r01d_cluster_tile_variants.txt)
// (one-CTA 2-D tiles with 16-32 warps for configs 2 / 3 -- (6,4,4,1024),
// (11,2,4,512), (3,4,8,1024), (6,2,8,512) -- ran 9-45 % slower than the row
// tiles: profiles/r01/r01d_2d_tiles_cfg2_cfg3.txt)
#endif

}  // namespace
}  // namespace nsw
