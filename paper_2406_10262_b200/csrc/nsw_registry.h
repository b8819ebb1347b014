// Registry of compiled fused-step tile variants (one entry per template
// instantiation; filled by static initialisers in nsw_inst*.cu).
#pragma once
#include <cstddef>
#include <vector>

namespace nsw {

struct Variant {
  int dtype;  // 0 = f32, 1 = f64
  int M;      // compile-time column count (m <= M, padded)
  int R;      // rows per thread
  int NT;     // threads per CTA
  const void* fn;
  size_t (*smem)(int T);
  int CL = 1;     // CTAs per user (thread-block cluster) ; 1 = one CTA per user
  int rows = 0;   // items per CTA (R * NT for the 1-D tiles)
  int minb = 1;   // __launch_bounds__ min CTAs per SM (register cap)
};

std::vector<Variant>& variant_registry();

struct Registrar {
  explicit Registrar(Variant v) {
    if (v.rows == 0) v.rows = v.R * v.NT;
    variant_registry().push_back(v);
  }
};

}  // namespace nsw
