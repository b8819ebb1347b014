// Registry of compiled fused-step tile variants (one entry per template
// instantiation; filled by static initialisers in nsw_inst.cu).
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
};

std::vector<Variant>& variant_registry();

struct Registrar {
  explicit Registrar(const Variant& v) { variant_registry().push_back(v); }
};

}  // namespace nsw
