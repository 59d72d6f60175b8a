// Template instances of the fused sweep, layers L == 1 (see pg_sweep_fused.cu).
#include "pg_sweep_fused.cuh"

namespace pgb {

cudaError_t launch_fused_inst_1(int key, pg_grid *g, const FusedParams &P, dim3 grid, bool *found) {
  *found = true;
#define X(l, f, s, d, w)                                                         \
  if constexpr (l == 1) {                                                        \
    if (key == fused_key(l, f, s, d, w)) return launch_fused_t<l, f, s, d, w, false>(g, P, grid); \
  }
  PG_FUSED_CASES(X)
#undef X
#define X(l, f, s, d, w)                                                         \
  if constexpr (l == 1) {                                                        \
    if (key == fused_key(l, f, s, d, w, true)) return launch_fused_t<l, f, s, d, w, true>(g, P, grid); \
  }
  PG_FUSED_SLAB_CASES(X)
#undef X
  *found = false;
  return cudaErrorInvalidValue;
}

}  // namespace pgb
