// Host side and template instances of the two-level red-black SOR pipeline
// (kernel: pg_sweep2.cuh).  Used for full F = 2 launches of the mesh sweep when
// option "pipe" is on (default); partial launches (fewer than 2 sweeps left)
// and other F run k_rb_sweep_fused.
#include "pg_sweep2.cuh"

#include <algorithm>

namespace pgb {

namespace {

template <int L, int W, bool SLAB>
cudaError_t launch2_t(pg_grid *g, const FusedParams &P, dim3 grid, bool pdl) {
  auto kern = k_rb_sweep2<L, W, SLAB>;
  const size_t smem = Sweep2Geo<L, W>::SMEM;
  if (g->tma_kernel_set != (const void *)kern || g->tma_smem_set != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
    g->tma_kernel_set = (const void *)kern;
    g->tma_smem_set = smem;
  }
  // programmatic dependent launch: this grid may start (prologue, constant
  // rows) while the previous sweep launch drains; it waits for it in-kernel
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(Sweep2Geo<L, W>::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = g->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, P);
}

template <int L, int W, bool SLAB>
int occupancy_t() {
  auto kern = k_rb_sweep2<L, W, SLAB>;
  const size_t smem = Sweep2Geo<L, W>::SMEM;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, Sweep2Geo<L, W>::NT, smem) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  return n < 1 ? 1 : n;
}

}  // namespace

int sweep2_width(int L) {
  switch (L) {
#define X(l, w) \
  case l:       \
    return w;
    PG_SWEEP2_CASES(X)
#undef X
    default:
      return 0;
  }
}

int sweep2_ctas_per_sm(int L, bool slab) {
  static int cache[2][kMaxLayers + 1] = {};
  if (L < 1 || L > kMaxLayers) return 1;
  int &c = cache[slab ? 1 : 0][L];
  if (c == 0) {
    switch (L) {
#define X(l, w) \
  case l:       \
    c = slab ? occupancy_t<l, w, true>() : occupancy_t<l, w, false>(); \
    break;
      PG_SWEEP2_CASES(X)
#undef X
      default:
        c = 1;
    }
  }
  return c;
}

// CTAs of one k_rb_sweep2 launch over the grid's (owned) rows
int64_t sweep2_grid_ctas(const pg_grid *g) {
  const int W = sweep2_width(g->md.L);
  if (W == 0) return 0;
  const int y0 = g->slab ? g->y_begin : 0, y1 = g->slab ? g->y_end : g->md.NY;
  const int H = g->rows > 0 ? std::max(1, std::min(g->rows, y1 - y0)) : sweep2_rows_per_cta(g, y1 - y0);
  const int I = W - 4;
  return (int64_t)((g->md.HP + I - 1) / I) * ((y1 - y0 + H - 1) / H);
}

int sweep2_rows_per_cta(const pg_grid *g, int ny) {
  const int W = sweep2_width(g->md.L);
  const int I = W - 4;
  const int strips = (g->md.HP + I - 1) / I;
  int chunks = (g->num_sms * sweep2_ctas_per_sm(g->md.L, g->slab && g->hx.G > 0)) / strips;
  if (chunks < 1) chunks = 1;
  int H = (ny + chunks - 1) / chunks;
  return H < 1 ? 1 : H;
}

cudaError_t launch_rb_sweep2(pg_grid *g, double omega, double tol, int j, int rows_per_cta, int y_begin,
                             int y_end, int ypar, bool pdl) {
  const int L = g->md.L;
  const int W = sweep2_width(L);
  if (W == 0) return cudaErrorInvalidValue;
  FusedParams P;
  if (!fill_fused_params(g, P, omega, tol, j, 2, W, rows_per_cta, y_begin, y_end, ypar))
    return cudaErrorNotSupported;
  P.pre = pdl ? 1 : 0;
  {
    const SlabHalo &h = g->hx;
    // the peer protocol waits on the other slabs: armed only while the group
    // runs (a slab grid used alone, e.g. pg_dc, sweeps without it)
    P.p2p = (g->slab && h.G > 0 && h.p2p && g->group_active) ? 1 : 0;
    P.nranks = h.nranks;
    for (int k = 0; k < 2; ++k) {
      P.peer_lo[k] = h.peer_lo[k];
      P.peer_hi[k] = h.peer_hi[k];
    }
    for (int k = 0; k < kMaxPeers; ++k) {
      P.sig_all[k] = h.sig_all[k];
      P.pnorm_all[k] = h.pnorm_all[k];
    }
    const int wi = W == 64 ? 1 : 0;
    if (P.p2p && h.has_lo) P.mRlo_b = h.mlo_b[wi];
    if (P.p2p && h.has_hi) P.mRhi_b = h.mhi_b[wi];
  }
  // L2 policy (auto): a mesh whose per-launch footprint (56 B per storage
  // element) is below twice the L2 streams its reads evict_first and writes V
  // evict_last, so the next launch finds V in L2 (config 1: +4 %); larger
  // meshes read with the normal policy (evict_first there evicts the halo lines
  // the neighbouring strip reads next: -22 % on config 4; profiles/README.md)
  static int l2_bytes = 0;
  if (l2_bytes == 0 && cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, g->dev) != cudaSuccess) {
    cudaGetLastError();
    l2_bytes = 126 << 20;
  }
  const bool small = 56.0 * (double)g->md.np < 2.0 * (double)l2_bytes;
  P.l2keep = g->l2keep >= 0 ? g->l2keep : (small ? 32 : 0);
  P.l2first = g->l2first >= 0 ? g->l2first : (small ? 63 : 0);
  const bool halo = g->slab && g->hx.G > 0;
  const int I = W - 4;
  const dim3 grid((g->md.HP + I - 1) / I, (y_end - y_begin + rows_per_cta - 1) / rows_per_cta);
  switch (L) {
#define X(l, w) \
  case l:       \
    return halo ? launch2_t<l, w, true>(g, P, grid, pdl) : launch2_t<l, w, false>(g, P, grid, pdl);
    PG_SWEEP2_CASES(X)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace pgb
