// Host side of the temporally blocked red-black SOR sweep: tensor maps,
// variant table, launch configuration (kernel: pg_sweep_fused.cuh; template
// instances: pg_sweep_fused_i*.cu, compiled in parallel).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "pg_sweep_fused.cuh"

namespace pgb {

cudaError_t launch_fused_inst_1(int key, pg_grid *g, const FusedParams &P, dim3 grid, bool *found);
cudaError_t launch_fused_inst_2(int key, pg_grid *g, const FusedParams &P, dim3 grid, bool *found);
cudaError_t launch_fused_inst_3(int key, pg_grid *g, const FusedParams &P, dim3 grid, bool *found);
cudaError_t launch_fused_inst_4(int key, pg_grid *g, const FusedParams &P, dim3 grid, bool *found);
cudaError_t launch_fused_inst_5(int key, pg_grid *g, const FusedParams &P, dim3 grid, bool *found);

// ------------------------------------------------------------------ host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 4-D view of a parity-split mesh array: (half-column, parity, row, layer),
// box {W half-columns, 2 parities, 1 row, L layers}
CUtensorMapL2promotion promo_of(int bytes) {
  switch (bytes) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 128: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

bool encode(CUtensorMap *m, const double *base, const MeshDims &d, int W, int promo) {
  auto fn = get_encoder();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)d.HP, 2, (cuuint64_t)d.NY, (cuuint64_t)d.L};
  cuuint64_t strides[3] = {(cuuint64_t)d.HP * 8, (cuuint64_t)d.NXP * 8, (cuuint64_t)d.layer_stride * 8};
  cuuint32_t box[4] = {(cuuint32_t)W, 2, 1, (cuuint32_t)d.L};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  promo_of(promo), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}


// 4-D view of a slab's ghost-row receive buffer: [L][G][NXP] parity-split rows
bool encode_rows(CUtensorMap *m, const double *base, const MeshDims &d, int G, int W, int promo) {
  auto fn = get_encoder();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)d.HP, 2, (cuuint64_t)G, (cuuint64_t)d.L};
  cuuint64_t strides[3] = {(cuuint64_t)d.HP * 8, (cuuint64_t)d.NXP * 8, (cuuint64_t)G * d.NXP * 8};
  cuuint32_t box[4] = {(cuuint32_t)W, 2, 1, (cuuint32_t)d.L};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  promo_of(promo), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

bool encode_halo_maps(pg_grid *g) {
  SlabHalo &h = g->hx;
  bool ok = true;
  for (int w = 0; w < 2; ++w) {
    if (h.has_lo) ok = ok && encode_rows(&h.mlo[w], h.recv_lo, g->md, h.G, w ? 64 : 32, g->l2promo);
    if (h.has_hi) ok = ok && encode_rows(&h.mhi[w], h.recv_hi, g->md, h.G, w ? 64 : 32, g->l2promo);
    if (h.p2p && h.has_lo) ok = ok && encode_rows(&h.mlo_b[w], h.recv_lo_b, g->md, h.G, w ? 64 : 32, g->l2promo);
    if (h.p2p && h.has_hi) ok = ok && encode_rows(&h.mhi_b[w], h.recv_hi_b, g->md, h.G, w ? 64 : 32, g->l2promo);
  }
  return ok;
}

// cycle counters of the instrumented build (-DPG_PROF), else null
unsigned long long *prof_buffer() {
#ifdef PG_PROF
  static unsigned long long *p = nullptr;
  if (!p) {
    cudaMalloc((void **)&p, sizeof(unsigned long long) * 8);
    cudaMemset(p, 0, sizeof(unsigned long long) * 8);
  }
  return p;
#else
  return nullptr;
#endif
}

int fused_exact_lanes(int F, int W) { return W - 2 * ((F + 1) & ~1); }

bool tma_available(pg_grid *g) {
  if (g->kind != 0) return false;
  if (g->tma_state == 0) {
    g->tma_state = -1;
    static_assert(sizeof(FusedParams) <= 4096, "kernel params too large");
    const double *bufs[7] = {g->V[0], g->V[1], g->gx, g->gy, g->gze, g->b, g->invd};
    bool ok = get_encoder() != nullptr;
    for (int w = 0; w < 2; ++w)
      for (int k = 0; ok && k < 7; ++k) ok = encode(&g->tmap[w][k], bufs[k], g->md, w ? 64 : 32, g->l2promo);
    if (ok) g->tma_state = 1;
  }
  return g->tma_state == 1;
}

int fused_default_stages(int L, int F, int D) {
  // D (F-1) + 4 resident rows + 2 prefetch stages
  return D * (F - 1) + 6;
}

bool fused_variant_exists(int L, int F, int S, int D, int W, bool slab) {
  if (slab) {
    switch (fused_key(L, F, S, D, W, true)) {
#define X(l, f, s, d, w) case fused_key(l, f, s, d, w, true):
      PG_FUSED_SLAB_CASES(X)
#undef X
      return true;
      default:
        return false;
    }
  }
  switch (fused_key(L, F, S, D, W)) {
#define X(l, f, s, d, w) case fused_key(l, f, s, d, w):
    PG_FUSED_CASES(X)
#undef X
    return true;
    default:
      return false;
  }
}

int fused_ctas_per_sm(int L, int S, int W) {
  const size_t smem = fused_smem(L, S, W) + 1024;
  int c = (int)((228 * 1024) / smem);
  return c < 1 ? 1 : c;
}

bool fill_fused_params(pg_grid *g, FusedParams &P, double omega, double tol, int j, int nsw, int W,
                       int rows_per_cta, int y_begin, int y_end, int ypar) {
  if (!tma_available(g)) return false;
  const CUtensorMap *tm = g->tmap[W == 64 ? 1 : 0];
  P.mV0 = tm[0];
  P.mV1 = tm[1];
  P.mgx = tm[2];
  P.mgy = tm[3];
  P.mgz = tm[4];
  P.mb = tm[5];
  P.mid = tm[6];
  P.V0 = g->V[0];
  P.V1 = g->V[1];
  P.NX = g->md.NX;
  P.NXP = g->md.NXP;
  P.HP = g->md.HP;
  P.NY = g->md.NY;
  P.y_begin = y_begin;
  P.y_end = y_end;
  P.ypar = ypar & 1;
  P.layer_stride = g->md.layer_stride;
  P.omega = omega;
  P.tol = tol;
  P.ctl = g->ctl;
  P.rows_per_cta = rows_per_cta;
  P.launch_idx = j;
  P.nsw = nsw;
  P.prof = prof_buffer();
  P.pre = 0;
  P.p2p = 0;
  P.nranks = 1;
  const SlabHalo &h = g->hx;
  const bool halo = g->slab && h.G > 0;
  P.has_rlo = halo && h.has_lo;
  P.has_rhi = halo && h.has_hi;
  P.G = h.G;
  P.send_lo = halo && h.has_lo ? h.send_lo : nullptr;
  P.send_hi = halo && h.has_hi ? h.send_hi : nullptr;
  if (P.has_rlo) P.mRlo = h.mlo[W == 64 ? 1 : 0];
  if (P.has_rhi) P.mRhi = h.mhi[W == 64 ? 1 : 0];
  return true;
}

cudaError_t launch_rb_sweep_fused(pg_grid *g, double omega, double tol, int j, int nsw, int F,
                                  int S, int D, int W, int rows_per_cta, int y_begin, int y_end,
                                  int ypar) {
  FusedParams P;
  if (!fill_fused_params(g, P, omega, tol, j, nsw, W, rows_per_cta, y_begin, y_end, ypar))
    return cudaErrorNotSupported;
  const bool halo = g->slab && g->hx.G > 0;
  const int strips = (g->md.HP + fused_exact_lanes(F, W) - 1) / fused_exact_lanes(F, W);
  const dim3 grid(strips, (y_end - y_begin + rows_per_cta - 1) / rows_per_cta);
  const int key = fused_key(g->md.L, F, S, D, W, halo);
  bool found = false;
  cudaError_t e = launch_fused_inst_1(key, g, P, grid, &found);
  if (!found) e = launch_fused_inst_2(key, g, P, grid, &found);
  if (!found) e = launch_fused_inst_3(key, g, P, grid, &found);
  if (!found) e = launch_fused_inst_4(key, g, P, grid, &found);
  if (!found) e = launch_fused_inst_5(key, g, P, grid, &found);
  return found ? e : cudaErrorInvalidValue;
}

}  // namespace pgb

#ifdef PG_PROF
extern "C" PG_API int pg_debug_prof(unsigned long long *out8, int reset) {
  unsigned long long *p = pgb::prof_buffer();
  cudaMemcpy(out8, p, sizeof(unsigned long long) * 8, cudaMemcpyDeviceToHost);
  if (reset) cudaMemset(p, 0, sizeof(unsigned long long) * 8);
  return 0;
}
#endif
