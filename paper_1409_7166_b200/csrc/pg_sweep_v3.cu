// Optimised TMA-staged streaming red-black SOR sweep (sm_100a) -- the default
// mesh sweep ("kernel" option 3).
//
// Arithmetic and ordering are those of k_rb_sweep (Eq. (13) in red-black
// numbering + SOR Eq. (15); one full sweep = red then black in a single pass
// over y).  Rows of the six per-node arrays (V, gx, gy, gz_eff, b, 1/d) of a
// CTA's strip are staged by TMA (cp.async.bulk.tensor, boxes {64 x, 1 y, L})
// into a ring of S row-stages with mbarrier completion, S-4 rows ahead of use
// (S = 6 by default).
// Compared with k_rb_sweep_staged this version is built for instruction count:
//   * L (layers) and S (ring depth) are template parameters, so ring indexing
//     is a constant modulo and all array offsets are immediates;
//   * each thread keeps one precomputed column offset; every neighbour is a
//     fixed displacement from it (+-1 in x, +-64 across layers, other stages
//     for y +- 1); the ring has 64-double guard bands so no read is clamped
//     (out-of-strip reads only feed halo results that are never used);
//   * the neighbour sum is split in two partial sums (shorter FMA chain).
// CTA = 32 lanes x L warps; lane q owns x-pair q of the strip; lanes 0/31 are
// halo pairs (recomputed, never stored); strip s covers pairs [30 s - 1, 30 s + 31).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "pg_internal.h"

namespace pgb {

namespace {

constexpr int kRow = 64;   // doubles per layer row of a strip
constexpr int kGuard = 64; // guard band (doubles) before and after the ring

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(0)
      : "memory");
}

struct V3Params {
  CUtensorMap mV0, mV1, mgx, mgy, mgz, mb, mid;
  double *V0, *V1;
  int32_t NX, NXP, NY;
  int64_t layer_stride;
  double omega, tol;
  DevCtl *ctl;
  int32_t rows_per_cta;
  int32_t launch_idx;
};

}  // namespace

template <int L, int S>
__global__ void __launch_bounds__(32 * L) k_rb_sweep_v3(const __grid_constant__ V3Params P) {
  static_assert(S >= 6, "ring needs >= 6 stages (4 resident rows + lookahead)");
  constexpr int LAY = L * kRow;       // doubles per array per stage
  constexpr int SE = 6 * LAY;         // doubles per stage
  constexpr int GX = 1 * LAY, GY = 2 * LAY, GZ = 3 * LAY, BB = 4 * LAY, ID = 5 * LAY;
  constexpr uint32_t STAGE_BYTES = SE * 8u;
  extern __shared__ __align__(128) double smem_v3[];
  __shared__ uint64_t full_bar[S];
  __shared__ double wmax[L];
  double *ring = smem_v3 + kGuard;

  const int lane = threadIdx.x, l = threadIdx.y;
  const bool leader = lane == 0 && l == 0;
  DevCtl *ctl = P.ctl;
  const int j = P.launch_idx;

  if (*(volatile int32_t *)&ctl->done) return;
  if (j > 0) {
    const double prev = __longlong_as_double(
        (long long)(*(volatile unsigned long long *)&ctl->dmax[(j - 1) & (kRing - 1)]));
    if (prev < P.tol) {
      if (blockIdx.x == 0 && blockIdx.y == 0 && leader) {
        ctl->done = 1;
        ctl->launches_done = j;
      }
      return;
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && leader) ctl->dmax[(j + 1) & (kRing - 1)] = 0ull;

  const int par = (*(volatile int32_t *)&ctl->base + j) & 1;
  const CUtensorMap *mVin = par ? &P.mV1 : &P.mV0;
  double *Vout = par ? P.V0 : P.V1;

  const int x0 = 2 * (blockIdx.x * kInterior - 1);
  const int ys = blockIdx.y * P.rows_per_cta;
  const int ye = min(ys + P.rows_per_cta, P.NY);
  const int r_first = ys - 2, r_last = ye + 1;

  // guard bands (never written by TMA) and barriers
  {
    const int t = l * 32 + lane;
    for (int k = t; k < kGuard; k += 32 * L) {
      smem_v3[k] = 0.0;
      ring[S * SE + k] = 0.0;
    }
  }
  if (leader) {
    for (int s = 0; s < S; ++s) mbar_init(&full_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int r) {
    const int s = (r - r_first) % S;
    double *st = ring + s * SE;
    mbar_expect_tx(&full_bar[s], STAGE_BYTES);
    tma3(st, mVin, &full_bar[s], x0, r);
    tma3(st + GX, &P.mgx, &full_bar[s], x0, r);
    tma3(st + GY, &P.mgy, &full_bar[s], x0, r);
    tma3(st + GZ, &P.mgz, &full_bar[s], x0, r);
    tma3(st + BB, &P.mb, &full_bar[s], x0, r);
    tma3(st + ID, &P.mid, &full_bar[s], x0, r);
  };
  auto wait_row = [&](int r) {
    const int k = r - r_first;
    mbar_wait(&full_bar[k % S], (uint32_t)((k / S) & 1));
  };
  if (leader)
    for (int r = r_first; r < r_first + S && r <= r_last; ++r) issue(r);

  const double w = P.omega;
  const int col = l * kRow + 2 * lane;             // my pair's offset inside an array block
  const int gxp = x0 + 2 * lane;                   // global x of my pair
  const bool interior = lane >= 1 && lane <= kInterior && gxp >= 0 && gxp < P.NXP;
  const bool ok0 = gxp >= 0 && gxp < P.NX;
  const bool ok1 = gxp + 1 >= 0 && gxp + 1 < P.NX;
  const bool has_down = l > 0;
  double *vout_col = Vout + (int64_t)l * P.layer_stride + gxp;
  double dmax = 0.0;

  wait_row(ys - 2);
  wait_row(ys - 1);
  wait_row(ys);
  for (int y = ys - 1; y <= ye; ++y) {
    wait_row(y + 1);
    const int er = (l + y) & 1;
    const bool okr = er ? ok1 : ok0;
    const int xr = col + er;
    double *Ry = ring + ((y - r_first) % S) * SE;
    double *Rn = ring + ((y - 1 - r_first) % S) * SE;
    const double *Rs = ring + ((y + 1 - r_first) % S) * SE;
    // ------------------------------------------------ red(y): black_old neighbours
    {
      double *v = Ry + xr;
      const double Vc = v[0];
      double s1 = fma(Ry[GX + xr - 1], v[-1], Ry[BB + xr]);
      s1 = fma(Ry[GX + xr], v[1], s1);
      s1 = fma(Rn[GY + xr], Rn[xr], s1);
      double s2 = Ry[GY + xr] * Rs[xr];
      s2 = fma(Ry[GZ + xr], v[kRow], s2);
      if (has_down) s2 = fma(Ry[GZ + xr - kRow], v[-kRow], s2);
      double vn = fma(w, (s1 + s2) * Ry[ID + xr] - Vc, Vc);
      vn = okr ? vn : Vc;
      v[0] = vn;
      const bool cnt = interior && okr && y >= ys && y < ye;
      dmax = fmax(dmax, cnt ? fabs(vn - Vc) : 0.0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (leader && y - 3 >= r_first && y - 3 + S <= r_last) issue(y - 3 + S);
    // ------------------------------------------------ black(y-1): red_new neighbours
    if (y - 1 >= ys) {
      const double *Rm = ring + ((y - 2 - r_first) % S) * SE;  // row y-2
      double *v = Rn + xr;  // black element of row y-1 sits at the same offset
      const double Vc = v[0];
      double s1 = fma(Rn[GX + xr - 1], v[-1], Rn[BB + xr]);
      s1 = fma(Rn[GX + xr], v[1], s1);
      s1 = fma(Rm[GY + xr], Rm[xr], s1);
      double s2 = Rn[GY + xr] * Ry[xr];
      s2 = fma(Rn[GZ + xr], v[kRow], s2);
      if (has_down) s2 = fma(Rn[GZ + xr - kRow], v[-kRow], s2);
      double vn = fma(w, (s1 + s2) * Rn[ID + xr] - Vc, Vc);
      vn = okr ? vn : Vc;
      v[0] = vn;
      dmax = fmax(dmax, (interior && okr) ? fabs(vn - Vc) : 0.0);
      if (interior) {
        const double2 v2 = *reinterpret_cast<const double2 *>(Rn + col);
        *reinterpret_cast<double2 *>(vout_col + (int64_t)(y - 1) * P.NXP) = v2;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) wmax[l] = dmax;
  __syncthreads();
  if (leader) {
    double m = 0.0;
#pragma unroll
    for (int k = 0; k < L; ++k) m = fmax(m, wmax[k]);
    atomicMax(&ctl->dmax[j & (kRing - 1)], static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// ------------------------------------------------------------------ host side
template <int L, int S>
static cudaError_t launch_v3_t(pg_grid *g, const V3Params &P, dim3 grid) {
  auto kern = k_rb_sweep_v3<L, S>;
  const size_t smem = ((size_t)S * 6 * L * kRow + 2 * kGuard) * 8;
  if (g->tma_kernel_set != (const void *)kern || g->tma_smem_set != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
    g->tma_kernel_set = (const void *)kern;
    g->tma_smem_set = smem;
  }
  kern<<<grid, dim3(32, L), smem, g->stream>>>(P);
  return cudaGetLastError();
}

int v3_stages(const pg_grid *g) {
  // 6 stages (default): 4 resident rows + 2 in flight; the smaller ring lets 3
  // CTAs (12 warps) share an SM at L = 4, which hides more shared-memory and
  // FP64 latency than a deeper ring (measured on config 1, profiles/README.md)
  if (g->stages >= 16 && g->md.L <= 4) return 16;
  if (g->stages == 8) return 8;
  return 6;
}

int v3_ctas_per_sm(const pg_grid *g) {
  const size_t smem = ((size_t)v3_stages(g) * 6 * g->md.L * kRow + 2 * kGuard) * 8 + 1024;
  int c = (int)((228 * 1024) / smem);
  return c < 1 ? 1 : c;
}

cudaError_t launch_rb_sweep_v3(pg_grid *g, double omega, double tol, int j, int rows_per_cta) {
  if (!tma_available(g)) return cudaErrorNotSupported;
  V3Params P;
  P.mV0 = g->tmap[0];
  P.mV1 = g->tmap[1];
  P.mgx = g->tmap[2];
  P.mgy = g->tmap[3];
  P.mgz = g->tmap[4];
  P.mb = g->tmap[5];
  P.mid = g->tmap[6];
  P.V0 = g->V[0];
  P.V1 = g->V[1];
  P.NX = g->md.NX;
  P.NXP = g->md.NXP;
  P.NY = g->md.NY;
  P.layer_stride = g->md.layer_stride;
  P.omega = omega;
  P.tol = tol;
  P.ctl = g->ctl;
  P.rows_per_cta = rows_per_cta;
  P.launch_idx = j;
  const int strips = (g->md.NXP / 2 + kInterior - 1) / kInterior;
  const dim3 grid(strips, (g->md.NY + rows_per_cta - 1) / rows_per_cta);
  const int S = v3_stages(g);
  switch (g->md.L * 100 + S) {
    case 108: return launch_v3_t<1, 8>(g, P, grid);
    case 208: return launch_v3_t<2, 8>(g, P, grid);
    case 308: return launch_v3_t<3, 8>(g, P, grid);
    case 408: return launch_v3_t<4, 8>(g, P, grid);
    case 508: return launch_v3_t<5, 8>(g, P, grid);
    case 608: return launch_v3_t<6, 8>(g, P, grid);
    case 708: return launch_v3_t<7, 8>(g, P, grid);
    case 808: return launch_v3_t<8, 8>(g, P, grid);
    case 106: return launch_v3_t<1, 6>(g, P, grid);
    case 206: return launch_v3_t<2, 6>(g, P, grid);
    case 306: return launch_v3_t<3, 6>(g, P, grid);
    case 406: return launch_v3_t<4, 6>(g, P, grid);
    case 506: return launch_v3_t<5, 6>(g, P, grid);
    case 606: return launch_v3_t<6, 6>(g, P, grid);
    case 706: return launch_v3_t<7, 6>(g, P, grid);
    case 806: return launch_v3_t<8, 6>(g, P, grid);
    case 116: return launch_v3_t<1, 16>(g, P, grid);
    case 216: return launch_v3_t<2, 16>(g, P, grid);
    case 316: return launch_v3_t<3, 16>(g, P, grid);
    case 416: return launch_v3_t<4, 16>(g, P, grid);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pgb
