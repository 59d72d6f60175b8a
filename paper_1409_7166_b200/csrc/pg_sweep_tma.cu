// Shared-memory-staged streaming red-black SOR sweep (sm_100a).
//
// Same arithmetic and ordering as k_rb_sweep (Eq. (13) in red-black numbering
// + SOR Eq. (15), one full sweep = red then black, single pass over y), but the
// rows of all six per-node arrays (V, gx, gy, gz_eff, b, 1/d) of a CTA's strip
// are staged in a shared-memory ring of S row-stages, S-4 rows ahead of use:
//   MODE 1 (TMA): one elected thread issues cp.async.bulk.tensor boxes
//          {64 x, 1 y, L layers} per array with mbarrier completion; TMA's
//          out-of-bounds zero fill supplies halos and rows outside [0, NY).
//   MODE 2 (LDGSTS): every thread copies its own x-pair of each array with
//          cp.async (16 B, zero fill when out of range); cp.async groups, one
//          per row, give the completion order.
// The via conductance of the layer below comes from the same stage (no second
// global load of gz) and every neighbour value comes from shared memory, with
// one __syncthreads per row.
// CTA = 32 lanes x L warps; lane q owns the x-pair q of the strip, lanes 0/31
// are halo pairs (recomputed, never stored); strip s covers pairs
// [30 s - 1, 30 s + 31).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "pg_internal.h"

namespace pgb {

namespace {

constexpr int kArrays = 6;  // V, gx, gy, gz, b, id
constexpr int kRowElems = 64;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
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
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
  const int n = valid ? 16 : 0;  // src-size 0 -> zero fill, source not read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ unsigned long long d2u(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double u2d(unsigned long long x) {
  return __longlong_as_double(static_cast<long long>(x));
}

struct StagedParams {
  CUtensorMap mV0, mV1, mgx, mgy, mgz, mb, mid;  // 64-B aligned members (MODE 1)
  double *V0, *V1;
  const double *gx, *gy, *gz, *b, *id;           // MODE 2
  MeshDims d;
  double omega, tol;
  DevCtl *ctl;
  int32_t rows_per_cta;
  int32_t stages;
  int32_t launch_idx;
};

}  // namespace

// SC: compile-time stage count for MODE 2 (cp.async.wait_group needs an immediate)
template <int MODE, int SC>
__global__ void __launch_bounds__(256) k_rb_sweep_staged(const __grid_constant__ StagedParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[16];
  __shared__ double wmax[kMaxLayers];
  const int lane = threadIdx.x, l = threadIdx.y, L = P.d.L;
  const bool leader = lane == 0 && l == 0;
  DevCtl *ctl = P.ctl;
  const int j = P.launch_idx;

  // ---- device-side convergence: uniform early exit of queued launches
  if (*(volatile int32_t *)&ctl->done) return;
  if (j > 0) {
    const double prev = u2d(*(volatile unsigned long long *)&ctl->dmax[(j - 1) & (kRing - 1)]);
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
  const double *Vin = par ? P.V1 : P.V0;
  double *Vout = par ? P.V0 : P.V1;

  const int S = MODE == 2 ? SC : P.stages;
  const int lay = L * kRowElems;  // doubles per array per stage
  const int stage_elems = kArrays * lay;
  double *ring = reinterpret_cast<double *>(smem_raw);
  const uint32_t stage_bytes = (uint32_t)stage_elems * 8u;

  const int x0 = 2 * (blockIdx.x * kInterior - 1);  // global x of local element 0 (may be -2)
  const int ys = blockIdx.y * P.rows_per_cta;
  const int ye = min(ys + P.rows_per_cta, P.d.NY);
  const int r_first = ys - 2, r_last = ye + 1;  // rows staged: row r <-> stage (r - r_first) % S

  if (MODE == 1 && leader) {
    for (int s = 0; s < S; ++s) mbar_init(&full_bar[s], 1);
    fence_mbar_init();
  }
  if (MODE == 1) __syncthreads();

  auto issue_tma = [&](int r) {  // leader only
    const int s = (r - r_first) % S;
    double *st = ring + (size_t)s * stage_elems;
    mbar_expect_tx(&full_bar[s], stage_bytes);
    tma_load_3d(st + 0 * lay, mVin, &full_bar[s], x0, r, 0);
    tma_load_3d(st + 1 * lay, &P.mgx, &full_bar[s], x0, r, 0);
    tma_load_3d(st + 2 * lay, &P.mgy, &full_bar[s], x0, r, 0);
    tma_load_3d(st + 3 * lay, &P.mgz, &full_bar[s], x0, r, 0);
    tma_load_3d(st + 4 * lay, &P.mb, &full_bar[s], x0, r, 0);
    tma_load_3d(st + 5 * lay, &P.mid, &full_bar[s], x0, r, 0);
  };
  const int gx_own = x0 + 2 * lane;
  auto issue_async = [&](int r) {  // every thread: its own pair of each array; one group per row
    if (r <= r_last) {
      const int s = (r - r_first) % S;
      double *st = ring + (size_t)s * stage_elems + l * kRowElems + 2 * lane;
      const bool ok = r >= 0 && r < P.d.NY && gx_own >= 0 && gx_own < P.d.NXP;
      const int64_t o = ok ? (int64_t)l * P.d.layer_stride + (int64_t)r * P.d.NXP + gx_own : 0;
      cp_async16(st + 0 * lay, Vin + o, ok);
      cp_async16(st + 1 * lay, P.gx + o, ok);
      cp_async16(st + 2 * lay, P.gy + o, ok);
      cp_async16(st + 3 * lay, P.gz + o, ok);
      cp_async16(st + 4 * lay, P.b + o, ok);
      cp_async16(st + 5 * lay, P.id + o, ok);
    }
    cp_async_commit();  // possibly empty group: keeps group k <-> row r_first + k
  };
  auto wait_row_tma = [&](int r) {
    const int k = r - r_first;
    mbar_wait(&full_bar[k % S], (uint32_t)((k / S) & 1));
  };

  // ---- prologue: fill the ring
  if (MODE == 1) {
    if (leader)
      for (int r = r_first; r < r_first + S && r <= r_last; ++r) issue_tma(r);
    wait_row_tma(ys - 2);
    wait_row_tma(ys - 1);
    wait_row_tma(ys);
  } else {
    for (int r = r_first; r < r_first + S; ++r) issue_async(r);
    cp_async_wait<SC - 3>();  // rows ys-2, ys-1, ys (groups 0..2) landed
    __syncthreads();
  }

  const double w = P.omega;
  const int q = lane;
  const int gxp = x0 + 2 * q;  // global x of my pair
  const bool interior = lane >= 1 && lane <= kInterior && gxp >= 0 && gxp < P.d.NXP;
  double dmax = 0.0;

  auto row_ptr = [&](int r, int arr) -> double * {
    const int s = (r - r_first) % S;
    return ring + (size_t)s * stage_elems + arr * lay;
  };

  for (int y = ys - 1; y <= ye; ++y) {
    // row y+1 must be present: TMA -> barrier of its stage; LDGSTS -> own copies
    // (groups committed so far: S + max(0, y - ys - 1); row y+1 is group y+3-ys)
    if (MODE == 1) wait_row_tma(y + 1);
    else cp_async_wait<SC - 5>();
    const int er = (l + y) & 1;
    // ------------------------------------------------------------ red(y)
    {
      const int xr = 2 * q + er;
      const int xw = max(xr - 1, 0), xe = min(xr + 1, kRowElems - 1);
      double *Vy = row_ptr(y, 0) + l * kRowElems;
      const double *Vn = row_ptr(y - 1, 0) + l * kRowElems;
      const double *Vs = row_ptr(y + 1, 0) + l * kRowElems;
      const double *gxy = row_ptr(y, 1) + l * kRowElems;
      const double *gyy = row_ptr(y, 2) + l * kRowElems;
      const double *gyn = row_ptr(y - 1, 2) + l * kRowElems;
      const double *gzy = row_ptr(y, 3);
      const double by = row_ptr(y, 4)[l * kRowElems + xr];
      const double idy = row_ptr(y, 5)[l * kRowElems + xr];
      const double Vc = Vy[xr];
      double s = by;
      s = fma(gxy[xw], Vy[xw], s);
      s = fma(gxy[xr], Vy[xe], s);
      s = fma(gyn[xr], Vn[xr], s);
      s = fma(gyy[xr], Vs[xr], s);
      if (l + 1 < L) s = fma(gzy[l * kRowElems + xr], Vy[kRowElems + xr], s);
      if (l > 0) s = fma(gzy[(l - 1) * kRowElems + xr], Vy[xr - kRowElems], s);
      double vn = fma(w, s * idy - Vc, Vc);
      const bool xok = gxp + er < P.d.NX && gxp + er >= 0;
      if (!xok) vn = Vc;
      Vy[xr] = vn;
      if (interior && xok && y >= ys && y < ye) dmax = fmax(dmax, fabs(vn - Vc));
    }
    if (MODE == 1) fence_proxy_async();  // generic smem writes before later TMA refills
    __syncthreads();
    // all threads finished iteration y-1 -> the stage of row y-3 is free: refill
    if (MODE == 1) {
      if (leader && y - 3 >= r_first && y - 3 + S <= r_last) issue_tma(y - 3 + S);
    } else if (y >= ys + 1) {
      issue_async(y - 3 + S);
    }
    // ---------------------------------------------------------- black(y-1)
    if (y - 1 >= ys) {
      const int xb = 2 * q + er;  // black element of row y-1
      const int xw = max(xb - 1, 0), xe = min(xb + 1, kRowElems - 1);
      double *Vm = row_ptr(y - 1, 0) + l * kRowElems;
      const double *Vn = row_ptr(y - 2, 0) + l * kRowElems;
      const double *Vs = row_ptr(y, 0) + l * kRowElems;
      const double *gxm = row_ptr(y - 1, 1) + l * kRowElems;
      const double *gym = row_ptr(y - 1, 2) + l * kRowElems;
      const double *gyn = row_ptr(y - 2, 2) + l * kRowElems;
      const double *gzm = row_ptr(y - 1, 3);
      const double bm = row_ptr(y - 1, 4)[l * kRowElems + xb];
      const double idm = row_ptr(y - 1, 5)[l * kRowElems + xb];
      const double Vc = Vm[xb];
      double s = bm;
      s = fma(gxm[xw], Vm[xw], s);
      s = fma(gxm[xb], Vm[xe], s);
      s = fma(gyn[xb], Vn[xb], s);
      s = fma(gym[xb], Vs[xb], s);
      if (l + 1 < L) s = fma(gzm[l * kRowElems + xb], Vm[kRowElems + xb], s);
      if (l > 0) s = fma(gzm[(l - 1) * kRowElems + xb], Vm[xb - kRowElems], s);
      double vn = fma(w, s * idm - Vc, Vc);
      const bool xok = gxp + er < P.d.NX && gxp + er >= 0;
      if (!xok) vn = Vc;
      Vm[xb] = vn;
      if (MODE == 1) fence_proxy_async();
      if (interior && xok) dmax = fmax(dmax, fabs(vn - Vc));
      if (interior) {
        const double2 v2 = *reinterpret_cast<const double2 *>(Vm + 2 * q);
        *reinterpret_cast<double2 *>(Vout + (int64_t)l * P.d.layer_stride + (int64_t)(y - 1) * P.d.NXP +
                                     gxp) = v2;
      }
    }
  }
  if (MODE == 2) cp_async_wait<0>();
  // reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) wmax[l] = dmax;
  __syncthreads();
  if (leader) {
    double m = 0.0;
    for (int k = 0; k < L; ++k) m = fmax(m, wmax[k]);
    atomicMax(&ctl->dmax[j & (kRing - 1)], d2u(m));
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
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

static bool encode(CUtensorMap *m, const double *base, const MeshDims &d) {
  auto fn = get_encoder();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)d.NXP, (cuuint64_t)d.NY, (cuuint64_t)d.L};
  cuuint64_t strides[2] = {(cuuint64_t)d.NXP * 8, (cuuint64_t)d.layer_stride * 8};
  cuuint32_t box[3] = {(cuuint32_t)kRowElems, 1, (cuuint32_t)d.L};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int tma_ctas_per_sm(int L) { return L <= 2 ? 4 : (L <= 4 ? 2 : 1); }

static int default_stages(int L) {
  // ring of S stages x 6 arrays x L layers x 64 doubles; keep 2 CTAs/SM when L <= 4
  if (L <= 2) return 12;
  if (L <= 4) return 8;
  return 6;
}

int tma_stages_for(const pg_grid *g) {
  int S = g->stages > 0 ? g->stages : default_stages(g->md.L);
  if (g->kernel == 2) S = S >= 8 ? 8 : 6;  // compiled variants
  const size_t per = (size_t)kArrays * g->md.L * kRowElems * 8;
  while (S > 6 && S * per > 220 * 1024) S -= (g->kernel == 2 ? 2 : 1);  // 227 KB opt-in limit
  return S;
}

static size_t staged_smem_bytes(const pg_grid *g) {
  return (size_t)tma_stages_for(g) * kArrays * g->md.L * kRowElems * 8;
}

bool tma_available(pg_grid *g) {
  if (g->kind != 0) return false;
  if (g->tma_state == 0) {
    g->tma_state = -1;
    static_assert(sizeof(StagedParams) <= 4096, "kernel params too large");
    const MeshDims &d = g->md;
    const double *bufs[7] = {g->V[0], g->V[1], g->gx, g->gy, g->gze, g->b, g->invd};
    bool ok = get_encoder() != nullptr;
    for (int k = 0; ok && k < 7; ++k) ok = encode(&g->tmap[k], bufs[k], d);
    if (ok) g->tma_state = 1;
  }
  return g->tma_state == 1;
}

template <class K>
static cudaError_t set_smem(pg_grid *g, K kern, size_t smem) {
  if (smem != g->tma_smem_set || g->tma_kernel_set != (const void *)kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
    g->tma_smem_set = smem;
    g->tma_kernel_set = (const void *)kern;
  }
  return cudaSuccess;
}

cudaError_t launch_rb_sweep_tma(pg_grid *g, double omega, double tol, int j, int rows_per_cta) {
  StagedParams P;
  const MeshDims &d = g->md;
  P.mV0 = g->tmap[0];
  P.mV1 = g->tmap[1];
  P.mgx = g->tmap[2];
  P.mgy = g->tmap[3];
  P.mgz = g->tmap[4];
  P.mb = g->tmap[5];
  P.mid = g->tmap[6];
  P.V0 = g->V[0];
  P.V1 = g->V[1];
  P.gx = g->gx;
  P.gy = g->gy;
  P.gz = g->gze;
  P.b = g->b;
  P.id = g->invd;
  P.d = d;
  P.omega = omega;
  P.tol = tol;
  P.ctl = g->ctl;
  P.rows_per_cta = rows_per_cta;
  P.stages = tma_stages_for(g);
  P.launch_idx = j;
  const int pairs = d.NXP / 2;
  const int strips = (pairs + kInterior - 1) / kInterior;
  dim3 grid(strips, (d.NY + rows_per_cta - 1) / rows_per_cta);
  dim3 block(kLanes, d.L);
  const size_t smem = staged_smem_bytes(g);
  cudaError_t e;
  if (g->kernel == 2) {
    if (P.stages == 8) {
      if ((e = set_smem(g, k_rb_sweep_staged<2, 8>, smem)) != cudaSuccess) return e;
      k_rb_sweep_staged<2, 8><<<grid, block, smem, g->stream>>>(P);
    } else {
      if ((e = set_smem(g, k_rb_sweep_staged<2, 6>, smem)) != cudaSuccess) return e;
      k_rb_sweep_staged<2, 6><<<grid, block, smem, g->stream>>>(P);
    }
  } else {
    if ((e = set_smem(g, k_rb_sweep_staged<1, 0>, smem)) != cudaSuccess) return e;
    k_rb_sweep_staged<1, 0><<<grid, block, smem, g->stream>>>(P);
  }
  return cudaGetLastError();
}

}  // namespace pgb
