// Temporally blocked red-black SOR: F sweeps per streaming pass (sm_100a) --
// the mesh relaxation kernel (options "fuse" = F, "lag" = D, "stages" = S).
//
// Arithmetic per node update is Eq. (13) with the SOR blend of Eq. (15)
// (§IV), in the red-black numbering (R12): a full sweep is
// all red nodes from old black values, then all black nodes from new red
// values.  One launch performs `nsw` <= F such sweeps and writes the result of
// the last one, so the per-node HBM stream (V read + write, gx, gy, gz_eff, b,
// 1/d: 56 B) is paid once per F sweeps instead of once per sweep.
//
// Geometry.  A CTA owns a strip of 32 x-pairs (64 columns) x L layers x a chunk
// of rows [ys, ye); lane q of warp l owns the pair (2(ps+q), 2(ps+q)+1) of
// layer l (ps even: TMA boxes must start 16-byte aligned).  The rows [ys - 2F, ye + 2F) of all six arrays are streamed through
// a shared-memory ring of S row-stages by TMA (cp.async.bulk.tensor, one 4-D
// box {32 half-columns, 2 parities, 1 row, L layers} per array in the
// parity-split storage layout of pg_internal.h, so a stage holds, per array and
// layer, the 32 even columns then the 32 odd columns; out-of-range rows and
// columns are zero filled), and every sweep level updates the staged rows in
// place.  All nodes a warp updates in one phase have the same column parity,
// so every shared-memory access of the update is 32 consecutive doubles.
// Every half-sweep makes one more node at each strip edge and one more row at
// each chunk edge stale,
// so after F sweeps the lanes [F, 32 - F) and the rows [ys, ye) are exact (the
// x halo is rounded up to an even FH >= F lanes per side); only
// those are written back (to the other buffer of the V ping-pong pair) and
// counted in the convergence norm.
//
// Wavefront.  Level f (sweep f of the pass) trails level f - 1 by D rows.  In
// streaming step y a warp performs
//     phase A: red_f(y - D f)          for f = 0..nsw-1
//     phase B: black_f(y - D f - 1)    for f = 0..nsw-1, then writes row
//              y - D (nsw-1) - 1 of its layer (both colours final) to HBM.
// red_f(r) reads black_{f-1} of rows r-1..r+1, which the previous steps
// produced (D >= 3), and black_f(r) reads red_f of rows r-1..r+1, produced in
// phase A of this step or before; every value is overwritten only after its
// last reader ran.  Layers are coupled by vias (other warps), so phases are
// separated by __syncthreads: D = 3 needs a barrier after each phase, D = 4
// only between A and B (phase B(y) and phase A(y+1) touch disjoint values).
// Ring: the rows read in one step span D (F-1) + 4 rows; the remaining
// S - D(F-1) - 4 stages are TMA prefetch depth.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "pg_internal.h"

namespace pgb {

namespace {

constexpr int kRow = 64;    // doubles per layer row of a strip
constexpr int kGuard = 64;  // zeroed guard band (doubles) before and after the ring

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
// box {32 half-columns from c0, both parities, row y, all layers}
__device__ __forceinline__ void tma4(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int y) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(0), "r"(y), "r"(0)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace

// Optional cycle instrumentation (build with -DPG_PROF; debugging only):
// per-warp clock sums of the streaming-step phases, read by pg_debug_prof.
#ifdef PG_PROF
__device__ unsigned long long g_prof[8];
#define PROF_T(var) const long long var = clock64()
#define PROF_ADD(k, a, b) prof[k] += (unsigned long long)((b) - (a))
#else
#define PROF_T(var)
#define PROF_ADD(k, a, b)
#endif

struct FusedParams {
  CUtensorMap mV0, mV1, mgx, mgy, mgz, mb, mid;
  double *V0, *V1;
  int32_t NX, NXP, HP, NY;
  int32_t y_begin, y_end;   // rows updated/written: [y_begin, y_end) (slab: ghost rows outside)
  int32_t ypar;             // parity of the global row offset (red = (l + y + ypar + x) even)
  int64_t layer_stride;
  double omega, tol;
  DevCtl *ctl;
  int32_t rows_per_cta;
  int32_t launch_idx;
  int32_t nsw;              // sweeps in this launch, 1..F
};

// One red-black node update (Eq. (13) + (15)) of the node at offset `me` of
// row stage Ry (row r-1 in Rn, row r+1 in Rs); `ow`/`oe` are the offsets of
// its west/east neighbours (other parity half of the same layer row).
// Returns the new value; the caller stores it (the stores of all levels of a
// phase are issued after all their loads, so the levels' dependency chains
// overlap: the compiler cannot reorder a shared store before a later load).
// Padding columns (x >= NX) and out-of-grid columns (TMA zero fill) have
// V = b = 1/d = 0 and zero conductances, so the update leaves them at 0 and
// needs no mask.
template <int L>
__device__ __forceinline__ double node_update(const double *Ry, const double *Rn, const double *Rs,
                                              int me, int ow, int oe, double w, bool has_down,
                                              double &Vc) {
  constexpr int LAY = L * kRow;
  constexpr int GX = 1 * LAY, GY = 2 * LAY, GZ = 3 * LAY, BB = 4 * LAY, ID = 5 * LAY;
  Vc = Ry[me];
  double s1 = fma(Ry[GX + ow], Ry[ow], Ry[BB + me]);      // west link g(x-1,x) + K_i (b)
  s1 = fma(Ry[GX + me], Ry[oe], s1);                      // east link g(x,x+1)
  s1 = fma(Rn[GY + me], Rn[me], s1);                      // north (row r-1)
  double s2 = Ry[GY + me] * Rs[me];                       // south (row r+1)
  s2 = fma(Ry[GZ + me], Ry[me + kRow], s2);               // via up (layer l+1)
  if (has_down) s2 = fma(Ry[GZ + me - kRow], Ry[me - kRow], s2);  // via down (layer l-1)
  return fma(w, (s1 + s2) * Ry[ID + me] - Vc, Vc);
}

template <int L, int F, int S, int D>
__global__ void __launch_bounds__(32 * L) k_rb_sweep_fused(const __grid_constant__ FusedParams P) {
  static_assert(D >= 3, "levels must trail by >= 3 rows");
  static_assert(S >= D * (F - 1) + 5, "ring too small for the wavefront");
  constexpr int LAY = L * kRow;
  constexpr int SE = 6 * LAY;  // doubles per stage
  constexpr int GX = 1 * LAY, GY = 2 * LAY, GZ = 3 * LAY, BB = 4 * LAY, ID = 5 * LAY;
  constexpr uint32_t STAGE_BYTES = SE * 8u;
  // x halo: F pairs per side suffice; it is rounded up to even so that the TMA
  // box starts on a 16-byte boundary (odd pair offsets fault)
  constexpr int FH = (F + 1) & ~1;
  constexpr int I = 32 - 2 * FH;  // exact lanes per strip
  extern __shared__ __align__(128) double smem_f[];
  __shared__ uint64_t full_bar[S];
  __shared__ double wmax[L];
  double *ring = smem_f + kGuard;

  const int lane = threadIdx.x, l = threadIdx.y;
  const bool leader = lane == 0 && l == 0;
  DevCtl *ctl = P.ctl;
  const int j = *(volatile int32_t *)&ctl->jbase + P.launch_idx;
  const int nsw = P.nsw;

  // device-side convergence control (uniform over the grid): a launch after
  // the one that met tol does nothing
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

  const int ps = blockIdx.x * I - FH;  // first pair (half-column) of the strip, even
  const int ys = P.y_begin + blockIdx.y * P.rows_per_cta;
  const int ye = min(ys + P.rows_per_cta, P.y_end);
  const int r_first = ys - 2 * F, r_last = ye + 2 * F - 1;

  {
    const int t = l * 32 + lane;
    for (int k = t; k < kGuard; k += 32 * L) {
      smem_f[k] = 0.0;
      ring[S * SE + k] = 0.0;
    }
  }
  if (leader) {
    for (int s = 0; s < S; ++s) mbar_init(&full_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ring slot of row r is (r - r_first) mod S
  auto issue_slot = [&](int r, int s) {
    double *st = ring + s * SE;
    mbar_expect_tx(&full_bar[s], STAGE_BYTES);
    tma4(st, mVin, &full_bar[s], ps, r);
    tma4(st + GX, &P.mgx, &full_bar[s], ps, r);
    tma4(st + GY, &P.mgy, &full_bar[s], ps, r);
    tma4(st + GZ, &P.mgz, &full_bar[s], ps, r);
    tma4(st + BB, &P.mb, &full_bar[s], ps, r);
    tma4(st + ID, &P.mid, &full_bar[s], ps, r);
  };
  if (leader)
    for (int r = r_first; r < r_first + S && r <= r_last; ++r) issue_slot(r, r - r_first);

  const double w = P.omega;
  const int pe = l * kRow + lane;        // my even-column node in an array block
  const int po = pe + 32;                // my odd-column node
  const int gp = ps + lane;              // my pair (global half-column)
  const bool exact_lane = lane >= FH && lane < FH + I && gp < P.HP;
  const bool has_down = l > 0;
  const int lpar = (l + P.ypar) & 1;
  double *vout_e = Vout + (int64_t)l * P.layer_stride + gp;
  double *vout_o = vout_e + P.HP;
  double dmax = 0.0;

  // new value of the parity-e node of my pair in row r (slots sl, sn = row
  // r-1, ss = row r+1); *addr receives its shared-memory address
  auto upd = [&](int e, int sl, int sn, int ss, double &Vc, double *&addr) -> double {
    const int me = e ? po : pe;
    const int ow = e ? pe : po - 1;
    const int oe = e ? pe + 1 : po;
    addr = ring + sl * SE + me;
    return node_update<L>(ring + sl * SE, ring + sn * SE, ring + ss * SE, me, ow, oe, w, has_down, Vc);
  };
  auto wait_k = [&](int k, int s) { mbar_wait(&full_bar[s], (uint32_t)((k / S) & 1)); };
  constexpr auto md = [](int a) { return ((a % S) + S) % S; };

  wait_k(0, 0);
  if (r_first + 1 <= r_last) wait_k(1, 1 % S);
  // y = r_first + 1 + u (mod S): the loop is unrolled S times so every ring
  // slot below is a compile-time constant.  `last` (the level whose result is
  // written and whose |dV| is the convergence norm) is a compile-time constant
  // on the common path nsw == F.
#ifdef PG_PROF
  unsigned long long prof[6] = {0, 0, 0, 0, 0, 0};
#endif
  auto sweep_pass = [&](const int last) {
    const int y_end_loop = r_last + D * last;
    for (int y0 = r_first + 1; y0 <= y_end_loop; y0 += S) {
#pragma unroll
      for (int u = 0; u < S; ++u) {
        const int y = y0 + u;
        if (y > y_end_loop) break;
        PROF_T(t0);
        if (y + 1 <= r_last) wait_k(y + 1 - r_first, md(2 + u));
        PROF_T(t1);
        // -------------------------------------------- phase A: red_f(y - D f)
        double dA = 0.0;
        {
          double vn[F], vc[F], *ad[F];
#pragma unroll
          for (int f = 0; f < F; ++f) {
            const int r = y - D * f;
            vn[f] = upd(lpar ^ (r & 1), md(1 + u - D * f), md(u - D * f), md(2 + u - D * f), vc[f], ad[f]);
          }
#pragma unroll
          for (int f = 0; f < F; ++f) {
            const int r = y - D * f;
            if (f <= last && r > r_first && r < r_last) *ad[f] = vn[f];
            if (f == last) dA = fabs(vn[f] - vc[f]);
          }
        }
        {
          const int r = y - D * last;
          if (!(r >= ys && r < ye && exact_lane)) dA = 0.0;
        }
        PROF_T(t2);
        if constexpr (D >= 4) fence_proxy_async();
        __syncthreads();
        PROF_T(t3);
        if constexpr (D >= 4) {
          // phase B(y-1) has finished everywhere: its lowest row is dead
          const int R = y - D * (F - 1) - 3 + S;
          if (leader && R <= r_last && R >= r_first + S) issue_slot(R, md(u - D * (F - 1) - 2));
        }
        // -------------------------------------------- phase B: black_f(y - D f - 1)
        double dB = 0.0;
        {
          double vn[F], vc[F], *ad[F];
#pragma unroll
          for (int f = 0; f < F; ++f) {
            const int r = y - D * f - 1;
            vn[f] = upd(lpar ^ (r & 1) ^ 1, md(u - D * f), md(u - 1 - D * f), md(1 + u - D * f), vc[f], ad[f]);
          }
#pragma unroll
          for (int f = 0; f < F; ++f) {
            const int r = y - D * f - 1;
            if (f <= last && r > r_first && r < r_last) *ad[f] = vn[f];
            if (f == last) dB = fabs(vn[f] - vc[f]);
          }
        }
        PROF_T(t4);
        const int ro = y - D * last - 1;  // row finished by the last level
        const bool out_row = ro >= ys && ro < ye && exact_lane;
        if (!out_row) dB = 0.0;
        dA = dA > dB ? dA : dB;
        dmax = dA > dmax ? dA : dmax;
        if constexpr (D == 3) fence_proxy_async();
        if (out_row) {
          const double *R = ring + md(u - D * last) * SE;
          vout_e[(int64_t)ro * P.NXP] = R[pe];
          vout_o[(int64_t)ro * P.NXP] = R[po];
        }
        PROF_T(t5);
        if constexpr (D == 3) {
          __syncthreads();
          const int R = y - D * (F - 1) - 2 + S;
          if (leader && R <= r_last && R >= r_first + S) issue_slot(R, md(u - D * (F - 1) - 1));
        }
        PROF_T(t6);
        PROF_ADD(0, t0, t1);
        PROF_ADD(1, t1, t2);
        PROF_ADD(2, t2, t3);
        PROF_ADD(3, t3, t4);
        PROF_ADD(4, t4, t5);
        PROF_ADD(5, t5, t6);
      }
    }
  };
  if (nsw == F)
    sweep_pass(F - 1);
  else
    sweep_pass(nsw - 1);
#ifdef PG_PROF
  if (lane == 0)
    for (int k = 0; k < 6; ++k) atomicAdd(&g_prof[k], prof[k]);
  if (lane == 0) atomicAdd(&g_prof[6], 1ull);
#endif
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

// 4-D view of a parity-split mesh array: (half-column, parity, row, layer)
bool encode(CUtensorMap *m, const double *base, const MeshDims &d) {
  auto fn = get_encoder();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)d.HP, 2, (cuuint64_t)d.NY, (cuuint64_t)d.L};
  cuuint64_t strides[3] = {(cuuint64_t)d.HP * 8, (cuuint64_t)d.NXP * 8, (cuuint64_t)d.layer_stride * 8};
  cuuint32_t box[4] = {32, 2, 1, (cuuint32_t)d.L};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

constexpr size_t fused_smem(int L, int S) { return ((size_t)S * 6 * L * kRow + 2 * kGuard) * 8; }

template <int L, int F, int S, int D>
cudaError_t launch_fused_t(pg_grid *g, const FusedParams &P, dim3 grid) {
  auto kern = k_rb_sweep_fused<L, F, S, D>;
  const size_t smem = fused_smem(L, S);
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

// Compiled variants: every L in 1..8 with F = 1..4 at D = 3 and 2 prefetch
// stages (S = 3(F-1) + 6) where the ring fits in 227 KB, plus D = 4 and other
// prefetch depths for L = 4 (tuning via options "lag" and "stages").
#define PG_FUSED_CASES(X)                                                           \
  X(1, 1, 6, 3) X(1, 2, 9, 3) X(1, 3, 12, 3) X(1, 4, 15, 3)                          \
  X(2, 1, 6, 3) X(2, 2, 9, 3) X(2, 3, 12, 3) X(2, 4, 15, 3)                          \
  X(3, 1, 6, 3) X(3, 2, 9, 3) X(3, 3, 12, 3) X(3, 4, 15, 3)                          \
  X(4, 1, 6, 3) X(4, 2, 9, 3) X(4, 3, 12, 3) X(4, 4, 15, 3)                          \
  X(5, 1, 6, 3) X(5, 2, 9, 3) X(5, 3, 12, 3)                                         \
  X(6, 1, 6, 3) X(6, 2, 9, 3) X(6, 3, 12, 3)                                         \
  X(7, 1, 6, 3) X(7, 2, 9, 3)                                                        \
  X(8, 1, 6, 3) X(8, 2, 9, 3)                                                        \
  X(4, 2, 8, 3) X(4, 2, 10, 3) X(4, 2, 11, 4) X(4, 2, 10, 4) X(4, 3, 11, 3)          \
  X(4, 3, 14, 4) X(2, 2, 11, 4) X(2, 3, 14, 4) X(2, 4, 17, 4) X(8, 2, 8, 3)

constexpr int fused_key(int L, int F, int S, int D) { return ((L * 8 + F) * 32 + S) * 8 + D; }

}  // namespace

int fused_exact_lanes(int F) { return 32 - 2 * ((F + 1) & ~1); }

bool tma_available(pg_grid *g) {
  if (g->kind != 0) return false;
  if (g->tma_state == 0) {
    g->tma_state = -1;
    static_assert(sizeof(FusedParams) <= 4096, "kernel params too large");
    const double *bufs[7] = {g->V[0], g->V[1], g->gx, g->gy, g->gze, g->b, g->invd};
    bool ok = get_encoder() != nullptr;
    for (int k = 0; ok && k < 7; ++k) ok = encode(&g->tmap[k], bufs[k], g->md);
    if (ok) g->tma_state = 1;
  }
  return g->tma_state == 1;
}

int fused_default_stages(int L, int F, int D) {
  // D (F-1) + 4 resident rows + 2 prefetch stages
  return D * (F - 1) + 6;
}

bool fused_variant_exists(int L, int F, int S, int D) {
  switch (fused_key(L, F, S, D)) {
#define X(l, f, s, d) case fused_key(l, f, s, d):
    PG_FUSED_CASES(X)
#undef X
    return true;
    default:
      return false;
  }
}

int fused_ctas_per_sm(int L, int S) {
  const size_t smem = fused_smem(L, S) + 1024;
  int c = (int)((228 * 1024) / smem);
  return c < 1 ? 1 : c;
}

cudaError_t launch_rb_sweep_fused(pg_grid *g, double omega, double tol, int j, int nsw, int F,
                                  int S, int D, int rows_per_cta, int y_begin, int y_end, int ypar) {
  if (!tma_available(g)) return cudaErrorNotSupported;
  FusedParams P;
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
  const int strips = (g->md.HP + fused_exact_lanes(F) - 1) / fused_exact_lanes(F);
  const dim3 grid(strips, (y_end - y_begin + rows_per_cta - 1) / rows_per_cta);
  switch (fused_key(g->md.L, F, S, D)) {
#define X(l, f, s, d) \
  case fused_key(l, f, s, d): return launch_fused_t<l, f, s, d>(g, P, grid);
    PG_FUSED_CASES(X)
#undef X
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace pgb

#ifdef PG_PROF
extern "C" PG_API int pg_debug_prof(unsigned long long *out8, int reset) {
  cudaMemcpyFromSymbol(out8, pgb::g_prof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(pgb::g_prof, z, sizeof(z));
  }
  return 0;
}
#endif
