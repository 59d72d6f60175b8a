// Device kernels of the B200 power-grid transient solver (sm_100a).
//
// Hot path per backward-Euler step (Algorithm 1):
//   k_rhs_fused        fused RHS: C_i/h x_i(t) + pad G0 Vdd (+ companion history)
//                      - PWL loads I_i(t+h), one launch per step   (Eq. (2) / (12))
//   (pg_sweep_fused.cu) k_rb_sweep_fused: F red-black SOR sweeps per streaming
//                      pass (Eq. (13) in red-black numbering + Eq. (15)), fused
//                      warp-shuffle max|dV| reduction                  (line 7-8)
//   k_jacobi_mesh      weighted Jacobi sweep (comparison)
//   k_rb_colour_mesh   red-black SOR one colour per launch (meshes of any layer count)
//   k_csr_sweep        multi-colour Gauss-Seidel/SOR on the CSR store (irregular grids)
//   k_ind_update_*     companion inductor currents i(t+h) = g_e v + alpha i(t)  (Eq. (10))
//   k_step_end         device-side bookkeeping of the step (sweep count, buffer parity)
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cooperative_groups.h>

#include "pg_internal.h"

namespace cg = cooperative_groups;

namespace pgb {

#define FULLMASK 0xffffffffu

__device__ __forceinline__ double2 ld2(const double *p) {
  return __ldg(reinterpret_cast<const double2 *>(p));
}
__device__ __forceinline__ void st2(double *p, double a, double b) {
  *reinterpret_cast<double2 *>(p) = make_double2(a, b);
}
__device__ __forceinline__ unsigned long long d2u(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double u2d(unsigned long long x) {
  return __longlong_as_double(static_cast<long long>(x));
}

// ------------------------------------------------------------------ convergence
// Evaluated identically by every CTA of a sweep launch (uniform), so a converged
// step turns the remaining queued launches into no-ops.
__device__ __forceinline__ bool sweep_skip(DevCtl *c, int j, double tol, bool first_of_sweep) {
  if (*(volatile int32_t *)&c->done) return true;
  if (j > 0 && first_of_sweep) {
    double prev = u2d(*(volatile unsigned long long *)&c->dmax[(j - 1) & (kRing - 1)]);
    if (prev < tol) {
      if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0) {
        c->done = 1;
        c->launches_done = j;
      }
      return true;
    }
  }
  return false;
}

// max-reduce a CTA's |dV| into the launch's norm slot (bit pattern of a
// non-negative double orders like its value).  The slot only grows, so a CTA
// whose maximum does not exceed the value it reads skips the atomic: the
// same-address atomics of thousands of CTAs serialise in L2.
__device__ __forceinline__ void norm_max(unsigned long long *slot, double m) {
  const unsigned long long v = d2u(m);
  if (v > *(volatile unsigned long long *)slot) atomicMax(slot, v);
}

__device__ __forceinline__ void zero_next_slot(DevCtl *c, int j, bool first_of_sweep) {
  if (first_of_sweep && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    c->dmax[(j + 1) & (kRing - 1)] = 0ull;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULLMASK, v, o));
  return v;
}

// ------------------------------------------------------------ Jacobi (mesh)
// Weighted Jacobi (comparison baseline): every node from the previous iterate,
// V[(base + j) & 1] -> the other buffer.  One thread per storage element.
struct JacobiArgs {
  MeshDims d;
  const double *gx, *gy, *gz, *b, *invd;
  double *V0, *V1;
  double omega, tol;
  int32_t launch_idx;
  DevCtl *ctl;
};

__global__ void __launch_bounds__(256) k_jacobi_mesh(JacobiArgs a) {
  // one row (layer l, row y) of the parity-split layout per blockIdx.y step,
  // storage position p = threadIdx.x + blockIdx.x * blockDim.x inside the row:
  // no integer division per node, x neighbours at fixed offsets (the even
  // node 2p has odd neighbours at HP + p - 1 and HP + p, the odd node 2q + 1
  // even neighbours at q and q + 1), coalesced loads of every array
  __shared__ double wmax[8];
  a.launch_idx += *(volatile int32_t *)&a.ctl->jbase;
  if (sweep_skip(a.ctl, a.launch_idx, a.tol, true)) return;
  zero_next_slot(a.ctl, a.launch_idx, true);
  const MeshDims d = a.d;
  const int par = (*(volatile int32_t *)&a.ctl->base + a.launch_idx) & 1;
  const double *Vin = par ? a.V1 : a.V0;
  double *Vout = par ? a.V0 : a.V1;
  const double w = a.omega;
  double dmax = 0.0;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const bool odd = p >= d.HP;
  const int h = odd ? p - d.HP : p;
  const int x = 2 * h + (odd ? 1 : 0);
  // storage offsets (within the row) of the west / east neighbours
  const int pw = odd ? h : d.HP + h - 1, pe = odd ? h + 1 : d.HP + h;
  const bool in_row = p < d.NXP;
  for (int64_t r = blockIdx.y; r < (int64_t)d.L * d.NY; r += gridDim.y) {
    if (!in_row) continue;
    const int64_t l = r / d.NY, y = r - l * d.NY;
    const int64_t base = l * d.layer_stride + y * d.NXP;
    const int64_t i = base + p;
    const double vc = __ldg(Vin + i);
    if (x >= d.NX) {
      Vout[i] = vc;
      continue;
    }
    double s = __ldg(a.b + i);
    if (x + 1 < d.NX) s = fma(__ldg(a.gx + i), __ldg(Vin + base + pe), s);
    if (x > 0) s = fma(__ldg(a.gx + base + pw), __ldg(Vin + base + pw), s);
    if (y + 1 < d.NY) s = fma(__ldg(a.gy + i), __ldg(Vin + i + d.NXP), s);
    if (y > 0) s = fma(__ldg(a.gy + i - d.NXP), __ldg(Vin + i - d.NXP), s);
    if (l + 1 < d.L) s = fma(__ldg(a.gz + i), __ldg(Vin + i + d.layer_stride), s);
    if (l > 0) s = fma(__ldg(a.gz + i - d.layer_stride), __ldg(Vin + i - d.layer_stride), s);
    const double vn = fma(w, s * __ldg(a.invd + i) - vc, vc);
    Vout[i] = vn;
    dmax = fmax(dmax, fabs(vn - vc));
  }
  dmax = warp_max(dmax);
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) wmax[wid] = dmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmax(m, wmax[k]);
    norm_max(&a.ctl->dmax[a.launch_idx & (kRing - 1)], m);
  }
}

// ------------------------------------------- red-black SOR, one colour per launch
// Mesh sweep for any layer count (meshes taller than the strip kernels'
// kMaxLayers, or option "colour"): one sweep of Eq. (13) + (15) in the
// red-black numbering (R12) is two launches, colour 0 (red,
// (l + y + x) even) then colour 1.  In the parity-split layout the nodes of one
// colour in a row are one half row, x parity (colour + l + y) & 1, so thread p
// of a row updates storage element xpar * HP + p: coalesced, no idle lanes.
// Ping-pong like the streaming sweep: colour 0 reads iterate k - 1 from V[par]
// and writes its nodes to V[!par]; colour 1 reads its own old value from V[par]
// and its neighbours (all red: the mesh is bipartite) from V[!par].  Same
// operand order as upd_c, absent neighbours with g = 0 and V = 0 (what the
// TMA zero fill gives the streaming kernels), so the iterates equal theirs bit
// for bit.  max|dV| of both colours goes to the launch's norm slot.
struct ColourArgs {
  MeshDims d;
  const double *gx, *gy, *gz, *b, *invd;
  double *V0, *V1;
  double omega, tol;
  int32_t launch_idx, colour;
  DevCtl *ctl;
};

__global__ void __launch_bounds__(128) k_rb_colour_mesh(ColourArgs a) {
  __shared__ double wmax[4];
  a.launch_idx += *(volatile int32_t *)&a.ctl->jbase;
  const bool first = a.colour == 0;
  if (sweep_skip(a.ctl, a.launch_idx, a.tol, first)) return;
  zero_next_slot(a.ctl, a.launch_idx, first);
  const MeshDims d = a.d;
  const int par = (*(volatile int32_t *)&a.ctl->base + a.launch_idx) & 1;
  const double *Vold = par ? a.V1 : a.V0;
  double *Vnew = par ? a.V0 : a.V1;
  const double *Vnb = first ? Vold : Vnew;  // the other colour's latest values
  const double w = a.omega;
  double dmax = 0.0;
  // two column pairs per thread, p0 = 2t and p0 + 1: 16-byte loads of every
  // array at the node's own positions (HP is even, so p0 + 1 < HP and every
  // pair of positions is 16-byte aligned).  Padding nodes (x >= NX) have
  // g = 0, 1/d = 0, b = 0 and V = 0 and stay 0, so they need no mask.
  const int p0 = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (p0 < d.HP) {
    for (int r = blockIdx.y; r < d.L * d.NY; r += gridDim.y) {
      const int l = r / d.NY, y = r - l * d.NY;
      const int xpar = (a.colour + l + y) & 1;
      const int64_t base = (int64_t)l * d.layer_stride + (int64_t)y * d.NXP;
      const int64_t i = base + xpar * d.HP + p0;
      // own pair = columns (2p, 2p + 1); "other" = the x neighbour outside it:
      // odd nodes (xpar 1): own = even column p, other = even column p + 1;
      // even nodes: own = odd column p, other = odd column p - 1
      const int64_t iown = xpar ? base + p0 : base + d.HP + p0;
      const double2 gxo = ld2(a.gx + base + p0);      // link of pair p (gxOwn)
      const double2 vo = ld2(Vnb + iown);
      double2 gxt, vt;                               // gxOth, Voth of the two nodes
      if (xpar) {
        gxt = ld2(a.gx + base + d.HP + p0);
        vt.x = vo.y;
        vt.y = p0 + 2 < d.HP ? __ldg(Vnb + base + p0 + 2) : 0.0;
      } else {
        const double2 g2 = ld2(a.gx + base + d.HP + p0);
        gxt.x = p0 > 0 ? __ldg(a.gx + base + d.HP + p0 - 1) : 0.0;
        gxt.y = g2.x;
        vt.x = p0 > 0 ? __ldg(Vnb + base + d.HP + p0 - 1) : 0.0;
        vt.y = vo.x;
      }
      const bool hN = y > 0, hS = y + 1 < d.NY, hU = l + 1 < d.L, hD = l > 0;
      const double2 z2 = make_double2(0.0, 0.0);
      const double2 gyN = hN ? ld2(a.gy + i - d.NXP) : z2, VN = hN ? ld2(Vnb + i - d.NXP) : z2;
      const double2 gyS = ld2(a.gy + i), VS = hS ? ld2(Vnb + i + d.NXP) : z2;
      const double2 gzU = ld2(a.gz + i), VU = hU ? ld2(Vnb + i + d.layer_stride) : z2;
      const double2 gzD = hD ? ld2(a.gz + i - d.layer_stride) : z2;
      const double2 VD = hD ? ld2(Vnb + i - d.layer_stride) : z2;
      const double2 Vc = ld2(Vold + i), bb = ld2(a.b + i), id = ld2(a.invd + i);
      auto upd = [&](double gxOwn, double Vown, double gxOth, double Voth, double gn, double vn_, double gs,
                     double vs, double gu, double vu, double gd, double vd, double b, double idd, double vc) {
        double s1 = fma(gxOwn, Vown, b);
        s1 = fma(gxOth, Voth, s1);
        s1 = fma(gn, vn_, s1);
        double s2 = gs * vs;
        s2 = fma(gu, vu, s2);
        s2 = fma(gd, vd, s2);
        return fma(w, (s1 + s2) * idd - vc, vc);
      };
      const double n0 = upd(gxo.x, vo.x, gxt.x, vt.x, gyN.x, VN.x, gyS.x, VS.x, gzU.x, VU.x, gzD.x, VD.x, bb.x,
                            id.x, Vc.x);
      const double n1 = upd(gxo.y, vo.y, gxt.y, vt.y, gyN.y, VN.y, gyS.y, VS.y, gzU.y, VU.y, gzD.y, VD.y, bb.y,
                            id.y, Vc.y);
      st2(Vnew + i, n0, n1);
      dmax = fmax(dmax, fmax(fabs(n0 - Vc.x), fabs(n1 - Vc.y)));  // NaN / Inf: the RHS kernel's check of V(t)
    }
  }
  dmax = warp_max(dmax);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = dmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmax(m, wmax[k]);
    norm_max(&a.ctl->dmax[a.launch_idx & (kRing - 1)], m);
  }
}

// ------------------------------------------------------------------ CSR sweeps
struct CsrArgs {
  const int32_t *rowptr;
  const int32_t *col;
  const double *val, *b, *invd;
  double *V0, *V1;  // GS: in place on V[base]; Jacobi: V[(base+j)&1] -> the other
  int64_t r0, r1;   // rows of this colour (GS) / all rows (Jacobi)
  double omega, tol;
  int32_t launch_idx;
  int32_t first;    // first colour of the sweep
  int32_t pre;      // staged sweep launched with programmatic stream serialisation after a sweep launch
  DevCtl *ctl;
};

// streamed loads with an L2 eviction policy (createpolicy); not volatile: they
// read arrays no kernel of the sweep writes, so the compiler may schedule them
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ldf(const double *p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ldi(const int32_t *p, uint64_t pol) {
  int32_t v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__global__ void __launch_bounds__(256) k_csr_sweep(CsrArgs a) {
  __shared__ double wmax[8];
  a.launch_idx += *(volatile int32_t *)&a.ctl->jbase;
  if (sweep_skip(a.ctl, a.launch_idx, a.tol, a.first != 0)) return;
  zero_next_slot(a.ctl, a.launch_idx, a.first != 0);
  double *V = (*(volatile int32_t *)&a.ctl->base) ? a.V1 : a.V0;
  double dmax = 0.0;
  // the row data (structure, values, b, 1/d) streams through L2 evict_first so
  // that the gathered neighbour voltages stay resident
  const uint64_t pf = pol_first();
  for (int64_t i = a.r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.r1;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = ldf(a.b + i, pf);
    const int32_t k1 = ldi(a.rowptr + i + 1, pf);
    for (int32_t k = ldi(a.rowptr + i, pf); k < k1; ++k) s = fma(ldf(a.val + k, pf), V[ldi(a.col + k, pf)], s);
    const double vc = V[i];
    const double vn = fma(a.omega, s * ldf(a.invd + i, pf) - vc, vc);
    V[i] = vn;
    dmax = fmax(dmax, fabs(vn - vc));
  }
  dmax = warp_max(dmax);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = dmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmax(m, wmax[k]);
    norm_max(&a.ctl->dmax[a.launch_idx & (kRing - 1)], m);
  }
}

__global__ void __launch_bounds__(256) k_csr_jacobi(CsrArgs a) {
  __shared__ double wmax[8];
  a.launch_idx += *(volatile int32_t *)&a.ctl->jbase;
  if (sweep_skip(a.ctl, a.launch_idx, a.tol, true)) return;
  zero_next_slot(a.ctl, a.launch_idx, true);
  const int par = (*(volatile int32_t *)&a.ctl->base + a.launch_idx) & 1;
  const double *Vin = par ? a.V1 : a.V0;
  double *Vout = par ? a.V0 : a.V1;
  double dmax = 0.0;
  for (int64_t i = a.r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.r1;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = __ldg(a.b + i);
    const int32_t k1 = a.rowptr[i + 1];
    for (int32_t k = a.rowptr[i]; k < k1; ++k) s = fma(__ldg(a.val + k), __ldg(Vin + __ldg(a.col + k)), s);
    const double vc = __ldg(Vin + i);
    const double vn = fma(a.omega, s * __ldg(a.invd + i) - vc, vc);
    Vout[i] = vn;
    dmax = fmax(dmax, fabs(vn - vc));
  }
  dmax = warp_max(dmax);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = dmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmax(m, wmax[k]);
    norm_max(&a.ctl->dmax[a.launch_idx & (kRing - 1)], m);
  }
}

// ------------------------------------------------- staged CSR sweep (bulk copies)
// Multi-colour Gauss-Seidel / SOR of one colour's rows (Eq. (13)/(15) on an
// arbitrary graph, colour-permuted rows, §IV), with the row data of
// every tile of kCsrR rows -- row pointers, b, 1/d, column indices, values: all
// contiguous in the colour-permuted store -- moved into shared memory by 1-D
// bulk copies (cp.async.bulk, mbarrier completion, L2 evict_first).  The only
// dependent global loads left are the gathers V[col] (the other colours' rows,
// L2-resident for these grid sizes); each thread keeps the gathers of its two
// rows in flight together.  What bounds the sweep is the number of rows whose
// gathers are outstanding per SM, capped by the rows staged in shared memory
// and by the register file (measured), so the default is ONE
// stage per CTA and many small persistent CTAs per SM (256-row tiles, 128
// threads, 8 CTAs per SM, 64 registers): a CTA's bulk copies are covered by
// the other resident CTAs' compute, and about two thirds of the staged rows
// are computing at any time instead of the half of a two-stage ring
// (-DPG_CSR_S=2 and the other geometries stay as experiment builds).
// Per-row arithmetic and summation order are those of k_csr_sweep
// (bit-identical results).  Ranges are copied from 16-byte aligned starts and
// rounded up to 16 bytes (the arrays carry zero slack).
struct __align__(16) CsrStage {
  int32_t rp[kCsrR + 8];
  double b[kCsrR + 2];
  double invd[kCsrR + 2];
  int32_t col[kCsrE + 8];
  double val[kCsrE + 4];
};
#ifndef PG_CSR_T
#define PG_CSR_T 128
#endif
#ifndef PG_CSR_B
#define PG_CSR_B 8
#endif
#ifndef PG_CSR_S
#define PG_CSR_S 1
#endif
constexpr int kCsrT = PG_CSR_T;  // threads per CTA: kCsrR / kCsrT (1 or 2) rows each
constexpr int kCsrB = PG_CSR_B;  // resident CTAs per SM
constexpr int kCsrS = PG_CSR_S;  // stages per CTA: kCsrS - 1 tiles in flight ahead of the compute (1: the
                                 // other resident CTAs cover a CTA's load)
static_assert(kCsrS >= 1 && kCsrS <= 8, "stage count");
static_assert(kCsrR == kCsrT || kCsrR == 2 * kCsrT, "one or two rows per thread");
constexpr int kCsrU = 6;         // gathers per row issued together (mesh-like degrees <= 6)

__device__ __forceinline__ uint32_t csr_su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void csr_bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(csr_su32(dst)), "l"(src), "r"(bytes), "r"(csr_su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint32_t r16(int64_t bytes) { return (uint32_t)((bytes + 15) & ~(int64_t)15); }

// tile t's entry range [k0, k1) = [rowptr[r0], rowptr[r1]) is passed in: the
// caller loads it one tile ahead, so the refill after a barrier does not wait
// on a global load (warp 0 would otherwise start every tile a round trip late)
__device__ void csr_issue(const CsrArgs &a, CsrStage *st, uint64_t *bar, int64_t t, int64_t k0, int64_t k1,
                          uint64_t pol) {
  const int64_t r0 = a.r0 + t * kCsrR, r1 = min(a.r1, r0 + kCsrR);
  const int64_t ra = r0 & ~3ll, rb = r0 & ~1ll, ca = k0 & ~3ll, va = k0 & ~1ll;
  const uint32_t n_rp = r16(4 * (r1 + 1 - ra)), n_b = r16(8 * (r1 - rb)), n_c = r16(4 * (k1 - ca)),
                 n_v = r16(8 * (k1 - va));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(csr_su32(bar)),
               "r"(n_rp + 2 * n_b + n_c + n_v)
               : "memory");
  csr_bulk(st->rp, a.rowptr + ra, n_rp, bar, pol);
  csr_bulk(st->b, a.b + rb, n_b, bar, pol);
  csr_bulk(st->invd, a.invd + rb, n_b, bar, pol);
  if (n_c) csr_bulk(st->col, a.col + ca, n_c, bar, pol);
  if (n_v) csr_bulk(st->val, a.val + va, n_v, bar, pol);
}

__global__ void __launch_bounds__(kCsrT, kCsrB) k_csr_sweep_staged(CsrArgs a) {
  extern __shared__ __align__(16) unsigned char csr_smem[];
  CsrStage *st = reinterpret_cast<CsrStage *>(csr_smem);
  __shared__ __align__(8) uint64_t bar[kCsrS];
  __shared__ double wmax[kCsrT / 32];
  const int64_t ntiles = (a.r1 - a.r0 + kCsrR - 1) / kCsrR;
  const int tid = threadIdx.x;
  const uint64_t pf = pol_first();
  // Programmatic dependent launch (a.pre: the previous launch in the stream is
  // a sweep launch, whose outputs are V and the control block only): the
  // first tiles' row data -- constants of the transient's step -- are
  // requested while that launch drains; V and the control block are read
  // after griddepcontrol.wait.  Otherwise the skip test comes first and a
  // converged step's queued launches cost no memory traffic.
  if (a.pre) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else {
    a.launch_idx += *(volatile int32_t *)&a.ctl->jbase;
    if (sweep_skip(a.ctl, a.launch_idx, a.tol, a.first != 0)) return;
  }
  if (tid == 0) {
    for (int k = 0; k < kCsrS; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(csr_su32(&bar[k])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < kCsrS; ++k) {
      const int64_t t = blockIdx.x + (int64_t)k * gridDim.x;
      if (t < ntiles) {
        const int64_t r0 = a.r0 + t * kCsrR;
        csr_issue(a, &st[k], &bar[k], t, a.rowptr[r0], a.rowptr[min(a.r1, r0 + kCsrR)], pf);
      }
    }
  }
  if (a.pre) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    a.launch_idx += *(volatile int32_t *)&a.ctl->jbase;
    if (sweep_skip(a.ctl, a.launch_idx, a.tol, a.first != 0)) {
      // the copies in flight target this CTA's shared memory: let them land
      if (tid == 0) {
        for (int k = 0; k < kCsrS; ++k) {
          if (blockIdx.x + (int64_t)k * gridDim.x >= ntiles) break;
          uint32_t done = 0;
          while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(csr_su32(&bar[k])), "r"(0u)
                : "memory");
        }
      }
      __syncthreads();
      return;
    }
  }
  zero_next_slot(a.ctl, a.launch_idx, a.first != 0);
  double *V = (*(volatile int32_t *)&a.ctl->base) ? a.V1 : a.V0;
  double dmax = 0.0;
  int sg = 0;          // stage of tile t
  uint32_t par = 0;    // its mbarrier phase parity (flips every kCsrS tiles)
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    CsrStage &S = st[sg];
    // entry range of the tile this stage is refilled with after the barrier
    const int64_t tn = t + kCsrS * (int64_t)gridDim.x;
    int32_t nk0 = 0, nk1 = 0;
    if (tid == 0 && tn < ntiles) {
      const int64_t nr0 = a.r0 + tn * kCsrR;
      nk0 = a.rowptr[nr0];
      nk1 = a.rowptr[min(a.r1, nr0 + kCsrR)];
    }
    {
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(csr_su32(&bar[sg])), "r"(par)
            : "memory");
    }
    const int64_t r0 = a.r0 + t * kCsrR;
    const int nr = (int)min((int64_t)kCsrR, a.r1 - r0);
    const int oa = (int)(r0 & 3), ob = (int)(r0 & 1);
    const int32_t k0 = S.rp[oa];
    const int32_t ca = k0 & ~3, va = k0 & ~1;
    // two rows per thread, their gathers issued together
    const int q0 = tid, q1 = tid + kCsrT;
    const bool h0 = q0 < nr, h1 = kCsrR > kCsrT && q1 < nr;
    int32_t e0 = h0 ? S.rp[oa + q0] : 0, f0 = h0 ? S.rp[oa + q0 + 1] : 0;
    int32_t e1 = h1 ? S.rp[oa + q1] : 0, f1 = h1 ? S.rp[oa + q1 + 1] : 0;
    double s0 = h0 ? S.b[ob + q0] : 0.0, s1 = h1 ? S.b[ob + q1] : 0.0;
    while (e0 < f0 || e1 < f1) {
      // the gathers of both rows in flight together; the branch values are
      // read from the stage when they have landed (not held in registers
      // beside them: 64 registers, 1024 resident threads per SM)
      double v0[kCsrU], v1[kCsrU];
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        v0[u] = e0 + u < f0 ? __ldg(V + S.col[e0 + u - ca]) : 0.0;
        v1[u] = e1 + u < f1 ? __ldg(V + S.col[e1 + u - ca]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        if (e0 + u < f0) s0 = fma(S.val[e0 + u - va], v0[u], s0);
        if (e1 + u < f1) s1 = fma(S.val[e1 + u - va], v1[u], s1);
      }
      e0 += kCsrU;
      e1 += kCsrU;
    }
    if (h0) {
      const int64_t i = r0 + q0;
      const double vc = V[i];
      const double vn = fma(a.omega, s0 * S.invd[ob + q0] - vc, vc);
      V[i] = vn;
      dmax = fmax(dmax, fabs(vn - vc));
    }
    if (h1) {
      const int64_t i = r0 + q1;
      const double vc = V[i];
      const double vn = fma(a.omega, s1 * S.invd[ob + q1] - vc, vc);
      V[i] = vn;
      dmax = fmax(dmax, fabs(vn - vc));
    }
    // every thread is done reading stage sg: refill it (generic-proxy reads
    // ordered before the async-proxy writes)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && tn < ntiles) csr_issue(a, &S, &bar[sg], tn, nk0, nk1, pf);
    if (++sg == kCsrS) {
      sg = 0;
      par ^= 1u;
    }
  }
  dmax = warp_max(dmax);
  if ((tid & 31) == 0) wmax[tid >> 5] = dmax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int k = 0; k < kCsrT / 32; ++k) m = fmax(m, wmax[k]);
    norm_max(&a.ctl->dmax[a.launch_idx & (kRing - 1)], m);
  }
}

// ------------------------------------------------------------------ RHS (fused)
__device__ __forceinline__ double pwl_eval(const double *t, const double *v, int64_t s, int64_t e,
                                           double tt) {
  if (tt <= t[s]) return v[s];
  if (tt >= t[e - 1]) return v[e - 1];
  for (int64_t k = s; k + 1 < e; ++k) {
    if (tt <= t[k + 1]) {
      const double w = (tt - t[k]) / (t[k + 1] - t[k]);
      return v[k] + w * (v[k + 1] - v[k]);
    }
  }
  return v[e - 1];
}

// One kernel per time step builds the whole right-hand side of Eq. (12) at
// t + h (Eq. (2): b = (C/h) x(t) + G0 Vdd - i(t+h); Eq. (10): the
// companion history of every inductor):
//   b_i = (C_i/h) V_i(t)
//         - [RLC vias] alpha i_z(t) of the via above + alpha i_z(t) of the via below
//         + sum over the node's pads (g_e Vdd - [series L] alpha i_pad(t))
//         - sum over the node's loads I_k(t + h)            (PWL, reading R8)
// Storage elements are processed in tiles of kRhsTile: the dense term goes to
// a shared-memory tile, then the tile's pad groups and load groups (sorted by
// storage index, one group per node, ranges precomputed per tile on the host)
// add into it -- each node's terms in a fixed order, no atomics, so the sum is
// deterministic -- and the tile is written once.  V(t) is also checked for
// NaN / Inf here (ctl->nonfinite).
struct RhsArgs {
  int64_t np;
  const double *cap;
  double inv_h;
  const double *V0, *V1;
  DevCtl *ctl;
  double *b;
  const double *lz, *gze, *iz;   // RLC vias (lz == nullptr: RC)
  int64_t layer_stride;
  int32_t L;
  const int64_t *pad_tile, *pad_grp, *pad_idx;
  const double *pad_ge, *pad_l, *pad_i;
  double vdd;
  const int64_t *src_tile, *src_grp, *src_idx, *src_ptr;
  const double *pwl_t, *pwl_i;
  double t;
  int64_t ntile;
};

__global__ void __launch_bounds__(256) k_rhs_fused(RhsArgs a) {
  __shared__ double bt[kRhsTile];
  const double *V = a.ctl->base ? a.V1 : a.V0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.ctl->done = 0;
    a.ctl->launches_done = 0;
    a.ctl->dmax[0] = 0ull;
    a.ctl->jbase = 0;
  }
  bool bad = false;
  for (int64_t tile = blockIdx.x; tile < a.ntile; tile += gridDim.x) {
    const int64_t i0 = tile * kRhsTile;
    const int n = (int)min((int64_t)kRhsTile, a.np - i0);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const int64_t i = i0 + k;
      const double v = V[i];
      bad |= !(fabs(v) <= 1.7976931348623157e308);
      double bb = a.cap[i] * a.inv_h * v;
      if (a.lz != nullptr) {
        const int64_t l = i / a.layer_stride;
        if (l + 1 < a.L) bb -= a.lz[i] * a.inv_h * a.gze[i] * a.iz[i];    // current leaving down->up
        if (l > 0) {
          const int64_t j = i - a.layer_stride;
          bb += a.lz[j] * a.inv_h * a.gze[j] * a.iz[j];                    // current arriving from below
        }
      }
      bt[k] = bb;
    }
    __syncthreads();
    if (a.pad_tile != nullptr) {
      const int64_t q1 = a.pad_tile[tile + 1];
      for (int64_t q = a.pad_tile[tile] + threadIdx.x; q < q1; q += blockDim.x) {
        double bb = 0.0;
        for (int64_t k = a.pad_grp[q]; k < a.pad_grp[q + 1]; ++k) {
          bb += a.pad_ge[k] * a.vdd;
          if (a.pad_l != nullptr) bb -= a.pad_l[k] * a.inv_h * a.pad_ge[k] * a.pad_i[k];
        }
        bt[a.pad_idx[a.pad_grp[q]] - i0] += bb;
      }
      __syncthreads();
    }
    if (a.src_tile != nullptr) {
      const int64_t q1 = a.src_tile[tile + 1];
      for (int64_t q = a.src_tile[tile] + threadIdx.x; q < q1; q += blockDim.x) {
        double bb = 0.0;
        for (int64_t k = a.src_grp[q]; k < a.src_grp[q + 1]; ++k)
          bb += pwl_eval(a.pwl_t, a.pwl_i, a.src_ptr[k], a.src_ptr[k + 1], a.t);
        bt[a.src_idx[a.src_grp[q]] - i0] -= bb;
      }
      __syncthreads();
    }
    for (int k = threadIdx.x; k < n; k += blockDim.x) a.b[i0 + k] = bt[k];
    __syncthreads();
  }
  if (bad) a.ctl->nonfinite = 1;
}

// one pass over the current iterate: flags NaN / Inf (end of a transient call;
// the RHS kernel checks V(t) of every other step)
__global__ void k_check_finite(int64_t np, const double *V0, const double *V1, DevCtl *ctl) {
  const double *V = ctl->base ? V1 : V0;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !(fabs(V[i]) <= 1.7976931348623157e308);
  if (__syncthreads_or(bad) && threadIdx.x == 0) ctl->nonfinite = 1;
}

// -------------------------------------------------------------- per-h setup
__global__ void k_setup_gze(int64_t np, const double *gz, const double *lz, double h, double *gze) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double g = gz[i];
    gze[i] = (lz != nullptr && lz[i] > 0.0 && g > 0.0) ? 1.0 / (1.0 / g + lz[i] / h) : g;
  }
}

__global__ void k_setup_pad_ge(int64_t npad, const double *pg, const double *pl, double h, double *ge) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < npad;
       k += (int64_t)gridDim.x * blockDim.x) {
    ge[k] = (pl != nullptr && pl[k] > 0.0) ? 1.0 / (1.0 / pg[k] + pl[k] / h) : pg[k];
  }
}

// d_i = sum of branch conductances + C_i/h (pads added by k_diag_pads)
__global__ void k_diag_mesh(MeshDims d, const double *gx, const double *gy, const double *gze,
                            const double *cap, double inv_h, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i / d.layer_stride;
    const int64_t y = (i - l * d.layer_stride) / d.NXP;
    const int64_t x = mesh_col(d, i);
    double s = gx[i] + gy[i] + gze[i];
    if (x > 0) s += gx[mesh_index(d, l, y, x - 1)];
    if (y > 0) s += gy[i - d.NXP];
    if (l > 0) s += gze[i - d.layer_stride];
    s += cap[i] * inv_h;
    out[i] = s;
  }
}

__global__ void k_diag_csr(int64_t n, const int32_t *rowptr, const double *val, const double *cap,
                           double inv_h, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) s += val[k];
    out[i] = s + cap[i] * inv_h;
  }
}

__global__ void k_diag_pads(int64_t ngrp, const int64_t *grp, const int64_t *idx, const double *ge,
                            double *d) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ngrp;
       q += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = grp[q]; k < grp[q + 1]; ++k) s += ge[k];
    d[idx[grp[q]]] += s;
  }
}

// invd = 1/d for real nodes (mesh padding -> 0); flags d <= 0 on real nodes
__global__ void k_invert(int64_t np, double *d, MeshDims md, int32_t mesh, DevCtl *ctl) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool real = !mesh || mesh_col(md, i) < md.NX;
    const double v = d[i];
    if (real && !(v > 0.0)) ctl->diag_bad = 1;
    d[i] = real && v > 0.0 ? 1.0 / v : 0.0;
  }
}

// ----------------------------------------------------- companion current update
// i(t+h) = g_e (v_a - v_b)(t+h) + (L/h) g_e i(t)  (backward Euler on R i + L di/dt = v)
__global__ void k_ind_update_mesh(MeshDims d, const double *V0, const double *V1, const DevCtl *ctl,
                                  const double *gze, const double *lz, double inv_h, double *iz) {
  const double *V = ctl->base ? V1 : V0;
  const int64_t n = d.np - d.layer_stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double L = lz[i];
    if (L > 0.0) {
      const double ge = gze[i];
      iz[i] = ge * (V[i] - V[i + d.layer_stride]) + L * inv_h * ge * iz[i];
    }
  }
}

__global__ void k_ind_update_pads(int64_t npad, const int64_t *idx, const double *ge, const double *pl,
                                  const double *V0, const double *V1, const DevCtl *ctl, double vdd,
                                  double inv_h, double *pi) {
  const double *V = ctl->base ? V1 : V0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < npad;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double L = pl[k];
    if (L > 0.0) pi[k] = ge[k] * (V[idx[k]] - vdd) + L * inv_h * ge[k] * pi[k];
  }
}

// ------------------------------------------------------------------ bookkeeping
__global__ void k_step_end(DevCtl *c, int64_t s, int32_t launched, int32_t flips, int32_t fused,
                           int64_t max_sweeps, double tol, int64_t *rec, int32_t count_epoch) {
  const int64_t ran = c->done ? c->launches_done : launched;
  if (count_epoch) c->epoch += ran;  // sweep launches that did work in an armed peer group
  int64_t sw = ran * fused;
  if (sw > max_sweeps) sw = max_sweeps;
  if (flips) c->base ^= (int32_t)(ran & 1);
  rec[s] = sw;
  c->sweeps_total += sw;
  if (sw > c->sweeps_max) c->sweeps_max = sw;
  const double last = ran > 0 ? u2d(c->dmax[(ran - 1) & (kRing - 1)]) : 0.0;
  c->last_delta = last;
  const bool conv = c->done || (ran > 0 && last < tol);
  if (!conv && tol > 0.0 && c->failed == 0) c->failed = (int32_t)s;
}

__global__ void k_batch_advance(DevCtl *c, int32_t nb) { c->jbase += nb; }

// ------------------------------------------------- resident sweep (small grids)
// All sweeps of one time step in ONE launch of one thread-block cluster: the
// mesh is cut into y-slabs of R rows (all layers), one per CTA of the cluster
// (<= 16 CTAs); each CTA keeps its slab of V in shared memory and each thread
// owns one red and one black node of a (layer, row, column pair), their
// conductances, b and 1/d in registers.  A red-black SOR sweep (Eq. (13) +
// (15), same numbering and arithmetic order as the streaming sweep) is: red
// updates, cluster barrier, black updates, cluster barrier; the rows just
// across a slab boundary are read from the neighbouring CTA's shared memory
// (distributed shared memory).  max|dV| is reduced per CTA with a shared
// atomic and read by every thread from all CTAs after the barrier, so the
// whole cluster stops after the same sweep (convergence tested after every
// sweep, R13).  For grids whose state fits a few SMs this replaces a launch
// (and its latency) per sweep by two cluster barriers.  V is updated in
// place (no ping-pong flip); the step's bookkeeping is done here.
struct ClusterArgs {
  MeshDims d;
  const double *gx, *gy, *gz, *b, *invd;
  double *V0, *V1;
  double omega, tol;
  int64_t max_sweeps, s;
  int64_t *rec;
  DevCtl *ctl;
  int32_t R;    // rows per CTA (the last CTA may hold fewer)
  int32_t HPx;  // column pairs per row, ceil(NX / 2)
};

// one node of a thread: its coefficients and where its neighbours live
struct CNode {
  double gE, gW, gN, gS, gU, gD, b, id;
  const double *pN, *pS;   // generic addresses (own or neighbouring CTA)
  int li, iE, iW, iU, iD;  // shared-memory indices (self where absent, g = 0)
  bool on;
};

__device__ __forceinline__ void cnode_init(CNode &n, const ClusterArgs &a, cg::cluster_group &cl,
                                           double *sv, int rank, int Rt, int l, int yy, int x) {
  const MeshDims &d = a.d;
  const int R = a.R, NX = d.NX;
  const int y = rank * R + yy;
  n.on = x < NX;
  if (!n.on) x = NX - 1;  // keep addresses valid; the node is never updated
  const int64_t i = mesh_index(d, l, y, x);
  const int li = (l * R + yy) * NX + x;
  n.li = li;
  const bool hE = x + 1 < NX, hW = x > 0, hN = y > 0, hS = y + 1 < d.NY;
  const bool hU = l > 0, hD = l + 1 < d.L;
  n.gE = hE ? a.gx[i] : 0.0;
  n.gW = hW ? a.gx[mesh_index(d, l, y, x - 1)] : 0.0;
  n.gN = hN ? a.gy[i - d.NXP] : 0.0;
  n.gS = hS ? a.gy[i] : 0.0;
  n.gU = hU ? a.gz[i - d.layer_stride] : 0.0;
  n.gD = hD ? a.gz[i] : 0.0;
  n.b = a.b[i];
  n.id = a.invd[i];
  n.iE = hE ? li + 1 : li;
  n.iW = hW ? li - 1 : li;
  n.iU = hU ? li - R * NX : li;
  n.iD = hD ? li + R * NX : li;
  n.pN = sv + li;
  n.pS = sv + li;
  if (hN) n.pN = yy > 0 ? sv + li - NX : cl.map_shared_rank(sv + (l * R + R - 1) * NX + x, rank - 1);
  if (hS) n.pS = yy + 1 < Rt ? sv + li + NX : cl.map_shared_rank(sv + (l * R) * NX + x, rank + 1);
}

// Eq. (13) + (15) for one node, the streaming sweep's order of operations
// (absent neighbours carry g = 0 and read the node itself: fma(0, v, s) == s)
__device__ __forceinline__ double cnode_update(const CNode &n, const double *sv, double w, double vc) {
  double s1 = fma(n.gE, sv[n.iE], n.b);
  s1 = fma(n.gW, sv[n.iW], s1);
  double s2 = n.gN * *n.pN;
  s2 = fma(n.gS, *n.pS, s2);
  s2 = fma(n.gU, sv[n.iU], s2);
  s2 = fma(n.gD, sv[n.iD], s2);
  return fma(w, (s1 + s2) * n.id - vc, vc);
}

__global__ void __launch_bounds__(512) k_rb_cluster(ClusterArgs a) {
  extern __shared__ double sv[];
  __shared__ unsigned long long slot[2];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int ncta = (int)cl.num_blocks();
  const MeshDims d = a.d;
  const int R = a.R, NX = d.NX, L = d.L;
  const int y0 = rank * R;
  const int Rt = min(R, d.NY - y0);
  double *V = a.ctl->base ? a.V1 : a.V0;
  for (int k = threadIdx.x; k < L * Rt * NX; k += blockDim.x) {
    const int x = k % NX, r = k / NX;
    const int yy = r % Rt, l = r / Rt;
    sv[(l * R + yy) * NX + x] = V[mesh_index(d, l, y0 + yy, x)];
  }
  if (threadIdx.x < 2) slot[threadIdx.x] = 0ull;
  CNode nr, nb;
  nr.on = nb.on = false;
  const int t = threadIdx.x;
  if (t < L * Rt * a.HPx) {
    const int p = t % a.HPx, r = t / a.HPx;
    const int yy = r % Rt, l = r / Rt;
    const int e = (l + y0 + yy) & 1;  // red: (l + y + x) even
    cnode_init(nr, a, cl, sv, rank, Rt, l, yy, 2 * p + e);
    cnode_init(nb, a, cl, sv, rank, Rt, l, yy, 2 * p + 1 - e);
  }
  cl.sync();  // every slab and slot in place
  double vr = nr.on ? sv[nr.li] : 0.0, vb = nb.on ? sv[nb.li] : 0.0;
  const double w = a.omega;
  const int lane = threadIdx.x & 31;
  // max|dV| of sweep kk (its CTA maxima are final after sweep kk's last barrier)
  auto sweep_max = [&](int64_t kk) {
    double m = 0.0;
    if (lane < ncta)
      m = __longlong_as_double((long long)*cl.map_shared_rank(&slot[kk & 1], lane));
    return warp_max(m);
  };
  // The stop test of sweep k is taken one half-sweep late: sweep k + 1's red
  // half runs first and is undone (each thread restores its own red node) if
  // sweep k converged, so the convergence read overlaps useful work.
  int64_t k = 0;
  double last = 0.0;
  bool conv = false;
  while (k < a.max_sweeps) {
    double vrn = vr, vbn = vb;
    if (nr.on) {
      vrn = cnode_update(nr, sv, w, vr);
      sv[nr.li] = vrn;
    }
    // slot (k + 1) & 1 was last read during sweep k (before its last barrier)
    if (threadIdx.x == 0) slot[(k + 1) & 1] = 0ull;
    cl.sync();
    double m = 0.0;
    if (k > 0) m = sweep_max(k);
    if (nb.on) vbn = cnode_update(nb, sv, w, vb);
    if (k > 0) {
      last = m;
      if (a.tol > 0.0 && m < a.tol) {
        if (nr.on) sv[nr.li] = vr;  // sweep k converged: undo sweep k + 1's red half
        conv = true;
        break;
      }
    }
    if (nb.on) sv[nb.li] = vbn;
    double dm = fmax(fabs(vrn - vr), fabs(vbn - vb));
    vr = vrn;
    vb = vbn;
    ++k;
    dm = warp_max(dm);
    // |dV| >= 0: its bit pattern orders like the value
    if (lane == 0 && dm > 0.0) atomicMax(&slot[k & 1], (unsigned long long)__double_as_longlong(dm));
    cl.sync();
  }
  if (!conv && k > 0) last = sweep_max(k);
  cl.sync();  // no CTA leaves while another may still read its shared memory
  for (int q = threadIdx.x; q < L * Rt * NX; q += blockDim.x) {
    const int x = q % NX, r = q / NX;
    const int yy = r % Rt, l = r / Rt;
    V[mesh_index(d, l, y0 + yy, x)] = sv[(l * R + yy) * NX + x];
  }
  if (rank == 0 && threadIdx.x == 0) {
    DevCtl *c = a.ctl;
    a.rec[a.s] = k;
    c->sweeps_total += k;
    if (k > c->sweeps_max) c->sweeps_max = k;
    c->last_delta = last;
    if (a.tol > 0.0 && !(last < a.tol) && c->failed == 0) c->failed = (int32_t)a.s;
  }
}

// cluster shape of the resident sweep: R rows per CTA, ncta CTAs (<= 16),
// T threads (<= 512, one per column pair of the slab); false if it does not fit
struct ClusterPlan {
  int R, ncta, T;
};
static bool cluster_plan(const MeshDims &d, ClusterPlan *p) {
  const int per_row = d.L * ((d.NX + 1) / 2);
  if (per_row > 512) return false;
  const int rmax = std::min(512 / per_row, d.NY);
  const int ncta = (d.NY + rmax - 1) / rmax;
  if (ncta > 16) return false;
  p->ncta = ncta;
  p->R = (d.NY + ncta - 1) / ncta;  // even out the slabs
  p->T = ((p->R * per_row + 31) / 32) * 32;
  return true;
}

bool resident_ok(const pg_grid *g, int method) {
  ClusterPlan p;
  return g->kind == 0 && method == PG_METHOD_RBSOR && !g->slab && g->resident &&
         cluster_plan(g->md, &p);
}

cudaError_t launch_rb_resident(pg_grid *g, double omega, double tol, int64_t max_sweeps, int64_t s) {
  ClusterPlan p;
  if (!cluster_plan(g->md, &p)) return cudaErrorInvalidConfiguration;
  ClusterArgs a;
  a.d = g->md;
  a.gx = g->gx; a.gy = g->gy; a.gz = g->gze; a.b = g->b; a.invd = g->invd;
  a.V0 = g->V[0];
  a.V1 = g->V[1];
  a.omega = omega;
  a.tol = tol;
  a.max_sweeps = max_sweeps;
  a.s = s;
  a.rec = g->dev_sweeps;
  a.ctl = g->ctl;
  a.R = p.R;
  a.HPx = (g->md.NX + 1) / 2;
  const size_t smem = sizeof(double) * (size_t)p.R * g->md.L * g->md.NX;
  // function attributes apply to the device current when they are set: set
  // once per device (the flags are atomics, so concurrent grids on other
  // threads at worst set them twice)
  static std::atomic<bool> attr_set[64];
  if (g->dev < 0 || g->dev >= 64) return cudaErrorInvalidDevice;
  if (!attr_set[g->dev].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(k_rb_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_rb_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr_set[g->dev].store(true, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.ncta);
  cfg.blockDim = dim3(p.T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = g->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_rb_cluster, a);
}

// D-weighted squared 2-norms of both V buffers, sum_i d_i V_i^2 (d_i = 1 / invd_i,
// real nodes only), one partial per block (summed on the host in block order:
// deterministic for a fixed grid)
__global__ void k_dnorm2(int64_t np, const double *invd, const double *V0, const double *V1, double *part) {
  __shared__ double s0[256 / 32], s1[256 / 32];
  double a = 0.0, b = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
    const double id = invd[i];
    if (id > 0.0) {
      a += V0[i] * V0[i] / id;
      b += V1[i] * V1[i] / id;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s0[threadIdx.x >> 5] = a;
    s1[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      x += s0[k];
      y += s1[k];
    }
    part[2 * blockIdx.x] = x;
    part[2 * blockIdx.x + 1] = y;
  }
}

__global__ void k_probe(const double *V0, const double *V1, const DevCtl *c, const int64_t *idx,
                        int64_t n, double *out) {
  const double *V = c->base ? V1 : V0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = V[idx[k]];
}

__global__ void k_gather_mesh(MeshDims d, const double *V0, const double *V1, const DevCtl *c,
                              int64_t n, double *dst) {
  const double *V = c == nullptr ? V0 : (c->base ? V1 : V0);
  const int64_t per_layer = (int64_t)d.NY * d.NX;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = k / per_layer;
    const int64_t r = k - l * per_layer;
    const int64_t y = r / d.NX;
    const int64_t x = r - y * d.NX;
    dst[k] = V[mesh_index(d, l, y, x)];
  }
}

__global__ void k_scatter_mesh(MeshDims d, const double *src, int64_t n, double *dst) {
  const int64_t per_layer = (int64_t)d.NY * d.NX;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = k / per_layer;
    const int64_t r = k - l * per_layer;
    const int64_t y = r / d.NX;
    const int64_t x = r - y * d.NX;
    dst[mesh_index(d, l, y, x)] = src[k];
  }
}

__global__ void k_gather_perm(const int64_t *iperm, const double *V0, const double *V1,
                              const DevCtl *c, int64_t n, double *dst) {
  const double *V = c == nullptr ? V0 : (c->base ? V1 : V0);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = V[iperm[k]];
}

__global__ void k_scatter_perm(const int64_t *iperm, const double *src, int64_t n, double *dst) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[iperm[k]] = src[k];
}

__global__ void k_reset_state(DevCtl *c, int32_t keep_base) {
  if (!keep_base) c->base = 0;
  c->nonfinite = 0;
  c->done = 0;
  c->failed = 0;
  c->sweeps_total = 0;
  c->sweeps_max = 0;
  c->last_delta = 0.0;
  c->launches_done = 0;
  c->jbase = 0;
  c->diag_bad = 0;
  for (int k = 0; k < kRing; ++k) c->dmax[k] = 0ull;
}

// ================================================================= launchers
static inline int grid_for(int64_t work, int block, int num_sms) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = (int64_t)num_sms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// Resolved (F, S, D) of the temporally blocked mesh sweep: the requested
// options if that variant is compiled, else the largest compiled F <= fuse.
struct FusedCfg {
  int F, S, D, W;
};
int auto_rows_per_cta(const pg_grid *g, int F, int S, int W, int ny);
static FusedCfg fused_cfg_for(const pg_grid *g, int fuse);


// fuse = 0 (auto): F = 2 sweeps per launch (fastest per sweep on every
// measured grid, including the 8192-node config 0)
static FusedCfg fused_cfg(const pg_grid *g) { return fused_cfg_for(g, g->fuse > 0 ? g->fuse : 2); }

static FusedCfg fused_cfg_for(const pg_grid *g, int fuse) {
  const int L = g->md.L;
  const bool sl = g->slab && g->hx.G > 0;  // slab of a group: exchange-aware variants
  for (int F = fuse; F >= 1; --F) {
    // auto width: 64 column pairs per strip (half the x-halo share) for fused
    // launches where that variant fits in shared memory, else 32 (measured,
    // profiles/README.md)
    const int first = g->width == 64 || (g->width == 0 && F >= 2) ? 64 : 32;
    const int widths[2] = {first, 32};
    for (int W : widths) {
      const int D = g->lag;
      if (g->stages > 0 && fused_variant_exists(L, F, g->stages, D, W, sl)) return {F, g->stages, D, W};
      const int S = fused_default_stages(L, F, D);
      if (fused_variant_exists(L, F, S, D, W, sl)) return {F, S, D, W};
      const int S3 = fused_default_stages(L, F, 3);
      if (fused_variant_exists(L, F, S3, 3, W, sl)) return {F, S3, 3, W};
    }
  }
  return {1, 6, 3, 32};
}

bool colour_sweep(const pg_grid *g) { return g->kind == 0 && !g->slab && (g->colour || g->md.L > kMaxLayers); }

int sweeps_per_launch(pg_grid *g, int method) {
  if (resident_ok(g, method)) return 1;  // convergence tested after every sweep
  if (colour_sweep(g)) return 1;
  return (g->kind == 0 && method == PG_METHOD_RBSOR) ? fused_cfg(g).F : 1;
}

int fused_rows_per_cta(const pg_grid *g, int F, int S, int W, int ny) {
  if (g->rows > 0) return std::max(1, std::min(g->rows, ny));
  return auto_rows_per_cta(g, F, S, W, ny);
}

// rows per CTA so that strips x chunks fill one wave of resident CTAs
int auto_rows_per_cta(const pg_grid *g, int F, int S, int W, int ny) {
  const int I = fused_exact_lanes(F, W);
  const int strips = (g->md.HP + I - 1) / I;
  int chunks = (g->num_sms * fused_ctas_per_sm(g->md.L, S, W)) / strips;
  if (chunks < 1) chunks = 1;
  int H = (ny + chunks - 1) / chunks;
  if (H < 1) H = 1;
  return H;
}

cudaError_t launch_setup(pg_grid *g, double h) {
  const double inv_h = 1.0 / h;
  const int B = 256;
  if (g->kind == 0) {
    k_setup_gze<<<grid_for(g->np, B, g->num_sms), B, 0, g->stream>>>(g->np, g->gz, g->lz, h, g->gze);
    // no via above the top layer (the staged sweeps rely on it)
    cudaMemsetAsync(g->gze + (int64_t)(g->md.L - 1) * g->md.layer_stride, 0,
                    sizeof(double) * g->md.layer_stride, g->stream);
    k_diag_mesh<<<grid_for(g->np, B, g->num_sms), B, 0, g->stream>>>(g->md, g->gx, g->gy, g->gze,
                                                                      g->cap, inv_h, g->invd);
  } else {
    k_diag_csr<<<grid_for(g->np, B, g->num_sms), B, 0, g->stream>>>(g->np, g->rowptr, g->val, g->cap,
                                                                     inv_h, g->invd);
  }
  if (g->npad > 0) {
    k_setup_pad_ge<<<grid_for(g->npad, B, g->num_sms), B, 0, g->stream>>>(g->npad, g->pad_g, g->pad_l,
                                                                            h, g->pad_ge);
    k_diag_pads<<<grid_for(g->npad_grp, B, g->num_sms), B, 0, g->stream>>>(
        g->npad_grp, g->pad_grp, g->pad_idx, g->pad_ge, g->invd);
  }
  k_invert<<<grid_for(g->np, B, g->num_sms), B, 0, g->stream>>>(g->np, g->invd, g->md, g->kind == 0,
                                                                  g->ctl);
  return cudaGetLastError();
}

// right-hand side of the step ending at time t (loads evaluated at t); h may
// be +inf (DC analysis: capacitors open, inductor history dropped)
cudaError_t launch_rhs(pg_grid *g, double h, double t) {
  RhsArgs a;
  a.np = g->np;
  a.cap = g->cap;
  a.inv_h = 1.0 / h;
  a.V0 = g->V[0];
  a.V1 = g->V[1];
  a.ctl = g->ctl;
  a.b = g->b;
  const bool rlc_vias = g->kind == 0 && g->lz != nullptr;
  a.lz = rlc_vias ? g->lz : nullptr;
  a.gze = g->gze;
  a.iz = g->iz;
  a.layer_stride = g->kind == 0 ? g->md.layer_stride : 1;
  a.L = g->kind == 0 ? g->md.L : 1;
  a.pad_tile = g->npad > 0 ? g->pad_tile : nullptr;
  a.pad_grp = g->pad_grp;
  a.pad_idx = g->pad_idx;
  a.pad_ge = g->pad_ge;
  a.pad_l = g->pad_l;
  a.pad_i = g->pad_i;
  a.vdd = g->vdd;
  a.src_tile = g->nsrc > 0 ? g->src_tile : nullptr;
  a.src_grp = g->src_grp;
  a.src_idx = g->src_idx;
  a.src_ptr = g->src_ptr;
  a.pwl_t = g->pwl_t;
  a.pwl_i = g->pwl_i;
  a.t = t;
  a.ntile = g->ntile;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(g->ntile, (int64_t)g->num_sms * 8));
  k_rhs_fused<<<grid, 256, 0, g->stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(pg_grid *g) {
  k_check_finite<<<grid_for(g->np, 256, g->num_sms), 256, 0, g->stream>>>(g->np, g->V[0], g->V[1], g->ctl);
  return cudaGetLastError();
}

std::vector<int64_t> rhs_tile_starts(const std::vector<int64_t> &group_node, int64_t np) {
  const int64_t ntile = (np + kRhsTile - 1) / kRhsTile;
  std::vector<int64_t> t((size_t)ntile + 1);
  size_t q = 0;
  for (int64_t k = 0; k <= ntile; ++k) {
    const int64_t lo = k * (int64_t)kRhsTile;
    while (q < group_node.size() && group_node[q] < lo) ++q;
    t[(size_t)k] = (int64_t)q;
  }
  return t;
}

cudaError_t launch_sweep(pg_grid *g, int method, double omega, double tol, int j, int nsweeps,
                         int64_t *launches) {
  if (g->kind == 0) {
    if (method == PG_METHOD_RBSOR && colour_sweep(g)) {
      ColourArgs a;
      a.d = g->md;
      a.gx = g->gx; a.gy = g->gy; a.gz = g->gze; a.b = g->b; a.invd = g->invd;
      a.V0 = g->V[0];
      a.V1 = g->V[1];
      a.omega = omega; a.tol = tol; a.ctl = g->ctl; a.launch_idx = j;
      const int bx = (g->md.HP / 2 + 127) / 128;
      const int64_t rows = (int64_t)g->md.L * g->md.NY;
      const int by = (int)std::min<int64_t>(rows, std::max<int64_t>(1, (int64_t)g->num_sms * 16 / bx));
      for (int c = 0; c < 2; ++c) {
        a.colour = c;
        k_rb_colour_mesh<<<dim3(bx, by), 128, 0, g->stream>>>(a);
      }
      ++*launches;
      return cudaGetLastError();
    }
    if (method == PG_METHOD_RBSOR) {
      if (!tma_available(g)) return cudaErrorNotSupported;
      const FusedCfg c = fused_cfg(g);
      const int y0 = g->slab ? g->y_begin : 0, y1 = g->slab ? g->y_end : g->md.NY;
      ++*launches;
      if (g->pipe && c.F == 2 && nsweeps == 2 && sweep2_width(g->md.L) == c.W) {
        const int H2 = g->rows > 0 ? std::max(1, std::min(g->rows, y1 - y0)) : sweep2_rows_per_cta(g, y1 - y0);
        return launch_rb_sweep2(g, omega, tol, j, H2, y0, y1, g->slab ? g->ypar : 0, g->pdl_ok && j > 0);
      }
      const int H = fused_rows_per_cta(g, c.F, c.S, c.W, y1 - y0);
      return launch_rb_sweep_fused(g, omega, tol, j, nsweeps, c.F, c.S, c.D, c.W, H, y0, y1,
                                   g->slab ? g->ypar : 0);
    }
    JacobiArgs a;
    a.d = g->md;
    a.gx = g->gx; a.gy = g->gy; a.gz = g->gze; a.b = g->b; a.invd = g->invd;
    a.omega = omega; a.tol = tol; a.ctl = g->ctl; a.launch_idx = j;
    a.V0 = g->V[0];
    a.V1 = g->V[1];
    {
      const int bx = (g->md.NXP + 255) / 256;
      const int64_t rows = (int64_t)g->md.L * g->md.NY;
      const int by = (int)std::min<int64_t>(rows, std::max<int64_t>(1, (int64_t)g->num_sms * 8 / bx));
      k_jacobi_mesh<<<dim3(bx, by), 256, 0, g->stream>>>(a);
    }
    ++*launches;
  } else {
    CsrArgs a;
    a.rowptr = g->rowptr; a.col = g->col; a.val = g->val; a.b = g->b; a.invd = g->invd;
    a.omega = omega; a.tol = tol; a.launch_idx = j; a.ctl = g->ctl;
    a.V0 = g->V[0];
    a.V1 = g->V[1];
    if (method == PG_METHOD_RBSOR) {
      const bool staged = g->csr_stage && g->csr_staged_ok;
      if (staged) {
        static std::atomic<bool> attr_set[64];
        if (g->dev < 0 || g->dev >= 64) return cudaErrorInvalidDevice;
        if (!attr_set[g->dev].load(std::memory_order_acquire)) {
          cudaError_t e = cudaFuncSetAttribute(k_csr_sweep_staged, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(kCsrS * sizeof(CsrStage)));
          if (e != cudaSuccess) return e;
          // the shared-memory carveout is left to the driver: it fits the kCsrB
          // CTAs per SM, and asking for the maximum costs the gathers their L1
          // (126.4 vs 123.2 us per sweep on config 2, profiles/r2_s4/s4_csr_carve.txt)
          attr_set[g->dev].store(true, std::memory_order_release);
        }
      }
      bool prev_staged = staged;  // launch j - 1 (same grid, same kernel choice)
      a.pre = 0;
      for (int c = 0; c < g->ncolor; ++c) {
        a.r0 = g->color_ptr[c];
        a.r1 = g->color_ptr[c + 1];
        a.first = c == 0;
        const int64_t rows = a.r1 - a.r0;
        if (staged) {
          const int64_t tiles = (rows + kCsrR - 1) / kCsrR;
          const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, kCsrB * (int64_t)g->num_sms));
          // option "pdl": overlap this launch's first bulk copies with the
          // previous sweep launch (never with the RHS kernel, which writes b)
          a.pre = g->pdl_ok && (j > 0 || c > 0) && prev_staged ? 1 : 0;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(grid);
          cfg.blockDim = dim3(kCsrT);
          cfg.dynamicSmemBytes = kCsrS * sizeof(CsrStage);
          cfg.stream = g->stream;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          attr[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = attr;
          cfg.numAttrs = a.pre ? 1 : 0;
          cudaError_t e = cudaLaunchKernelEx(&cfg, k_csr_sweep_staged, a);
          if (e != cudaSuccess) return e;
          prev_staged = true;
        } else {
          k_csr_sweep<<<grid_for(rows, 256, g->num_sms), 256, 0, g->stream>>>(a);
        }
        ++*launches;
      }
    } else {
      a.r0 = 0;
      a.r1 = g->np;
      a.first = 1;
      k_csr_jacobi<<<grid_for(g->np, 256, g->num_sms), 256, 0, g->stream>>>(a);
      ++*launches;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_batch_advance(pg_grid *g, int nb) {
  k_batch_advance<<<1, 1, 0, g->stream>>>(g->ctl, nb);
  return cudaGetLastError();
}

cudaError_t launch_step_end(pg_grid *g, int64_t s, int launched, int flips, int fused,
                            int64_t max_sweeps, double tol) {
  const int count_epoch = g->slab && g->hx.G > 0 && g->hx.p2p && g->group_active;
  k_step_end<<<1, 1, 0, g->stream>>>(g->ctl, s, launched, flips, fused, max_sweeps, tol, g->dev_sweeps,
                                     count_epoch);
  return cudaGetLastError();
}

cudaError_t launch_inductor_update(pg_grid *g, double h) {
  const double inv_h = 1.0 / h;
  const int B = 256;
  if (g->kind == 0 && g->lz != nullptr && g->md.L > 1)
    k_ind_update_mesh<<<grid_for(g->np - g->md.layer_stride, B, g->num_sms), B, 0, g->stream>>>(
        g->md, g->V[0], g->V[1], g->ctl, g->gze, g->lz, inv_h, g->iz);
  if (g->npad > 0 && g->pad_l != nullptr)
    k_ind_update_pads<<<grid_for(g->npad, B, g->num_sms), B, 0, g->stream>>>(
        g->npad, g->pad_idx, g->pad_ge, g->pad_l, g->V[0], g->V[1], g->ctl, g->vdd, inv_h, g->pad_i);
  return cudaGetLastError();
}

cudaError_t launch_probe(pg_grid *g, const int64_t *probe_idx, int64_t n_probe, double *out) {
  if (n_probe <= 0) return cudaSuccess;
  k_probe<<<grid_for(n_probe, 256, g->num_sms), 256, 0, g->stream>>>(g->V[0], g->V[1], g->ctl,
                                                                      probe_idx, n_probe, out);
  return cudaGetLastError();
}

cudaError_t launch_reset_state(pg_grid *g, bool keep_base) {
  k_reset_state<<<1, 1, 0, g->stream>>>(g->ctl, keep_base ? 1 : 0);
  return cudaGetLastError();
}

int dnorm2_blocks(const pg_grid *g) { return grid_for(g->np, 256, g->num_sms); }

cudaError_t launch_dnorm2(pg_grid *g, double *part) {
  k_dnorm2<<<dnorm2_blocks(g), 256, 0, g->stream>>>(g->np, g->invd, g->V[0], g->V[1], part);
  return cudaGetLastError();
}

cudaError_t launch_gather_user(pg_grid *g, double *dst) {
  if (g->kind == 0)
    k_gather_mesh<<<grid_for(g->n, 256, g->num_sms), 256, 0, g->stream>>>(g->md, g->V[0], g->V[1],
                                                                          g->ctl, g->n, dst);
  else
    k_gather_perm<<<grid_for(g->n, 256, g->num_sms), 256, 0, g->stream>>>(g->iperm, g->V[0], g->V[1],
                                                                          g->ctl, g->n, dst);
  return cudaGetLastError();
}

cudaError_t launch_scatter_user(pg_grid *g, const double *src, double *dst) {
  if (g->kind == 0)
    k_scatter_mesh<<<grid_for(g->n, 256, g->num_sms), 256, 0, g->stream>>>(g->md, src, g->n, dst);
  else
    k_scatter_perm<<<grid_for(g->n, 256, g->num_sms), 256, 0, g->stream>>>(g->iperm, src, g->n, dst);
  return cudaGetLastError();
}

}  // namespace pgb
