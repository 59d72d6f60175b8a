// Kernel templates of the temporally blocked red-black SOR sweep (included by
// pg_sweep_fused.cu and the instantiation units pg_sweep_fused_i*.cu).
#pragma once
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
// last reader ran.  Layers are coupled by vias (other warps) and a via joins
// nodes of the same row, so a node's z-neighbours are read only in the same
// phase of the same row: one __syncthreads between phase A and phase B per
// step orders every cross-warp access (for D >= 3, phase B(y) and phase A(y+1)
// touch no common value of another warp).  The TMA refill of the slot of row
// y - D(F-1) - 3 (last read in phase B(y-1)) is issued right after that
// barrier, after a proxy fence (the slot was written by generic stores).
// Ring: the rows read around one barrier span D (F-1) + 5 rows; the remaining
// stages are TMA prefetch depth.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <type_traits>

#include "pg_internal.h"

namespace pgb {

namespace {

// W = column pairs per strip (32: one warp per layer row, 64: two); a strip
// row of one layer holds RW = 2 W doubles (W even columns, then W odd ones)

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
// tx-count only (no arrival): the phase still needs its arrival
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
// box {32 half-columns from c0, both parities, row y, all layers}
__device__ __forceinline__ void tma4(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int y) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(0), "r"(y), "r"(0)
      : "memory");
}
// the same box with an L2 cache-eviction policy (createpolicy)
__device__ __forceinline__ void tma4h(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int y,
                                      uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(0), "r"(y), "r"(0), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void stg_hint(double *p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// L2 prefetch of the same box (no shared memory, no completion): rows beyond
// the ring are pulled into L2 early so the ring's TMA loads see L2 latency
__device__ __forceinline__ void tma4_prefetch(const CUtensorMap *map, int c0, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(0), "r"(y), "r"(0)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace

// Optional cycle instrumentation (build with -DPG_PROF; debugging only):
// per-warp clock sums of the streaming-step phases, read by pg_debug_prof.
#ifdef PG_PROF
#define PROF_T(var) const long long var = clock64()
#define PROF_ADD(k, a, b) prof[k] += (unsigned long long)((b) - (a))
#else
#define PROF_T(var)
#define PROF_ADD(k, a, b)
#endif

#ifndef PG_L2_AHEAD
#define PG_L2_AHEAD 4  // rows of L2 prefetch beyond the shared-memory ring
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
  unsigned long long *prof; // PG_PROF builds: 8 cycle counters (else unused)
  // slab of a partitioned mesh (pg_group): the G ghost rows below y_begin /
  // from y_end are read from the receive buffers the exchange filled (maps
  // mRlo / mRhi, rows [0, G) each), and the G owned rows next to each boundary
  // are also written to the send buffers ([L][G][NXP] rows, parity-split)
  CUtensorMap mRlo, mRhi;
  double *send_lo, *send_hi;
  int32_t has_rlo, has_rhi, G;
  int32_t pre;      // k_rb_sweep2: the previous kernel in the stream is a sweep launch (PDL prologue)
  int32_t l2keep;   // k_rb_sweep2: bit a < 5: constant array a (gx, gy, gz_eff, b, 1/d) read with L2 evict_last;
                    // bit 5: V written with evict_last (the next launch reads it)
  int32_t l2first;  // k_rb_sweep2: arrays read with evict_first (bits as above, bit 5: V reads); others evict_normal
  // k_rb_sweep2 slab with the peer-memory exchange (SlabHalo::p2p)
  CUtensorMap mRlo_b, mRhi_b;  // parity-1 receive buffers
  int32_t p2p, nranks;
  double *peer_lo[2], *peer_hi[2];
  unsigned long long *sig_all[8], *pnorm_all[8];
};

// The constants of one node update: x links (west, east), y links (north,
// south), vias (up, down), b and 1/d.
struct NodeC {
  double gxOwn, gxOth, gyN, gyS, gzU, gzD, b, id;
};

// Loads a node's constants from its staged row Ry (row r-1 in Rn).  The x
// links are taken by neighbour rather than by direction: the link to the
// other node of my own pair is always the even node's gx (offset pe), the link
// to the neighbouring lane's node is gx at `oth_link` (the odd node's for an
// odd node, the previous pair's odd node's for an even node), so the update
// needs no parity-dependent value selects.  The south link is taken from `gyS`
// when the caller already holds it (gyS_known).
template <int L, int RW, bool gyS_known = false>
__device__ __forceinline__ NodeC load_c(const double *Ry, const double *Rn, int me, int pe, int oth_link,
                                        bool has_down, double gyS = 0.0) {
  constexpr int LAY = L * RW;
  constexpr int GX = 1 * LAY, GY = 2 * LAY, GZ = 3 * LAY, BB = 4 * LAY, ID = 5 * LAY;
  NodeC c;
  c.gxOwn = Ry[GX + pe];
  c.gxOth = Ry[GX + oth_link];
  c.gyN = Rn[GY + me];
  c.gyS = gyS_known ? gyS : Ry[GY + me];
  c.gzU = Ry[GZ + me];
  c.gzD = has_down ? Ry[GZ + me - RW] : 0.0;
  c.b = Ry[BB + me];
  c.id = Ry[ID + me];
  return c;
}

// Eq. (13) + (15) from the constants and the neighbour values: Vown / Voth the
// x neighbours in my lane / the neighbouring lane, VN / VS rows r-1 / r+1,
// VU / VD via neighbours in layers l+1 / l-1 (gzD = 0 in layer 0 cancels VD).
__device__ __forceinline__ double upd_c(const NodeC &c, double w, double Vc, double Vown, double Voth,
                                        double VN, double VS, double VU, double VD) {
#ifdef PG_DIAG_NOFP
  // diagnostic build only (tools/power_trace.py experiments): every operand is
  // still loaded, but the update is integer bit mixing masked to zero by a
  // runtime condition the compiler cannot fold (omega is never > 100), so the
  // kernel moves the same data without its fp64 arithmetic
  const unsigned long long m = w > 100.0 ? ~0ull : 0ull;
  auto u = [](double x) { return (unsigned long long)__double_as_longlong(x); };
  const unsigned long long x = u(c.gxOwn) ^ u(Vown) ^ u(c.gxOth) ^ u(Voth) ^ u(c.gyN) ^ u(VN) ^ u(c.gyS) ^
                               u(VS) ^ u(c.gzU) ^ u(VU) ^ u(c.gzD) ^ u(VD) ^ u(c.b) ^ u(c.id);
  return __longlong_as_double((long long)(u(Vc) ^ (x & m)));
#endif
  double s1 = fma(c.gxOwn, Vown, c.b);
  s1 = fma(c.gxOth, Voth, s1);
  s1 = fma(c.gyN, VN, s1);
  double s2 = c.gyS * VS;
  s2 = fma(c.gzU, VU, s2);
  s2 = fma(c.gzD, VD, s2);
  return fma(w, (s1 + s2) * c.id - Vc, Vc);
}

template <int L, int F, int S, int D, int W, bool SLAB>
__global__ void __launch_bounds__(W * L) k_rb_sweep_fused(const __grid_constant__ FusedParams P) {
  static_assert(D >= 3, "levels must trail by >= 3 rows");
  static_assert(S >= D * (F - 1) + 5, "ring too small for the wavefront");
  static_assert(S % D == 0, "S must be a multiple of D (compile-time register FIFO index)");
  static_assert(W == 32 || W == 64, "strip width W must be 32 or 64 pairs");
  constexpr int RW = 2 * W;      // doubles per layer row of a strip
  constexpr int kGuard = RW;     // zeroed guard band (doubles) before and after the ring
  constexpr int NWL = W / 32;    // warps per layer row
  constexpr int LAY = L * RW;
  constexpr int SE = 6 * LAY;  // doubles per stage
  constexpr int GX = 1 * LAY, GY = 2 * LAY, GZ = 3 * LAY, BB = 4 * LAY, ID = 5 * LAY;
  constexpr uint32_t STAGE_BYTES = SE * 8u;
  // x halo: F pairs per side suffice; it is rounded up to even so that the TMA
  // box starts on a 16-byte boundary (odd pair offsets fault)
  constexpr int FH = (F + 1) & ~1;
  constexpr int I = W - 2 * FH;  // exact pairs per strip
  extern __shared__ __align__(128) double smem_f[];
  __shared__ uint64_t full_bar[S];
  __shared__ double wmax[L * NWL];
  double *ring = smem_f + kGuard;

  const int lane = threadIdx.x, l = threadIdx.y;  // lane: pair index in the strip, 0..W-1
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
    const int t = l * W + lane;
    for (int k = t; k < kGuard; k += W * L) {
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
  // V of row r: ghost rows of a slab come from the exchange's receive buffers
  auto v_src = [&](int r, int &rr) -> const CUtensorMap * {
    if constexpr (SLAB) {
      if (P.has_rlo && r < P.y_begin) {
        rr = r - (P.y_begin - P.G);
        return &P.mRlo;
      }
      if (P.has_rhi && r >= P.y_end) {
        rr = r - P.y_end;
        return &P.mRhi;
      }
    }
    rr = r;
    return mVin;
  };
  auto issue_slot = [&](int r, int s) {
    double *st = ring + s * SE;
    mbar_expect_tx(&full_bar[s], STAGE_BYTES);
    int rv;
    const CUtensorMap *mv = v_src(r, rv);
    tma4(st, mv, &full_bar[s], ps, rv);
    tma4(st + GX, &P.mgx, &full_bar[s], ps, r);
    tma4(st + GY, &P.mgy, &full_bar[s], ps, r);
    tma4(st + GZ, &P.mgz, &full_bar[s], ps, r);
    tma4(st + BB, &P.mb, &full_bar[s], ps, r);
    tma4(st + ID, &P.mid, &full_bar[s], ps, r);
  };
  // rows R + kL2Ahead are prefetched into L2 when row R is loaded into the ring
  constexpr int kL2Ahead = PG_L2_AHEAD;
  auto prefetch_row = [&](int r) {
    int rv;
    const CUtensorMap *mv = v_src(r, rv);
    tma4_prefetch(mv, ps, rv);
    tma4_prefetch(&P.mgx, ps, r);
    tma4_prefetch(&P.mgy, ps, r);
    tma4_prefetch(&P.mgz, ps, r);
    tma4_prefetch(&P.mb, ps, r);
    tma4_prefetch(&P.mid, ps, r);
  };
  if (leader) {
    for (int r = r_first; r < r_first + S && r <= r_last; ++r) issue_slot(r, r - r_first);
    if (kL2Ahead > 0)
      for (int r = r_first + S; r < r_first + S + kL2Ahead && r <= r_last; ++r) prefetch_row(r);
  }

  const double w = P.omega;
  const int pe = l * RW + lane;          // my even-column node in an array block
  const int po = pe + W;                 // my odd-column node
  const int gp = ps + lane;              // my pair (global half-column)
  const bool exact_lane = lane >= FH && lane < FH + I && gp < P.HP;
  const bool has_down = l > 0;
  const int lpar = (l + P.ypar) & 1;
  double *vout_e = Vout + (int64_t)l * P.layer_stride + gp;
  double *vout_o = vout_e + P.HP;
  double dmax = 0.0;

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
  // FIFO index of step y: (y - r_first - 1) mod D == u mod D
  constexpr auto md3 = [](int a) { return ((a % D) + D) % D; };
  auto sweep_pass = [&](const int last) {
    const int y_end_loop = r_last + D * last;
    double redF[F][D], blkF[F][D];  // values this thread stored at the last D steps
    // F == 2: constants level 0 loaded at the last D steps (level 1 reuses them)
    constexpr bool kReuseC = F == 2;
    NodeC cRedF[kReuseC ? D : 1], cBlkF[kReuseC ? D : 1];
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
      for (int k = 0; k < D; ++k) redF[f][k] = blkF[f][k] = 0.0;
    // one streaming step; `steady`: the D previous steps ran in this launch, so
    // operands this thread produced come from the register FIFOs
    auto step = [&](const int u, const int y, auto steady_tag) {
      constexpr bool steady = decltype(steady_tag)::value;
      PROF_T(t0);
      if (y + 1 <= r_last) wait_k(y + 1 - r_first, md(2 + u));
      PROF_T(t1);
      // -------------------------------------------- phase A: red_f(y - D f)
      // Operands this thread produced earlier come from registers: for level
      // f >= 1, red_{f-1}(r) (D steps ago) and black_{f-1}(r+1), (r), (r-1)
      // (D-2, D-1, D steps ago), once the stream is steady.
      double dA = 0.0;
      double vA[F], cA[F], nA[F], gA[F];
      {
        double *ad[F];
        NodeC c0;
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const int r = y - D * f;
          const int e = lpar ^ (r & 1);
          const double *Ry = ring + md(1 + u - D * f) * SE;
          const double *Rn = ring + md(u - D * f) * SE;
          const double *Rs = ring + md(2 + u - D * f) * SE;
          const int me = e ? po : pe, own = e ? pe : po, oth = e ? pe + 1 : po - 1;
          double Vc, Vown, VN, VS;
          if (f > 0 && steady) Vc = redF[f - 1][md3(u - D)]; else Vc = Ry[me];
          if (f > 0 && steady) Vown = blkF[f - 1][md3(u - D + 1)]; else Vown = Ry[own];
          if (f > 0 && steady) VN = blkF[f - 1][md3(u - D)]; else VN = Rn[me];
          if (f > 0 && steady) VS = blkF[f - 1][md3(u - D + 2)]; else VS = Rs[me];
          const double Voth = Ry[oth];
          // constants: level 1 of a 2-sweep launch reuses those level 0 loaded
          // for the same node D steps ago
          NodeC c;
          if (kReuseC && f == 1 && steady) c = cRedF[md3(u - D)];  // (== md3(u): read before the push)
          else c = load_c<L, RW>(Ry, Rn, me, pe, e ? po : po - 1, has_down);
          if (kReuseC && f == 0) c0 = c;
          ad[f] = const_cast<double *>(Ry) + me;
          vA[f] = upd_c(c, w, Vc, Vown, Voth, VN, VS, Ry[me + RW], Ry[me - RW]);
          cA[f] = Vc;
          nA[f] = VN;
          gA[f] = c.gyN;
        }
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const int r = y - D * f;
          const bool in = f <= last && r > r_first && r < r_last;
          if (in) *ad[f] = vA[f];
          const double d = fabs(vA[f] - cA[f]);
          dA = f == last ? d : dA;
          vA[f] = in ? vA[f] : cA[f];  // the value the row now holds
        }
        if (kReuseC) cRedF[md3(u)] = c0;
      }
      {
        const int r = y - D * last;
        if (!(r >= ys && r < ye && exact_lane)) dA = 0.0;
      }
      PROF_T(t2);
      fence_proxy_async();
      __syncthreads();
      PROF_T(t3);
      {
        // phase B(y-1) has finished in every warp: its lowest row is dead
        const int R = y - D * (F - 1) - 3 + S;
        if (leader && R <= r_last && R >= r_first + S) {
          issue_slot(R, md(u - D * (F - 1) - 2));
          if (kL2Ahead > 0 && R + kL2Ahead <= r_last) prefetch_row(R + kL2Ahead);
        }
      }
      // -------------------------------------------- phase B: black_f(y - D f - 1)
      // black_f(r-1) has the column parity of red_f(r): its own value and
      // south link are phase A's north operands, its south neighbour is
      // red_f(r), its north neighbour red_f(r-2) (2 steps ago) and its
      // own-lane x neighbour red_f(r-1) (1 step ago).
      double dB = 0.0;
      double vB[F];
      {
        double cB[F], *ad[F];
        NodeC c0;
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const int r = y - D * f - 1;
          const int e = lpar ^ (r & 1) ^ 1;
          const double *Ry = ring + md(u - D * f) * SE;
          const double *Rn = ring + md(u - 1 - D * f) * SE;
          const int me = e ? po : pe, own = e ? pe : po, oth = e ? pe + 1 : po - 1;
          const double Vc = nA[f];
          double Vown, VN;
          if (steady) Vown = redF[f][md3(u - 1)]; else Vown = Ry[own];
          if (steady) VN = redF[f][md3(u - 2)]; else VN = Rn[me];
          const double Voth = Ry[oth];
          NodeC c;
          if (kReuseC && f == 1 && steady) c = cBlkF[md3(u - D)];
          else c = load_c<L, RW, true>(Ry, Rn, me, pe, e ? po : po - 1, has_down, gA[f]);
          if (kReuseC && f == 0) c0 = c;
          ad[f] = const_cast<double *>(Ry) + me;
          vB[f] = upd_c(c, w, Vc, Vown, Voth, VN, vA[f], Ry[me + RW], Ry[me - RW]);
          cB[f] = Vc;
        }
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const int r = y - D * f - 1;
          const bool in = f <= last && r > r_first && r < r_last;
          if (in) *ad[f] = vB[f];
          const double d = fabs(vB[f] - cB[f]);
          dB = f == last ? d : dB;
          vB[f] = in ? vB[f] : cB[f];
        }
        if (kReuseC) cBlkF[md3(u)] = c0;
      }
      PROF_T(t4);
      // register FIFOs: entry (step index mod D); S % D == 0 keeps it a
      // compile-time index across blocks of S unrolled steps
#pragma unroll
      for (int f = 0; f < F; ++f) {
        redF[f][md3(u)] = vA[f];
        blkF[f][md3(u)] = vB[f];
      }
      const int ro = y - D * last - 1;  // row finished by the last level
      const bool out_row = ro >= ys && ro < ye && exact_lane;
      if (!out_row) dB = 0.0;
      dA = dA > dB ? dA : dB;
      dmax = dA > dmax ? dA : dmax;
      if (out_row) {
        // both colours of row ro are final: black from this step, red from the
        // previous one (registers on the steady path, else the staged row)
        double ve, vo;
        if (steady && last == F - 1) {
          const double vb = vB[F - 1], vr = redF[F - 1][md3(u - 1)];
          const bool eb = lpar ^ (ro & 1) ^ 1;
          ve = eb ? vr : vb;
          vo = eb ? vb : vr;
        } else {
          const double *R = ring + md(u - D * last) * SE;
          ve = R[pe];
          vo = R[po];
        }
        vout_e[(int64_t)ro * P.NXP] = ve;
        vout_o[(int64_t)ro * P.NXP] = vo;
        // slab boundary rows also go to the exchange's send buffers
        if constexpr (SLAB) {
          if (P.send_lo && ro < P.y_begin + P.G) {
            double *sb = P.send_lo + ((int64_t)l * P.G + (ro - P.y_begin)) * P.NXP;
            sb[gp] = ve;
            sb[gp + P.HP] = vo;
          }
          if (P.send_hi && ro >= P.y_end - P.G) {
            double *sb = P.send_hi + ((int64_t)l * P.G + (ro - (P.y_end - P.G))) * P.NXP;
            sb[gp] = ve;
            sb[gp + P.HP] = vo;
          }
        }
      }
      PROF_T(t5);
      PROF_T(t6);
      PROF_ADD(0, t0, t1);
      PROF_ADD(1, t1, t2);
      PROF_ADD(2, t2, t3);
      PROF_ADD(3, t3, t4);
      PROF_ADD(4, t4, t5);
      PROF_ADD(5, t5, t6);
    };
    // warm-up steps y = r_first + 1 .. r_first + D, then the steady stream
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const int y = r_first + 1 + u;
      if (y > y_end_loop) break;
      step(u, y, std::false_type{});
    }
    for (int y0 = r_first + 1; y0 <= y_end_loop; y0 += S) {
#pragma unroll
      for (int u = 0; u < S; ++u) {
        const int y = y0 + u;
        if (y > y_end_loop) break;
        if (u < D && y0 == r_first + 1) continue;
        step(u, y, std::true_type{});
      }
    }
  };
  if (nsw == F)
    sweep_pass(F - 1);
  else
    sweep_pass(nsw - 1);
#ifdef PG_PROF
  if ((lane & 31) == 0)
    for (int k = 0; k < 6; ++k) atomicAdd(&P.prof[k], prof[k]);
  if ((lane & 31) == 0) atomicAdd(&P.prof[6], 1ull);
#endif
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if ((lane & 31) == 0) wmax[l * NWL + (lane >> 5)] = dmax;
  __syncthreads();
  if (leader) {
    double m = 0.0;
#pragma unroll
    for (int k = 0; k < L * NWL; ++k) m = fmax(m, wmax[k]);
    atomicMax(&ctl->dmax[j & (kRing - 1)], static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

constexpr size_t fused_smem(int L, int S, int W) { return ((size_t)S * 6 * L * 2 * W + 2 * 2 * W) * 8; }

template <int L, int F, int S, int D, int W, bool SLAB>
cudaError_t launch_fused_t(pg_grid *g, const FusedParams &P, dim3 grid) {
  auto kern = k_rb_sweep_fused<L, F, S, D, W, SLAB>;
  const size_t smem = fused_smem(L, S, W);
  if (g->tma_kernel_set != (const void *)kern || g->tma_smem_set != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
    g->tma_kernel_set = (const void *)kern;
    g->tma_smem_set = smem;
  }
  kern<<<grid, dim3(W, L), smem, g->stream>>>(P);
  return cudaGetLastError();
}

// Compiled variants (L, F, S, D, W): W = 32 for every L in 1..8 with F = 1..4
// at D = 3 and 2 prefetch stages (S = 3(F-1) + 6) where the ring fits in
// 227 KB, W = 64 (halved x-halo share) where it fits, and a few D = 4 / other
// prefetch depths for tuning (options "lag", "stages", "width").
#define PG_FUSED_CASES(X)                                                                   \
  X(1, 1, 6, 3, 32) X(1, 2, 9, 3, 32) X(1, 3, 12, 3, 32) X(1, 4, 15, 3, 32)                 \
  X(2, 1, 6, 3, 32) X(2, 2, 9, 3, 32) X(2, 3, 12, 3, 32) X(2, 4, 15, 3, 32)                 \
  X(3, 1, 6, 3, 32) X(3, 2, 9, 3, 32) X(3, 3, 12, 3, 32) X(3, 4, 15, 3, 32)                 \
  X(4, 1, 6, 3, 32) X(4, 2, 9, 3, 32) X(4, 3, 12, 3, 32) X(4, 4, 15, 3, 32)                 \
  X(5, 1, 6, 3, 32) X(5, 2, 9, 3, 32) X(5, 3, 12, 3, 32)                                    \
  X(6, 1, 6, 3, 32) X(6, 2, 9, 3, 32) X(6, 3, 12, 3, 32)                                    \
  X(7, 1, 6, 3, 32) X(7, 2, 9, 3, 32)                                                       \
  X(8, 1, 6, 3, 32) X(8, 2, 9, 3, 32)                                                       \
  X(1, 2, 12, 4, 32) X(2, 2, 12, 4, 32) X(3, 2, 12, 4, 32) X(4, 2, 12, 4, 32) \
  X(1, 1, 6, 3, 64) X(1, 2, 9, 3, 64) X(1, 3, 12, 3, 64) X(1, 4, 15, 3, 64)                 \
  X(2, 1, 6, 3, 64) X(2, 2, 9, 3, 64) X(2, 3, 12, 3, 64)                                    \
  X(3, 1, 6, 3, 64) X(3, 2, 9, 3, 64) X(4, 1, 6, 3, 64) X(4, 2, 9, 3, 64)

// Variants compiled with slab (ghost-row exchange) support: the defaults
// F = 2 (W = 64 where it fits, else 32) and F = 1 for every L.
#define PG_FUSED_SLAB_CASES(X)                                                                   \
  X(1, 2, 9, 3, 64) X(2, 2, 9, 3, 64) X(3, 2, 9, 3, 64) X(4, 2, 9, 3, 64)                          \
  X(5, 2, 9, 3, 32) X(6, 2, 9, 3, 32) X(7, 2, 9, 3, 32) X(8, 2, 9, 3, 32)                          \
  X(1, 1, 6, 3, 32) X(2, 1, 6, 3, 32) X(3, 1, 6, 3, 32) X(4, 1, 6, 3, 32)                          \
  X(5, 1, 6, 3, 32) X(6, 1, 6, 3, 32) X(7, 1, 6, 3, 32) X(8, 1, 6, 3, 32)

// FusedParams of a launch over rows [y_begin, y_end) (false: no TMA maps)
bool fill_fused_params(pg_grid *g, FusedParams &P, double omega, double tol, int j, int nsw, int W,
                       int rows_per_cta, int y_begin, int y_end, int ypar);

constexpr int fused_key(int L, int F, int S, int D, int W, bool slab = false) {
  return ((((L * 8 + F) * 32 + S) * 8 + D) * 2 + (W == 64)) * 2 + (slab ? 1 : 0);
}


}  // namespace pgb
