// Two-level red-black SOR pipeline (sm_100a): the default mesh relaxation
// kernel for full launches of F = 2 sweeps (option "pipe", default on).
#pragma once
//
// Same arithmetic and halo scheme as k_rb_sweep_fused<L, 2, ...> (header of
// pg_sweep_fused.cuh; Eq. (13) with the SOR blend of Eq. (15), §IV, in
// the red-black numbering of DESIGN.md R12): two sweeps per streaming pass,
// rows [ys - 4, ye + 4) staged, lanes [2, W - 2) and rows [ys, ye) exact.  What
// differs is the instruction stream of a streaming step:
//
// * Spread TMA issue.  W * L threads (lane = column pair, one layer per W
//   lanes); after the one CTA barrier per step the refill of the slots that
//   barrier proved dead is issued by lane 0 of several warps, one copy each
//   (the mbarrier's tx-count may go transiently negative, its single arrival
//   is the expect_tx), so no warp carries the whole issue sequence.  (A
//   separate producer warp would make 9 warps: 3 on one SM sub-partition,
//   which caps the registers at 168 per thread.)
// * Split rings.  V rows go through a 12-stage ring (4 KB per stage), the five
//   node-constant arrays (gx, gy, gz_eff, b, 1/d) through a 6-stage ring: the
//   second sweep level takes its constants from registers (loaded by the first
//   level 3 rows earlier), so constant rows are live for 2 steps only.  A
//   12-step unrolled body then makes every ring slot, mbarrier phase, register
//   FIFO index (depth 3) and red/black column parity a compile-time constant;
//   the only runtime parity is per warp (q below), folded into 7 per-thread
//   shared-memory offsets computed once.
// * One body for every step.  The first and last steps run the same
//   unguarded body as the steady state (no cold warm-up / tail code: the
//   kernel's whole streaming loop is one 12-step block); only the norm and the
//   write-out are masked to the owned rows.
// * Registers first.  Every V operand this thread produced or loaded earlier
//   comes from a register FIFO; shared memory is read only for values of other
//   threads (x neighbour in the next/previous lane, z neighbours in other
//   warps) and for new rows.  The second level's black values feed no later
//   update, so they are never stored to shared memory, only written out.
// * A zero "layer -1" block before the gz_eff array of each constant stage
//   makes the layer-0 lower via conductance 0 without a branch.
// * Small loop code: the 12-step body is larger than the instruction cache,
//   so each refill site holds one copy instruction sequence with computed
//   operands and an explicit L2 policy (auto: stream the reads, keep the
//   written V for the next launch), and the proxy fence that orders the
//   ring's generic accesses before its TMA refills runs every second step.
// * Programmatic dependent launch as an option ("pdl", off by default:
//   measured slower; constant rows requested before griddepcontrol.wait)
//   and, in a peer-memory slab group, the halo exchange and the global norm
//   fused into the kernel's tail.
//
// Streaming step y (u = y - r_first - 1, compile-time modulo 12):
//   phase A: red_0(y), red_1(y - 3)          | (fence.proxy.async); barrier
//   phase B: black_0(y - 1), black_1(y - 4)  | write row y - 4 (both colours)
// Phase B(y) and phase A(y + 1) run in one barrier interval (loop body).
// red_1(r) needs black_0(r - 1 .. r + 1) (steps <= y - 1), black_0(r) needs
// red_0(r - 1 .. r + 1) (phase A of this step or before), black_1(r) needs
// red_1(r - 1 .. r + 1).  Cross-warp operands (z neighbours, lanes 31/32 of a
// layer row) are read only in the phase after the barrier that follows their
// write, as in pg_sweep_fused.cuh.
// Barrier of step y: phase B(y - 1) is complete, so the constant row y - 2
// and the V row y - 6 (and older) are dead; they are refilled with
// constant row y + 4 and V row y + 5 (one mbarrier "group" per row pair).
#include "pg_sweep_fused.cuh"

#include <utility>

namespace pgb {

template <int L, int W>
struct Sweep2Geo {
  static constexpr int RW = 2 * W;                    // doubles per layer row of a strip
  static constexpr int LAY = L * RW;                  // doubles per array row (all layers)
  static constexpr int NC = W * L;                    // compute threads
  static constexpr int NT = NC;                       // threads per CTA
  static constexpr int NWARP = NC / 32;
  static constexpr int SV = 12, SC = 6;               // ring stages (V, constants)
  static constexpr int VST = LAY;                     // doubles per V stage
  static constexpr int CGX = 0, CGY = LAY, CZ0 = 2 * LAY, CGZ = 2 * LAY + RW, CB = 3 * LAY + RW,
                       CID = 4 * LAY + RW;            // constant stage: gx, gy, [zero layer], gz, b, 1/d
  static constexpr int CST = 5 * LAY + RW;            // doubles per constant stage
  static constexpr int GUARD = RW;                    // zero band before and after the V ring
  static constexpr int VOFF = GUARD;                  // V ring offset (doubles)
  static constexpr int COFF = GUARD + SV * VST + GUARD;
  static constexpr size_t SMEM = (size_t)(COFF + SC * CST) * 8;
  static constexpr uint32_t VBYTES = VST * 8u, CBYTES = 5u * LAY * 8u;
  static constexpr int FH = 2, I = W - 2 * FH;        // x halo (F = 2), exact pairs per strip
};

template <int L, int W, bool SLAB>
__global__ void __launch_bounds__(W * L, 1) k_rb_sweep2(const __grid_constant__ FusedParams P) {
  using Gm = Sweep2Geo<L, W>;
  constexpr int RW = Gm::RW, NT = Gm::NT, SV = Gm::SV, SC = Gm::SC;
  constexpr int VST = Gm::VST, CST = Gm::CST;
  constexpr int CGX = Gm::CGX, CGY = Gm::CGY, CGZ = Gm::CGZ, CB = Gm::CB, CID = Gm::CID;
  constexpr int FH = Gm::FH, I = Gm::I;
  extern __shared__ __align__(128) double sm2[];
  __shared__ uint64_t gbar[SC];
  double *vring = sm2 + Gm::VOFF;
  double *cring = sm2 + Gm::COFF;

  const int tid = threadIdx.x;
  DevCtl *ctl = P.ctl;
  const int ps = blockIdx.x * I - FH;  // first pair of the strip (even)
  const int ys = P.y_begin + blockIdx.y * P.rows_per_cta;
  const int ye = min(ys + P.rows_per_cta, P.y_end);
  const int r_first = ys - 4, r_last = ye + 3;
  const int n_init = min(SC, r_last - r_first + 1);  // groups issued before the loop

  // zero bands: before / after the V ring, the "layer -1" block of every constant stage
  for (int k = tid; k < RW; k += NT) {
    sm2[k] = 0.0;
    vring[SV * VST + k] = 0.0;
  }
  for (int k = tid; k < SC * RW; k += NT) cring[(k / RW) * CST + Gm::CZ0 + (k % RW)] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < SC; ++s) mbar_init(&gbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Programmatic dependent launch: when the previous kernel in the stream is
  // a sweep launch (P.pre), the node constants are not among its outputs, so
  // the first constant rows are requested before waiting for it; V and the
  // control block are read only after griddepcontrol.wait.  (Without the
  // launch attribute the wait is a no-op.)
  const CUtensorMap *mC = &P.mgx;
  // L2 eviction policy per array (options "l2keep" / "l2first", auto by
  // footprint, pg_sweep2.cu): evict_last / evict_first hints on the TMA
  // copies; policy 0 = plain copy without a cache hint (measured faster than
  // an explicit evict_normal hint on config 4)
  const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first(),
                 pol_normal = policy_evict_normal();
  auto pol = [&](int a) -> uint64_t {
    return (a < 5 && ((P.l2keep >> a) & 1)) ? pol_last : (((P.l2first >> a) & 1) ? pol_first : pol_normal);
  };
  // one copy instruction sequence per call site (the refill code is
  // replicated in each of the 12 unrolled steps)
  auto tma = [&](void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int y, uint64_t p) {
    tma4h(dst, map, bar, c0, y, p);
  };

  auto c_dst = [&](int r, int a) { return cring + ((r - r_first) % SC) * CST + a * Gm::LAY + (a >= 2 ? RW : 0); };
  auto c_bar = [&](int r) { return &gbar[(r - r_first) % SC]; };
  if (P.pre && tid == 0) {
    for (int r = r_first; r < r_first + n_init; ++r) {
      mbar_expect_tx_only(c_bar(r), Gm::CBYTES);
      for (int a = 0; a < 5; ++a) tma(c_dst(r, a), mC + a, c_bar(r), ps, r, pol(a));
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int j = *(volatile int32_t *)&ctl->jbase + P.launch_idx;
  // device-side convergence control, as in k_rb_sweep_fused (uniform)
  bool skip = *(volatile int32_t *)&ctl->done != 0;
  // peer-memory slab exchange: launch epoch e waits until every CTA of every
  // slab finished epoch e - 1 (their boundary rows are in this slab's parity
  // e & 1 receive buffers and their norms in pnorm[(e - 1) & 3]); the norm
  // test below then reads the global max
  int64_t e = 0;
  const bool p2p = SLAB && P.p2p;
  if (p2p && !skip) {
    e = *(volatile int64_t *)&ctl->epoch + j;
    if (e > 0 && tid == 0) {
      const unsigned long long target = (unsigned long long)e * (unsigned long long)P.nranks;
      const long long t0 = clock64();
      while (*(volatile unsigned long long *)&ctl->sig < target && !*(volatile int32_t *)&ctl->p2p_timeout) {
        if (clock64() - t0 > (1ll << 33)) {  // watchdog (~4 s): report, do not hang
          ctl->p2p_timeout = 1;
          break;
        }
        __nanosleep(64);
      }
      __threadfence();
      // the ghost rows arrived through the generic proxy (peer stores); this
      // CTA reads them with TMA (async proxy)
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
    if (j > 0 && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0)  // the global norm, for k_step_end
      ctl->dmax[(j - 1) & (kRing - 1)] = *(volatile unsigned long long *)&ctl->pnorm[(e - 1) & 3];
  }
  if (!skip && j > 0) {
    const double prev = __longlong_as_double((long long)(
        p2p ? *(volatile unsigned long long *)&ctl->pnorm[(e - 1) & 3]
            : *(volatile unsigned long long *)&ctl->dmax[(j - 1) & (kRing - 1)]));
    if (prev < P.tol) {
      if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
        ctl->done = 1;
        ctl->launches_done = j;
      }
      skip = true;
    }
  }
  if (skip) {
    // drain the constant copies already in flight into this CTA's shared memory
    if (P.pre && tid == 0)
      for (int r = r_first; r < r_first + n_init; ++r) {
        mbar_arrive(c_bar(r));
        mbar_wait(c_bar(r), 0u);
      }
    return;
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
    ctl->dmax[(j + 1) & (kRing - 1)] = 0ull;
    // pnorm[(e + 1) & 3] receives epoch e + 1's remote maxima, which start
    // only after every slab finished this epoch, i.e. after this store
    if (p2p) ctl->pnorm[(e + 1) & 3] = 0ull;
  }
  const int par = (*(volatile int32_t *)&ctl->base + j) & 1;

  // ---------------------------------------------------------------- TMA issue
  const CUtensorMap *mVin = par ? &P.mV1 : &P.mV0;
  auto v_src = [&](int r, int &rr) -> const CUtensorMap * {
    if constexpr (SLAB) {
      const bool b = p2p && (e & 1);  // peer exchange: parity-e receive buffers
      if (P.has_rlo && r < P.y_begin) {
        rr = r - (P.y_begin - P.G);
        return b ? &P.mRlo_b : &P.mRlo;
      }
      if (P.has_rhi && r >= P.y_end) {
        rr = r - P.y_end;
        return b ? &P.mRhi_b : &P.mRhi;
      }
    }
    rr = r;
    return mVin;
  };
  // group r: constant row r + V row r + 1 (+ V row r for the first group).
  // The five constant maps are consecutive in FusedParams (mgx, mgy, mgz, mb,
  // mid) and their stage offsets are a * LAY (+ RW from gz_eff on), so every
  // copy is the same instruction sequence (small code: it is replicated in
  // each of the 12 unrolled steps).
  auto v_copy = [&](int rv_row, int r) {  // V row rv_row into its slot, completing group r
    int rv;
    const CUtensorMap *m = v_src(rv_row, rv);
    tma(vring + ((rv_row - r_first) % SV) * VST, m, c_bar(r), ps, rv, pol(5));
  };
  if (tid == 0) {
    for (int r = r_first; r < r_first + n_init; ++r) {
      const bool v1 = r + 1 <= r_last, v0 = r == r_first;
      const uint32_t vbytes = (v1 ? Gm::VBYTES : 0u) + (v0 ? Gm::VBYTES : 0u);
      mbar_expect_tx(c_bar(r), vbytes + (P.pre ? 0u : Gm::CBYTES));
      if (!P.pre)
        for (int a = 0; a < 5; ++a) tma(c_dst(r, a), mC + a, c_bar(r), ps, r, pol(a));
      if (v1) v_copy(r + 1, r);
      if (v0) v_copy(r, r);
    }
  }
  const int warp = tid >> 5;
  // refill after the barrier of step y: group R = y + 4 (slots of constant row
  // y - 2 and V row y - 7).  Lane 0 of warp w issues op w (w + NWARP, ...):
  // ops 0..4 constant array a = op (op 0 also posts expect_tx), 5: V row
  // R + 1.  The operands are computed, so each unrolled step holds a single
  // copy instruction sequence (the loop body is larger than the instruction
  // cache: measured +4 % for halving the refill code).
  // cs / vs: ring slots of constant row R and V row R + 1 (compile-time in the
  // unrolled steps: (u + 5) mod SC and (u + 6) mod SV)
  // Per-warp copy plan (8 warps or more, no ghost-row sources): warp w < 6
  // always issues op w, so its map, smem base / stride, row offset and policy
  // are fixed for the launch and the per-step refill is a handful of
  // instructions on one lane.
  constexpr bool kPlan = Gm::NWARP >= 6;
  const int my_op = warp;
  const bool my_v = my_op == 5;
  const CUtensorMap *my_map = my_op < 5 ? mC + my_op : mVin;
  double *my_base = my_op < 5 ? cring + my_op * Gm::LAY + (my_op >= 2 ? RW : 0) : vring;
  const int my_stride = my_v ? VST : CST;
  const uint64_t my_pol = pol(my_op < 6 ? my_op : 0);
  const bool my_lane = (tid & 31) == 0 && my_op < 6;
  auto refill = [&](const int y, const int cs, const int vs) {
    const int R = y + 4;
    if constexpr (kPlan) {
      if (my_lane && R >= r_first + SC && R + (my_v ? 1 : 0) <= r_last) {
        uint64_t *bar = &gbar[cs];
        if (my_op == 0) mbar_expect_tx(bar, Gm::CBYTES + (R + 1 <= r_last ? Gm::VBYTES : 0u));
        int yy = R + (my_v ? 1 : 0);
        const CUtensorMap *m = my_map;
        if constexpr (SLAB) {
          if (my_v) m = v_src(R + 1, yy);  // a slab's ghost rows come from the receive buffers
        }
        tma(my_base + (my_v ? vs : cs) * my_stride, m, bar, ps, yy, my_pol);
      }
    } else if ((tid & 31) == 0 && R >= r_first + SC && R <= r_last) {
      uint64_t *bar = &gbar[cs];
#pragma unroll 1
      for (int op = warp; op < 6; op += Gm::NWARP) {
        if (op == 0) mbar_expect_tx(bar, Gm::CBYTES + (R + 1 <= r_last ? Gm::VBYTES : 0u));
        if (op == 5 && R + 1 > r_last) break;
        int yy = R;
        const CUtensorMap *m = op < 5 ? mC + op : v_src(R + 1, yy);
        double *dst = op < 5 ? cring + cs * CST + op * Gm::LAY + (op >= 2 ? RW : 0) : vring + vs * VST;
        tma(dst, m, bar, ps, yy, pol(op));
      }
    }
  };

  // -------------------------------------------------------------- compute warps
  const int l = tid / W, lane = tid % W;
  const int pe = l * RW + lane, po = pe + W;
  // red node of row r sits in the odd column of the pair iff q ^ ((r - r_first - 1) & 1)
  const int q = (l + P.ypar + r_first + 1) & 1;
  // per parity class k (column parity q ^ k): node, x neighbour in the next /
  // previous lane, gx index of the link to that neighbour
  const int ME0 = q ? po : pe, ME1 = q ? pe : po;
  const int OT0 = q ? pe + 1 : po - 1, OT1 = q ? po - 1 : pe + 1;
  const int GX0 = q ? po : po - 1, GX1 = q ? po - 1 : po;
  const int gp = ps + lane;
  const bool exact_lane = lane >= FH && lane < FH + I && gp < P.HP;
  double *Vout = par ? P.V0 : P.V1;
  double *vout_e = Vout + (int64_t)l * P.layer_stride + gp;
  double *vout_o = vout_e + P.HP;
  double *OUT0 = q ? vout_o : vout_e, *OUT1 = q ? vout_e : vout_o;  // red's column for class 0 / 1
  const double w = P.omega;
  const uint64_t pol_out = (P.l2keep & 32) ? pol_last : policy_evict_normal();
  double dmax = 0.0;
  bool wrote_peer = false;  // this thread stored boundary rows into a neighbour's buffer
  // only the first / last chunk of a slab writes rows for a neighbour
  const bool send_cta = SLAB && ((ys < P.y_begin + P.G && (P.send_lo || (p2p && P.peer_lo[0]))) ||
                                 (ye > P.y_end - P.G && (P.send_hi || (p2p && P.peer_hi[0]))));

  // register FIFOs (entry = step index mod 3): values this thread produced,
  // old black values it loaded, constants level 0 loaded for level 1
  double fR0[3], fB0[3], fR1[3], fWn[3];
  NodeC cR[3], cB[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    fR0[k] = fB0[k] = fR1[k] = fWn[k] = 0.0;
    cR[k] = NodeC{0, 0, 0, 0, 0, 0, 0, 0};
    cB[k] = NodeC{0, 0, 0, 0, 0, 0, 0, 0};
  }

  // Streaming step y (u: position modulo 12) = phase A(y) | barrier | phase
  // B(y).  Phase B(y) and phase A(y + 1) touch no value of another warp that
  // the other writes (header), so the loop body is barrier(y), refill, wait for
  // row group y + 1, then B(y) and A(y + 1) in one branch-free block: the
  // compiler interleaves their four independent update chains.  Every step
  // runs the same unguarded code, also the first and last ones: the updates
  // of rows outside (r_first, r_last) and of the stale halo rows only read
  // ring slots that are loaded or hold finite leftovers (never an exact row's
  // operand: an exact row's level-1 value depends on old values of rows
  // r - 4 .. r + 4 only, all in [r_first, r_last], and on intermediate values
  // inside that cone), and their stores go to slots whose next TMA refill is
  // ordered after them by the per-step proxy fence.  Only the norm and the
  // write-out are masked.  A(r_last + 1) runs without its (never issued) row
  // group and its results are discarded.
  double aR0 = 0.0, aR1 = 0.0, aVN = 0.0, aGyN = 0.0, aD = 0.0;  // phase A results phase B needs
  double woR = 0.0, woB = 0.0;                                    // row written out after the body
  auto phaseA = [&](auto U_, const int y) {
    constexpr int u = decltype(U_)::value % 12;
    constexpr int k = u & 1;
    constexpr int f0 = u % 3, f1 = (u + 2) % 3, f2 = (u + 1) % 3;  // FIFO: now / 1 / 2 (3 = f0) steps ago
    // ring slots: V row y + d -> (u + 1 + d) mod SV, constant row y + d -> (u + 1 + d) mod SC
    constexpr int vY = ((u + 1) % SV) * VST, vY1 = ((u + 2) % SV) * VST;
    constexpr int vY3 = ((u + SV - 2) % SV) * VST;
    constexpr int cY = ((u + 1) % SC) * CST, cYm = (u % SC) * CST;
    const int me = k ? ME1 : ME0, mo = k ? ME0 : ME1;
    const int ot = k ? OT1 : OT0, ot3 = k ? OT0 : OT1;
    const int gxo = k ? GX1 : GX0;
    (void)f2;
    // red_0(y): column class k; its north operand (old black of row y - 1) was
    // loaded as the previous step's own-pair operand
    const double Vc = vring[vY + me];
    const double Vown = vring[vY + mo];
    const double Voth = vring[vY + ot];
    const double VN = fWn[f1];
    NodeC c0;
#ifdef PG_DIAG_NOLDSC
    // diagnostic build only (power experiments): the staged constants are
    // loaded by TMA as usual but not read (fixed register values, no LDS)
    c0 = NodeC{0.5, 0.5, 0.5, 0.5, 0.5, 0.5, 0.0, 0.3};
    (void)cYm;
#else
    c0.gxOwn = cring[cY + CGX + pe];
    c0.gxOth = cring[cY + CGX + gxo];
    c0.gyN = cring[cYm + CGY + me];
    c0.gyS = cring[cY + CGY + me];
    c0.gzU = cring[cY + CGZ + me];
    c0.gzD = cring[cY + CGZ + me - RW];
    c0.b = cring[cY + CB + me];
    c0.id = cring[cY + CID + me];
#endif
    const double r0 = upd_c(c0, w, Vc, Vown, Voth, VN, vring[vY1 + me], vring[vY + me + RW], vring[vY + me - RW]);
    // red_1(y - 3): column class k ^ 1 (= mo); own value red_0(y - 3), x
    // neighbour black_0(y - 3), north / south black_0(y - 4) / black_0(y - 2)
    const double Vc1 = fR0[f0];
    const double r1 = upd_c(cR[f0], w, Vc1, fB0[(u + 1) % 3], vring[vY3 + ot3], fB0[f0], fB0[f1],
                            vring[vY3 + mo + RW], vring[vY3 + mo - RW]);
    vring[vY + me] = r0;
    vring[vY3 + mo] = r1;
    aD = fabs(r1 - Vc1);  // red_1(y - 3): counted with black_1 of the same row next step
    fR0[f0] = r0;
    fR1[f0] = r1;
    fWn[f0] = Vown;
    cR[f0] = c0;
    aR0 = r0;
    aR1 = r1;
    aVN = VN;
    aGyN = c0.gyN;
  };
  auto phaseB = [&](auto U_, const int y) {
    constexpr int u = decltype(U_)::value % 12;
    constexpr int k = u & 1;
    constexpr int f0 = u % 3, f1 = (u + 2) % 3, f2 = (u + 1) % 3;
    constexpr int vYm = (u % SV) * VST, vY4 = ((u + SV - 3) % SV) * VST;
    constexpr int cYm = (u % SC) * CST;
    const int me = k ? ME1 : ME0, mo = k ? ME0 : ME1;
    const int ot = k ? OT1 : OT0, ot3 = k ? OT0 : OT1;
    const int gxo = k ? GX1 : GX0;
    (void)mo;
    // black_0(y - 1): column class k (its old value is red_0(y)'s north operand)
    NodeC cb;
#ifdef PG_DIAG_NOLDSC
    cb = NodeC{0.5, 0.5, cR[f2].gyS, aGyN, 0.5, 0.5, 0.0, 0.3};
#else
    cb.gxOwn = cring[cYm + CGX + pe];
    cb.gxOth = cring[cYm + CGX + gxo];
    cb.gyN = cR[f2].gyS;  // gy of row y - 2 in this column: red_0(y - 2)'s own south link
    cb.gyS = aGyN;
    cb.gzU = cring[cYm + CGZ + me];
    cb.gzD = cring[cYm + CGZ + me - RW];
    cb.b = cring[cYm + CB + me];
    cb.id = cring[cYm + CID + me];
#endif
    const double b0 = upd_c(cb, w, aVN, fR0[f1], vring[vYm + ot], fR0[f2], aR0, vring[vYm + me + RW],
                            vring[vYm + me - RW]);
    // black_1(y - 4): column class k ^ 1; own value black_0(y - 4), x neighbour
    // red_1(y - 4), north / south red_1(y - 5) / red_1(y - 3)
    const double Vcb1 = fB0[f0];
    const double Vownb1 = fR1[f1];
    const double b1 = upd_c(cB[f0], w, Vcb1, Vownb1, vring[vY4 + ot3], fR1[f2], aR1, vring[vY4 + mo + RW],
                            vring[vY4 + mo - RW]);
    vring[vYm + me] = b0;
    const bool out = y >= ys + 4;  // row y - 4 owned (y - 4 < ye always)
    // row y - 4: black_1 now, red_1 from the previous step's phase A; the
    // norm covers the owned rows [ys, ye) only
    double dB = fabs(b1 - Vcb1);
    dB = aD > dB ? aD : dB;
    if (!out) dB = 0.0;
    dmax = dB > dmax ? dB : dmax;
    woR = Vownb1;  // row y - 4 is final: written after the body's proxy fence
    woB = b1;
    fB0[f0] = b0;
    cB[f0] = cb;
  };
  // loop body of step y: barrier, refill, wait for row group y + 1, B(y) + A(y + 1)
  // row y - 4 is final: red_1 (class k) and black_1 (class k ^ 1).  Issued
  // after the body's proxy fence, so the fence does not wait for these stores.
  auto writeout = [&](auto U_, const int y) {
    constexpr int u = decltype(U_)::value % 12;
    constexpr int k = u & 1;
    const double Vownb1 = woR, b1 = woB;
    const bool out = y >= ys + 4;
    if (out && exact_lane) {
      const int64_t ro = (int64_t)(y - 4) * P.NXP;
      // evict_last when the next launch should find this V buffer in L2
      stg_hint((k ? OUT1 : OUT0) + ro, Vownb1, pol_out);
      stg_hint((k ? OUT0 : OUT1) + ro, b1, pol_out);
      if (SLAB && send_cta) {
        const int rr = y - 4;
        const bool red_odd = (q ^ k) != 0;
        const double ve = red_odd ? b1 : Vownb1, vo = red_odd ? Vownb1 : b1;
        double *slo = p2p ? P.peer_lo[(e + 1) & 1] : P.send_lo;
        double *shi = p2p ? P.peer_hi[(e + 1) & 1] : P.send_hi;
        if (slo && rr < P.y_begin + P.G) {
          double *sb = slo + ((int64_t)l * P.G + (rr - P.y_begin)) * P.NXP;
          sb[gp] = ve;
          sb[gp + P.HP] = vo;
          wrote_peer = true;
        }
        if (shi && rr >= P.y_end - P.G) {
          double *sb = shi + ((int64_t)l * P.G + (rr - (P.y_end - P.G))) * P.NXP;
          sb[gp] = ve;
          sb[gp + P.HP] = vo;
          wrote_peer = true;
        }
      }
    }
  };
  auto body = [&](auto U_, const int y) {
    constexpr int u = decltype(U_)::value;
    __syncthreads();
    refill(y, (u + 5) % SC, (u + 6) % SV);
    if (y + 1 <= r_last) mbar_wait(&gbar[(u + 2) % SC], (uint32_t)(((u + 2) / SC) & 1));
    phaseB(U_, y);
    phaseA(std::integral_constant<int, u + 1>{}, y + 1);
    // generic accesses to a V slot end 3 (reads) / 5 (writes) bodies before the
    // barrier after which TMA refills it: a proxy fence every second body
    // orders them (the fence also waits for this thread's global write-out)
    if constexpr (u % 2 == 1) fence_proxy_async();
    writeout(U_, y);
  };

  // the first step's north operand: old black of row r_first in the column of
  // red(r_first + 1), then phase A of the first step
  mbar_wait(&gbar[0], 0u);
  fWn[2] = vring[ME0];
  mbar_wait(&gbar[1], 0u);
  phaseA(std::integral_constant<int, 0>{}, r_first + 1);
  fence_proxy_async();
  // y = r_first + 1 .. r_last (r_last - r_first = H + 7 >= 8), blocks of 12
  // steps (the exits jump straight out of the unrolled block: only dmax is
  // live after the loop, so the register FIFOs need no fixed registers there)
  int y = r_first + 1;
#define PG_STEP2(U)                                  \
  body(std::integral_constant<int, U>{}, y);         \
  if (++y > r_last) goto done;
  while (true) {
    PG_STEP2(0) PG_STEP2(1) PG_STEP2(2) PG_STEP2(3) PG_STEP2(4) PG_STEP2(5)
    PG_STEP2(6) PG_STEP2(7) PG_STEP2(8) PG_STEP2(9) PG_STEP2(10) PG_STEP2(11)
  }
#undef PG_STEP2
done:
  if (!exact_lane) dmax = 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  // one atomic per CTA (warp maxima combined in shared memory first)
  __shared__ unsigned long long cta_max;
  if (tid == 0) cta_max = 0ull;
  __syncthreads();
  if ((tid & 31) == 0) atomicMax(&cta_max, static_cast<unsigned long long>(__double_as_longlong(dmax)));
  // Peer exchange: boundary rows (plain stores into peer memory) are made
  // visible system wide by the threads that stored them before the CTA counts
  // itself done
  if (SLAB && p2p && wrote_peer) __threadfence_system();
  __syncthreads();
  if (tid == 0) atomicMax(&ctl->dmax[j & (kRing - 1)], cta_max);
  if constexpr (SLAB) {
    if (p2p) {
      // every CTA adds its norm to this slab's slot and counts itself done;
      // the last CTA of the launch then max-reduces the slab's norm into every
      // other slab's slot and bumps every slab's arrival counter (2 N remote
      // atomics per launch)
      if (tid == 0) {
        atomicMax(&ctl->pnorm[e & 3], cta_max);
        __threadfence();
        const unsigned int done = atomicAdd(&ctl->ccount[e & 3], 1u) + 1u;  // (after this CTA's norm)
        if (done == gridDim.x * gridDim.y) {  // last CTA of this slab's launch e
          // slot e + 2 is next counted by launch e + 2, which starts after every
          // slab finished e + 1; its previous user, launch e - 2, is complete
          ctl->ccount[(e + 2) & 3] = 0u;
          __threadfence_system();
          const unsigned long long m = *(volatile unsigned long long *)&ctl->pnorm[e & 3];
          for (int r = 0; r < P.nranks; ++r)
            if (P.pnorm_all[r] != ctl->pnorm) atomicMax_system(P.pnorm_all[r] + (e & 3), m);
          __threadfence_system();
          for (int r = 0; r < P.nranks; ++r) atomicAdd_system(P.sig_all[r], 1ull);
        }
      }
    }
  }
}

// Compiled (L, W): W = 64 for L <= 4, W = 32 for L = 5..8 (the fused sweep's default widths)
#define PG_SWEEP2_CASES(X) \
  X(1, 64) X(2, 64) X(3, 64) X(4, 64) X(5, 32) X(6, 32) X(7, 32) X(8, 32)

}  // namespace pgb
