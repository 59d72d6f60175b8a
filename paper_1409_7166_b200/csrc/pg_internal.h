// Internal declarations of the B200 power-grid transient library (not ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/pgrid.h"

namespace pgb {

// ---------------------------------------------------------------- device control
// One per grid, in device memory.  dmax[] is a ring of per-launch max|dV|
// (bit pattern of a non-negative double, so unsigned compare == double compare).
struct DevCtl {
  unsigned long long dmax[4];
  int32_t done;            // convergence detected in this step
  int32_t base;            // ping-pong parity: V[base] holds the current iterate
  int64_t launches_done;   // sweep launches that ran before `done` was detected
  int32_t diag_bad;        // a real node has d_i <= 0 (Lemma 1 precondition violated)
  int32_t failed;          // first step that hit max_sweeps (0: none)
  int64_t sweeps_total;
  int64_t sweeps_max;
  double last_delta;
  int32_t jbase;           // launch index of the first launch of the current batch:
                           // a sweep kernel's launch index is jbase + its argument,
                           // so one captured batch (CUDA graph) serves every batch
  // peer-memory slab exchange (pg_group kinds "p2p"): sweep launches that did
  // work since the group was formed (epoch of the next launch = epoch + its
  // index in the step), the count of this slab's finished CTAs, the arrival
  // counter every slab bumps (remotely) when its launch is complete, and the
  // norm ring indexed by epoch that every slab max-reduces into (remotely) --
  // none is reset per step or per transient, so early remote contributions are
  // never lost
  int64_t epoch;
  unsigned int ccount[4];  // CTAs of this slab that finished launch e, slot e & 3 (the last one publishes)
  unsigned long long sig;
  unsigned long long pnorm[4];
  int32_t p2p_timeout;     // a peer wait gave up (watchdog), results invalid
  int32_t nonfinite;       // an iterate held NaN / Inf (checked by the RHS kernel and at the end of a call)
  int64_t ipc_token;       // pg_group_p2p_selftest: this rank's mark, read by the peers through their mappings
};

constexpr int kRing = 4;
constexpr int kRhsTile = 2048;  // storage elements per tile of the fused RHS kernel
// staged CSR sweep: rows per tile and entry capacity per tile (6 per row)
#ifndef PG_CSR_R
#define PG_CSR_R 256
#endif
constexpr int kCsrR = PG_CSR_R;
constexpr int kCsrE = 6 * kCsrR;
constexpr int kMaxLayers = 8;   // CTA of the mesh sweep = 32 lanes x L warps
// taller meshes (up to kMaxMeshLayers) use the per-colour sweep k_rb_colour_mesh
constexpr int kMaxMeshLayers = 256;

// Mesh storage layout ("parity-split rows"), DESIGN.md §7.  Layer-major
// [L][NY][NXP] with row pitch NXP (a multiple of 64); inside a row the even
// columns come first and the odd columns second:
//     node (l, y, x)  ->  l * layer_stride + y * NXP + (x & 1) * HP + (x >> 1),
// HP = NXP / 2.  In the red-black numbering all nodes of one colour in one
// row and layer have the same column parity, so a warp updating a colour
// reads and writes 32 consecutive doubles (bank-conflict-free shared memory,
// coalesced global stores).  Padding elements (x >= NX) hold zero
// conductances, 1/d = 0 and are never updated.
struct MeshDims {
  int32_t L, NY, NX, NXP;   // NXP: row pitch (multiple of 64)
  int32_t HP;               // NXP / 2: half-row pitch
  int64_t layer_stride;     // NY * NXP
  int64_t np;               // L * NY * NXP
};

__host__ __device__ inline int64_t mesh_index(const MeshDims &d, int64_t l, int64_t y, int64_t x) {
  return l * d.layer_stride + y * d.NXP + (x & 1) * d.HP + (x >> 1);
}
// column of storage element i (may be >= NX for padding)
__host__ __device__ inline int64_t mesh_col(const MeshDims &d, int64_t i) {
  const int64_t o = i % d.NXP;
  return o >= d.HP ? 2 * (o - d.HP) + 1 : 2 * o;
}

// Ghost-row exchange buffers of a slab grid (set by its pg_group): the sweep
// writes the G owned rows next to each boundary to send_*, and reads the ghost
// rows from recv_* ([L][G][NXP] parity-split rows; maps per strip width).
struct SlabHalo {
  int G = 0;
  bool has_lo = false, has_hi = false;
  double *send_lo = nullptr, *send_hi = nullptr, *recv_lo = nullptr, *recv_hi = nullptr;
  CUtensorMap mlo[2], mhi[2];  // [W = 32 / 64] maps of recv_lo / recv_hi
  // peer-memory exchange: receive buffers double-buffered by launch epoch
  // (recv_* = parity 0, recv_*_b = parity 1); the sweep of epoch e reads its
  // ghost rows from parity e & 1 and stores its boundary rows straight into the
  // neighbours' parity (e + 1) & 1 buffers (peer_lo: the lower neighbour's
  // recv_hi pair, peer_hi: the upper neighbour's recv_lo pair)
  bool p2p = false;
  double *recv_lo_b = nullptr, *recv_hi_b = nullptr;
  CUtensorMap mlo_b[2], mhi_b[2];
  double *peer_lo[2] = {nullptr, nullptr}, *peer_hi[2] = {nullptr, nullptr};
  unsigned long long *sig_all[8] = {}, *pnorm_all[8] = {};  // every slab's DevCtl::sig / pnorm
  int nranks = 1;
};
constexpr int kMaxPeers = 8;

}  // namespace pgb

struct pg_grid {
  int kind = 0;              // 0 mesh, 1 csr
  int64_t n = 0;             // user nodes
  int64_t np = 0;            // storage elements
  double vdd = 1.0;
  bool rlc = false;
  cudaStream_t stream = nullptr;
  int dev = -1;               // set by creation (common_init)
  int num_sms = 148;

  // ---- mesh store (padded natural layout, SoA)
  pgb::MeshDims md{};
  double *gx = nullptr, *gy = nullptr, *gz = nullptr;   // raw conductances
  double *lz = nullptr;                                  // via inductance (RLC)
  double *gze = nullptr;                                 // effective via conductance (per h)
  double *iz = nullptr;                                  // via companion currents (RLC)

  // ---- csr store (colour-permuted)
  int32_t ncolor = 1;
  std::vector<int64_t> color_ptr;                        // host, ncolor+1
  int32_t *rowptr = nullptr;   // int32: nnz < 2^31 (checked at creation)
  bool csr_staged_ok = false;   // every tile of every colour fits the staged CSR sweep's buffers
  int32_t *col = nullptr;
  double *val = nullptr;
  int64_t *perm = nullptr;    // storage -> user
  int64_t *iperm = nullptr;   // user -> storage

  // ---- per-node arrays (storage layout)
  double *V[2] = {nullptr, nullptr};
  double *x0 = nullptr;
  double *cap = nullptr, *invd = nullptr, *b = nullptr;

  // ---- pads grouped by storage index (sorted), groups of equal index
  int64_t npad = 0, npad_grp = 0;
  int64_t *pad_idx = nullptr, *pad_grp = nullptr;
  double *pad_g = nullptr, *pad_l = nullptr, *pad_ge = nullptr, *pad_i = nullptr;

  // ---- sources grouped the same way
  int64_t nsrc = 0, nsrc_grp = 0, npts = 0;
  int64_t *src_idx = nullptr, *src_grp = nullptr, *src_ptr = nullptr;
  double *pwl_t = nullptr, *pwl_i = nullptr;
  // first pad / source group of every RHS tile of kRhsTile storage elements
  // (ntile + 1 entries each; the fused RHS kernel's per-tile ranges)
  int64_t ntile = 0;
  int64_t *pad_tile = nullptr, *src_tile = nullptr;

  // ---- trajectory: time steps of length traj_h completed since x(0) (the
  // state pg_transient_continue resumes from); 0 after create / set_voltages / dc
  int64_t traj_steps = 0;
  double traj_h = 0.0;
  // step-size-dependent setup (companion conductances, 1/d) valid for setup_h:
  // a call with the same h (e.g. the next pg_transient_continue window) skips it
  bool setup_ok = false;
  double setup_h = 0.0;

  // ---- control
  pgb::DevCtl *ctl = nullptr;
  pgb::DevCtl *ctl_host = nullptr;     // pinned mirror
  int32_t *done_host = nullptr;        // pinned ring of polled `done` flags
  int64_t *dev_sweeps = nullptr;       // per-step sweep counts (device)
  int64_t dev_sweeps_cap = 0;
  double *user_buf = nullptr;          // n doubles: user-order staging of pg_get/set_voltages (mesh: the create staging buffer; CSR: lazy)

  // ---- slab of a partitioned mesh (pg_set_slab): rows [y_begin, y_end) are
  // owned, the others are ghost rows refreshed by the group exchange
  bool slab = false;
  int32_t y_begin = 0, y_end = 0, ypar = 0;
  pgb::SlabHalo hx;

  // ---- options
  int fuse = 0;                        // F: sweeps per launch of the temporally blocked mesh sweep (0: auto)
  int lag = 3;                         // wavefront lag D between fused levels (3 or 4)
  int batch = 8;
  int timing = 0;                      // per-launch events for the sweep kernel
  int rows = 0;                        // rows per CTA (0: auto)
  int stages = 0;                      // TMA ring stages (0: auto)
  int width = 0;                       // strip width W in column pairs: 32, 64 (0: auto)
  size_t tma_smem_set = 0;             // dynamic smem attribute currently set
  const void *tma_kernel_set = nullptr;  // ... and for which kernel
  int tma_state = 0;                   // 0 unknown, 1 usable, -1 unavailable
  CUtensorMap tmap[2][7];              // [W = 32 / 64] V0, V1, gx, gy, gze, b, invd (encoded once)
  std::vector<cudaEvent_t> tev;        // timing event pool
  int use_graph = 1;                   // option "graph": replay captured sweep batches
  int resident = 1;                    // option "resident": one-CTA sweep loop for tiny meshes
  int pipe = 1;                        // option "pipe": two-level pipeline kernel for full F = 2 launches
  int l2first = -1;                    // option "l2first": arrays read with evict_first (bit mask, -1: auto)
  int l2keep = -1;                     // option "l2keep": arrays kept in L2 across launches (bit mask, -1: auto)
  int l2promo = 128;                   // option "l2promo": TMA L2 promotion bytes (0, 64, 128, 256)
  int pdl = 0;                         // option "pdl": programmatic dependent launch of consecutive sweeps
                                       // (off by default: 1.5-3 % slower on configs 1 and 4)
  int csr_stage = 1;                   // option "csr_stage": bulk-copy staged CSR sweep (k_csr_sweep_staged)
  int colour = 0;                      // option "colour": per-colour mesh sweep (k_rb_colour_mesh) for every
                                       // layer count (default: only meshes taller than kMaxLayers)
  bool pdl_ok = false;                 // set by run_transient: single grid, no exchange between launches
  bool group_active = false;           // inside pg_group_transient (peer exchange armed)
  cudaGraphExec_t batch_exec = nullptr;  // captured batch of `batch` full sweep launches
  cudaStream_t cap_stream = nullptr;     // private stream the batch graph is captured on
  double graph_key[7] = {0, 0, 0, 0, 0, 0, 0};  // omega, tol, method, F, batch, stream, exchange of the capture
};

namespace pgb {
void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

// kernels / launchers (pg_kernels.cu)
cudaError_t launch_setup(pg_grid *g, double h);
cudaError_t launch_rhs(pg_grid *g, double h, double t);
cudaError_t launch_sweep(pg_grid *g, int method, double omega, double tol, int launch_idx,
                         int nsweeps, int64_t *launches);
cudaError_t launch_batch_advance(pg_grid *g, int nb);
bool resident_ok(const pg_grid *g, int method);
cudaError_t launch_rb_resident(pg_grid *g, double omega, double tol, int64_t max_sweeps, int64_t s);
cudaError_t launch_step_end(pg_grid *g, int64_t s, int launched, int flips, int fused,
                            int64_t max_sweeps, double tol);
cudaError_t launch_inductor_update(pg_grid *g, double h);
cudaError_t launch_probe(pg_grid *g, const int64_t *probe_idx, int64_t n_probe, double *out);
cudaError_t launch_reset_state(pg_grid *g, bool keep_base = false);
cudaError_t launch_check_finite(pg_grid *g);
int dnorm2_blocks(const pg_grid *g);
cudaError_t launch_dnorm2(pg_grid *g, double *part);  // part[2 * blocks]: sum d V0^2, sum d V1^2 per block
cudaError_t launch_gather_user(pg_grid *g, double *dst_user_order);
cudaError_t launch_scatter_user(pg_grid *g, const double *src_user_order, double *dst_storage);
int sweeps_per_launch(pg_grid *g, int method);
// mesh grids swept colour by colour (two launches per sweep): taller than
// kMaxLayers or option "colour"
bool colour_sweep(const pg_grid *g);
// temporally blocked red-black sweep (pg_sweep_fused.cu)
bool tma_available(pg_grid *g);
bool encode_halo_maps(pg_grid *g);
int fused_exact_lanes(int F, int W);
int fused_default_stages(int L, int F, int D);
bool fused_variant_exists(int L, int F, int S, int D, int W, bool slab = false);
int fused_ctas_per_sm(int L, int S, int W);
cudaError_t launch_rb_sweep_fused(pg_grid *g, double omega, double tol, int j, int nsw, int F,
                                  int S, int D, int W, int rows_per_cta, int y_begin, int y_end,
                                  int ypar);
// two-level pipeline for full F = 2 launches (pg_sweep2.cu)
int sweep2_width(int L);  // strip width of the compiled variant, 0: none
int sweep2_ctas_per_sm(int L, bool slab);
int sweep2_rows_per_cta(const pg_grid *g, int ny);
int64_t sweep2_grid_ctas(const pg_grid *g);
// pdl: launch with programmatic stream serialisation after a sweep launch
cudaError_t launch_rb_sweep2(pg_grid *g, double omega, double tol, int j, int rows_per_cta, int y_begin,
                             int y_end, int ypar, bool pdl);

// Multi-grid driver (pg_api.cu): Algorithm 1 over ng grids in lockstep; `ex`
// (may be null) runs after every sweep launch of all grids.
struct Exchange {
  virtual ~Exchange() = default;
  // before the first step (initial state in V[0]) and after each step's last
  // sweep launch (before step_end)
  virtual cudaError_t begin() { return cudaSuccess; }
  virtual cudaError_t end_step(int64_t *launches) { return cudaSuccess; }
  // launch_idx: index of the launch in the time step; rel: index in its batch
  virtual cudaError_t after_sweep(int launch_idx, int rel, int64_t *launches) = 0;
  // the exchange happens inside the sweep kernels (nothing between launches):
  // a single slab per process may then use graph batches and PDL
  virtual bool fused() const { return false; }
  // after_sweep may be captured into a CUDA graph (its buffers do not depend on
  // the launch index beyond j % kRing)
  virtual bool capturable() const { return false; }
};
int run_transient(pg_grid **gs, int ng, Exchange *ex, double h, int64_t steps, double tol,
                  double omega, int method, int64_t max_sweeps, int64_t n_probe,
                  const int64_t *probe_node, double *probe_out, int mem, int64_t *sweeps_out,
                  pg_stats *stats, double t_dc = 0.0, bool cont = false);
// first group of every RHS tile: tiles[t] = first q with node_of_group[q] >= t * kRhsTile
std::vector<int64_t> rhs_tile_starts(const std::vector<int64_t> &group_node, int64_t np);
// the library's device allocator (pg_api.cu: stream-ordered pool, 256-byte
// aligned blocks, cudaMalloc / cudaFree semantics)
int dalloc_bytes(void **p, size_t bytes);
void dfree_bytes(void *p);
// device-side store construction (pg_store.cu)
int build_sources_device(pg_grid *g, int64_t n_src, const int64_t *node, const int64_t *ptr, const double *t,
                         const double *v, int64_t npts, int32_t *bad_bits, std::string &err);
cudaError_t mesh_check_async(pg_grid *g, const double *user_array, int which, int32_t *d_err);
// *d_err |= 1 if any of a[0..n) is NaN or infinite (on g->stream)
cudaError_t finite_check_async(pg_grid *g, const double *a, int64_t n, int32_t *d_err);

// host CSR construction (pg_csr_build.cpp)
struct CsrHost {
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<double> val;
  std::vector<int64_t> perm, iperm;
  std::vector<int64_t> color_ptr;
};
int build_csr(int64_t n, int64_t m, const int64_t *bu, const int64_t *bv, const double *bg,
              CsrHost &out, std::string &err);
// the same store built on the device into g (pg_csr_device.cu; device input
// arrays); *done = false (and g untouched) when the graph is not bipartite --
// the caller then uses build_csr
int build_csr_device(pg_grid *g, int64_t n, int64_t m, const int64_t *bu, const int64_t *bv, const double *bg,
                     const double *cap, bool *done, std::string &err);
}  // namespace pgb
