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
};

constexpr int kRing = 4;

// Red-black streaming sweep geometry: a warp covers 32 x-pairs (64 nodes) of one
// layer row; lanes 0 and 31 are halo (recomputed, never stored).
constexpr int kLanes = 32;
constexpr int kInterior = 30;
constexpr int kMaxLayers = 8;   // blockDim.y = layers <= 8 (multi-warp CTA)

struct MeshDims {
  int32_t L, NY, NX, NXP;   // NXP: row pitch (even, multiple of 16)
  int64_t layer_stride;     // NY * NXP
  int64_t np;               // L * NY * NXP
};

struct SweepArgs {
  MeshDims d;
  const double *gx, *gy, *gz, *b, *invd;
  double *V0, *V1;          // ping-pong pair; launch j of a step reads V[(base + j) & 1]
  double omega;
  int32_t rows_per_cta;
  int32_t nsweeps;          // sweeps fused in this launch (1 for the basic kernel)
  int32_t launch_idx;       // index of this launch within the time step
  double tol;
  DevCtl *ctl;
};

}  // namespace pgb

struct pg_grid {
  int kind = 0;              // 0 mesh, 1 csr
  int64_t n = 0;             // user nodes
  int64_t np = 0;            // storage elements
  double vdd = 1.0;
  bool rlc = false;
  cudaStream_t stream = nullptr;
  int dev = 0;
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
  int64_t *rowptr = nullptr;
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

  // ---- control
  pgb::DevCtl *ctl = nullptr;
  pgb::DevCtl *ctl_host = nullptr;     // pinned mirror
  int32_t *done_host = nullptr;        // pinned ring of polled `done` flags
  int64_t *dev_sweeps = nullptr;       // per-step sweep counts (device)
  int64_t dev_sweeps_cap = 0;

  // ---- options
  int fuse = 1;
  int batch = 8;
  int graph = 0;
  int timing = 0;                      // per-launch events for the sweep kernel
  int kernel = 3;                      // mesh sweep: 0 register streaming, 1 TMA ring, 2 cp.async ring, 3 optimised TMA
  int rows = 0;                        // rows per CTA (0: auto)
  int stages = 0;                      // TMA ring stages (0: auto)
  size_t tma_smem_set = 0;             // dynamic smem attribute currently set
  const void *tma_kernel_set = nullptr;  // ... and for which kernel
  int tma_state = 0;                   // 0 unknown, 1 usable, -1 unavailable
  CUtensorMap tmap[7];                 // V0, V1, gx, gy, gze, b, invd (encoded once)
  std::vector<cudaEvent_t> tev;        // timing event pool
};

namespace pgb {
void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

// kernels / launchers (pg_kernels.cu)
cudaError_t launch_setup(pg_grid *g, double h);
cudaError_t launch_rhs(pg_grid *g, double h, int64_t s);
cudaError_t launch_sweep(pg_grid *g, int method, double omega, double tol, int launch_idx,
                         int nsweeps, int64_t *launches);
cudaError_t launch_step_end(pg_grid *g, int64_t s, int launched, int flips, int fused,
                            int64_t max_sweeps, double tol);
cudaError_t launch_inductor_update(pg_grid *g, double h);
cudaError_t launch_probe(pg_grid *g, const int64_t *probe_idx, int64_t n_probe, double *out);
cudaError_t launch_reset_state(pg_grid *g);
cudaError_t launch_gather_user(pg_grid *g, double *dst_user_order);
cudaError_t launch_scatter_user(pg_grid *g, const double *src_user_order, double *dst_storage);
int sweeps_per_launch(pg_grid *g, int method);
bool tma_available(pg_grid *g);
cudaError_t launch_rb_sweep_tma(pg_grid *g, double omega, double tol, int launch_idx, int rows_per_cta);
int tma_stages_for(const pg_grid *g);
cudaError_t launch_rb_sweep_v3(pg_grid *g, double omega, double tol, int launch_idx, int rows_per_cta);
int v3_ctas_per_sm(const pg_grid *g);
int rows_per_cta_for(const pg_grid *g, int ctas_per_sm);

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
}  // namespace pgb
