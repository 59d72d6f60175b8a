// C ABI (include/pgrid.h): netlist store construction and the Algorithm 1
// time-step driver.  All numerics run in the kernels of pg_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "pg_internal.h"

namespace pgb {
static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }
int cuda_fail(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return PG_ECUDA;
}

__global__ void k_fill_real(double *x, int64_t np, MeshDims d, int32_t mesh, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (!mesh || mesh_col(d, i) < d.NX) ? v : 0.0;
}
}  // namespace pgb

using namespace pgb;

#define CK(call)                                          \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);   \
  } while (0)

#define REQUIRE(cond, msg)    \
  do {                        \
    if (!(cond)) {            \
      set_error(msg);         \
      return PG_EINVAL;       \
    }                         \
  } while (0)

namespace {

// PGB200_TRACE=1: phase times of the host-buffer calls (create, set_sources,
// get_voltages) on stderr, each phase closed by a device synchronisation
// (diagnostics of the end-to-end path; off by default, no synchronisation)
struct PhaseTrace {
  bool on;
  const char *call;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTrace(const char *c) : on(std::getenv("PGB200_TRACE") != nullptr), call(c) {
    if (on) {
      cudaDeviceSynchronize();
      t = std::chrono::steady_clock::now();
    }
  }
  void mark(const char *what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pgb200 trace] %s %s %.2f ms\n", call, what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Device memory of the grids comes from a library-owned stream-ordered pool
// per device (release threshold 48 GiB by default), so creating and destroying grids, the
// per-call scratch of pg_transient and pg_set_sources do not map and unmap
// device memory each time (cudaMalloc / cudaFree of large buffers took up to
// ~200 ms now and then inside the end-to-end call).  Blocks are handed out
// after the pool's stream reached the allocation and returned after a device
// synchronisation, so they are usable from any stream like cudaMalloc memory.
// DevCtl stays plain cudaMalloc memory: it is exported over CUDA IPC.
// Two pools per device: blocks of >= kLargeBlock bytes (the per-node arrays)
// and smaller ones (pads, load store, scratch).  A pool splits its cached free
// blocks to serve smaller requests, so with one pool a 256-byte flag or a
// 40 MB sort buffer carved out of a freed 1 GB array made the next grid's 1 GB
// arrays map fresh memory (10-140 ms per call on config 4, PGB200_TRACE).
constexpr size_t kLargeBlock = (size_t)32 << 20;
struct DevPool {
  bool init = false;
  cudaMemPool_t pool = nullptr;   // blocks >= kLargeBlock
  cudaMemPool_t small = nullptr;  // blocks < kLargeBlock
  cudaStream_t s = nullptr;
};
std::mutex g_pool_mu;
DevPool g_pools[64];
std::unordered_map<void *, int> g_pool_ptrs;  // pool block -> device

DevPool *pool_of(int dev) {
  if (dev < 0 || dev >= 64) return nullptr;
  DevPool &d = g_pools[dev];
  if (!d.init) {
    d.init = true;
    cudaMemPoolProps pr = {};
    pr.allocType = cudaMemAllocationTypePinned;
    pr.handleTypes = cudaMemHandleTypeNone;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = dev;
    // release threshold: freed blocks up to this size stay mapped for the next
    // grid (PGB200_POOL_GIB, default 48 GiB: a config-4-sized grid is ~11 GB,
    // and re-mapping it for every end-to-end create cost ~0.4 s); an allocation
    // the pool cannot serve trims it first (dalloc), so the cache never blocks
    // this library's own allocations
    uint64_t gib = 48;
    if (const char *e = std::getenv("PGB200_POOL_GIB")) gib = std::strtoull(e, nullptr, 10);
    uint64_t thr = gib << 30;
    uint64_t thr_small = (uint64_t)1 << 30;
    if (cudaMemPoolCreate(&d.pool, &pr) != cudaSuccess ||
        cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &thr) != cudaSuccess ||
        cudaMemPoolCreate(&d.small, &pr) != cudaSuccess ||
        cudaMemPoolSetAttribute(d.small, cudaMemPoolAttrReleaseThreshold, &thr_small) != cudaSuccess ||
        cudaStreamCreateWithFlags(&d.s, cudaStreamNonBlocking) != cudaSuccess) {
      cudaGetLastError();
      d.pool = nullptr;
    }
  }
  return d.pool ? &d : nullptr;
}

// synced: the caller already synchronized the device (free_grid does it once
// for all of a grid's blocks instead of once per block)
void dfree(void *p, bool synced = false) {
  if (!p) return;
  int dev = -1;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pool_ptrs.find(p);
    if (it != g_pool_ptrs.end()) {
      dev = it->second;
      g_pool_ptrs.erase(it);
    }
  }
  if (dev < 0) {
    cudaFree(p);
    return;
  }
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  if (!synced) cudaDeviceSynchronize();  // the block may still be in use on any stream (cudaFree semantics)
  DevPool *d;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    d = pool_of(dev);
  }
  if (d) cudaFreeAsync(p, d->s);
  if (cur != dev) cudaSetDevice(cur);
}

template <class T>
int dalloc(T **p, int64_t count, bool plain = false) {
  *p = nullptr;
  if (count <= 0) return PG_OK;
  const size_t bytes = sizeof(T) * (size_t)count;
  cudaError_t e = cudaErrorMemoryAllocation;
  int dev = 0;
  cudaGetDevice(&dev);
  DevPool *d = nullptr;
  if (!plain) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    d = pool_of(dev);
  }
  if (d) {
    // sizes rounded to 256 B so that every block keeps cudaMalloc's alignment
    // (TMA tensor maps and vector loads rely on it); checked below
    const size_t rb = (bytes + 255) & ~(size_t)255;
    cudaMemPool_t mp = rb >= kLargeBlock ? d->pool : d->small;
    e = cudaMallocFromPoolAsync((void **)p, rb, mp, d->s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->s);
    if (e != cudaSuccess) {
      // the pools' cached free blocks may be what is missing: release them to
      // the device and retry once before falling back to cudaMalloc
      cudaGetLastError();
      cudaStreamSynchronize(d->s);
      cudaMemPoolTrimTo(d->pool, 0);
      cudaMemPoolTrimTo(d->small, 0);
      e = cudaMallocFromPoolAsync((void **)p, rb, mp, d->s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(d->s);
    }
    if (e == cudaSuccess && ((uintptr_t)*p & 255)) {
      cudaFreeAsync(*p, d->s);
      cudaStreamSynchronize(d->s);
      *p = nullptr;
      d = nullptr;
    } else if (e == cudaSuccess) {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      g_pool_ptrs[(void *)*p] = dev;
    } else {
      cudaGetLastError();
      *p = nullptr;
      d = nullptr;  // pool exhausted or unusable: plain cudaMalloc
    }
  }
  if (!d) {
    e = cudaMalloc((void **)p, bytes);
  }
  if (e != cudaSuccess) {
    *p = nullptr;
    set_error(std::string("cudaMalloc of ") + std::to_string(sizeof(T) * (size_t)count) +
              " bytes failed: " + cudaGetErrorString(e));
    return PG_ENOMEM;
  }
  return PG_OK;
}

template <class T>
int to_host(const T *src, int64_t count, int mem, std::vector<T> &out) {
  out.resize((size_t)std::max<int64_t>(count, 0));
  if (count <= 0) return PG_OK;
  if (mem == PG_MEM_HOST) {
    std::memcpy(out.data(), src, sizeof(T) * (size_t)count);
    return PG_OK;
  }
  CK(cudaMemcpy(out.data(), src, sizeof(T) * (size_t)count, cudaMemcpyDeviceToHost));
  return PG_OK;
}

template <class T>
int upload(T *dst, const std::vector<T> &v) {
  if (v.empty()) return PG_OK;
  CK(cudaMemcpy(dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return PG_OK;
}

void free_grid(pg_grid *g) {
  if (!g) return;
  int cur = 0;
  cudaGetDevice(&cur);
  const bool other = g->dev >= 0 && cur != g->dev;
  if (other) cudaSetDevice(g->dev);
  cudaDeviceSynchronize();  // every block below may still be in use on some stream
  void *ptrs[] = {g->gx, g->gy, g->gz, g->lz, g->gze, g->iz, g->rowptr, g->col, g->val, g->perm,
                  g->iperm, g->V[0], g->V[1], g->x0, g->cap, g->invd, g->b, g->pad_idx,
                  g->pad_grp, g->pad_g, g->pad_l, g->pad_ge, g->pad_i, g->src_idx, g->src_grp,
                  g->src_ptr, g->pwl_t, g->pwl_i, g->pad_tile, g->src_tile, g->ctl, g->dev_sweeps,
                  g->user_buf};  // ctl: plain (dfree -> cudaFree)
  for (void *p : ptrs)
    if (p) dfree(p, true);
  for (cudaEvent_t e : g->tev) cudaEventDestroy(e);
  if (g->batch_exec) cudaGraphExecDestroy(g->batch_exec);
  if (g->cap_stream) cudaStreamDestroy(g->cap_stream);
  if (g->ctl_host) cudaFreeHost(g->ctl_host);
  if (g->done_host) cudaFreeHost(g->done_host);
  // the pools keep up to their release thresholds of freed memory cached for
  // the next grid (re-mapping ~10 GB for a config-4-sized grid costs ~1 s); an
  // allocation the pools cannot serve trims them before falling back to
  // cudaMalloc, and pg_release_memory hands the cache back explicitly
  if (other) cudaSetDevice(cur);
  delete g;
}

struct GridGuard {
  pg_grid *g;
  ~GridGuard() { free_grid(g); }
};

int64_t storage_index(const pg_grid *g, int64_t k, const std::vector<int64_t> *iperm_host) {
  if (g->kind == 0) {
    const int64_t per_layer = (int64_t)g->md.NY * g->md.NX;
    const int64_t l = k / per_layer, r = k % per_layer;
    const int64_t y = r / g->md.NX, x = r % g->md.NX;
    return mesh_index(g->md, l, y, x);
  }
  return (*iperm_host)[(size_t)k];
}

// group sorted storage indices: returns group start offsets (ngrp+1)
std::vector<int64_t> groups_of(const std::vector<int64_t> &sidx) {
  std::vector<int64_t> grp;
  for (size_t k = 0; k < sidx.size(); ++k)
    if (k == 0 || sidx[k] != sidx[k - 1]) grp.push_back((int64_t)k);
  grp.push_back((int64_t)sidx.size());
  return grp;
}

int common_init(pg_grid *g) {
  CK(cudaGetDevice(&g->dev));
  CK(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->dev));
  g->ntile = (g->np + kRhsTile - 1) / kRhsTile;
  int rc;
  // b and 1/d get 8 elements of slack: the staged CSR sweep bulk-copies
  // 16-byte-rounded row ranges that may end one element past np
  if ((rc = dalloc(&g->V[0], g->np)) || (rc = dalloc(&g->V[1], g->np)) || (rc = dalloc(&g->x0, g->np)) ||
      (rc = dalloc(&g->invd, g->np + 8)) || (rc = dalloc(&g->b, g->np + 8)) || (rc = dalloc(&g->ctl, 1, true)))
    return rc;
  CK(cudaMemset(g->V[0], 0, sizeof(double) * g->np));
  CK(cudaMemset(g->V[1], 0, sizeof(double) * g->np));
  CK(cudaMemset(g->b, 0, sizeof(double) * (g->np + 8)));
  CK(cudaMemset(g->invd, 0, sizeof(double) * (g->np + 8)));
  CK(cudaMemset(g->ctl, 0, sizeof(DevCtl)));
  CK(cudaMallocHost((void **)&g->ctl_host, sizeof(DevCtl)));
  CK(cudaMallocHost((void **)&g->done_host, sizeof(int32_t) * 8));
  const int B = 256;
  const int grid = (int)std::min<int64_t>((g->np + B - 1) / B, (int64_t)g->num_sms * 16);
  k_fill_real<<<std::max(grid, 1), B>>>(g->x0, g->np, g->md, g->kind == 0, g->vdd);
  CK(cudaGetLastError());
  CK(cudaMemcpy(g->V[0], g->x0, sizeof(double) * g->np, cudaMemcpyDeviceToDevice));
  CK(cudaDeviceSynchronize());
  return PG_OK;
}

int set_pads(pg_grid *g, int64_t n_pads, const int64_t *pad_node, const double *pad_g,
             const double *pad_l, int mem, const std::vector<int64_t> *iperm_host) {
  std::vector<int64_t> node;
  std::vector<double> pg, pl;
  int rc;
  if ((rc = to_host(pad_node, n_pads, mem, node)) || (rc = to_host(pad_g, n_pads, mem, pg))) return rc;
  if (pad_l && (rc = to_host(pad_l, n_pads, mem, pl))) return rc;
  std::vector<int64_t> sidx((size_t)n_pads);
  for (int64_t k = 0; k < n_pads; ++k) {
    REQUIRE(node[k] >= 0 && node[k] < g->n, "pad node index out of range");
    REQUIRE(pg[k] > 0.0 && std::isfinite(pg[k]), "pad conductance must be finite and > 0");
    if (pad_l) REQUIRE(pl[k] >= 0.0 && std::isfinite(pl[k]), "pad inductance must be finite and >= 0");
    sidx[k] = storage_index(g, node[k], iperm_host);
  }
  std::vector<int64_t> order((size_t)n_pads);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return sidx[a] < sidx[b]; });
  std::vector<int64_t> s2(n_pads);
  std::vector<double> g2(n_pads), l2(pad_l ? n_pads : 0);
  for (int64_t k = 0; k < n_pads; ++k) {
    s2[k] = sidx[order[k]];
    g2[k] = pg[order[k]];
    if (pad_l) l2[k] = pl[order[k]];
  }
  std::vector<int64_t> grp = groups_of(s2);
  g->npad = n_pads;
  g->npad_grp = (int64_t)grp.size() - 1;
  std::vector<int64_t> gnode((size_t)g->npad_grp);
  for (int64_t q = 0; q < g->npad_grp; ++q) gnode[q] = s2[grp[q]];
  const std::vector<int64_t> tiles = rhs_tile_starts(gnode, g->np);
  if ((rc = dalloc(&g->pad_idx, n_pads)) || (rc = dalloc(&g->pad_grp, (int64_t)grp.size())) ||
      (rc = dalloc(&g->pad_g, n_pads)) || (rc = dalloc(&g->pad_ge, n_pads)) ||
      (rc = dalloc(&g->pad_tile, (int64_t)tiles.size())))
    return rc;
  if ((rc = upload(g->pad_idx, s2)) || (rc = upload(g->pad_grp, grp)) || (rc = upload(g->pad_g, g2)) ||
      (rc = upload(g->pad_tile, tiles)))
    return rc;
  if (pad_l && n_pads > 0) {
    if ((rc = dalloc(&g->pad_l, n_pads)) || (rc = dalloc(&g->pad_i, n_pads))) return rc;
    if ((rc = upload(g->pad_l, l2))) return rc;
    CK(cudaMemset(g->pad_i, 0, sizeof(double) * n_pads));
    g->rlc = true;
  }
  return PG_OK;
}

}  // namespace

namespace pgb {
int dalloc_bytes(void **p, size_t bytes) {
  unsigned char *q = nullptr;
  const int rc = dalloc(&q, (int64_t)bytes);
  *p = q;
  return rc;
}
void dfree_bytes(void *p) { dfree(p); }
}  // namespace pgb

extern "C" {

PG_API const char *pg_last_error(void) { return g_err.c_str(); }

PG_API int pg_create_mesh(int32_t layers, int32_t ny, int32_t nx, const double *gx, const double *gy,
                          const double *gz, const double *lz, const double *cap, int64_t n_pads,
                          const int64_t *pad_node, const double *pad_g, const double *pad_l,
                          double vdd, int mem, pg_grid **out) {
  if (out) *out = nullptr;
  REQUIRE(out != nullptr, "out is NULL");
  REQUIRE(layers >= 1 && ny >= 1 && nx >= 1, "layers, ny, nx must be >= 1");
  REQUIRE(layers <= kMaxMeshLayers, "at most 256 layers per mesh grid");
  REQUIRE((int64_t)layers * ny < (int64_t)1 << 31, "layers * ny must be < 2^31");
  REQUIRE(mem == PG_MEM_HOST || mem == PG_MEM_DEVICE, "mem must be PG_MEM_HOST or PG_MEM_DEVICE");
  REQUIRE(gx && gy && gz && cap, "gx, gy, gz, cap are required");
  REQUIRE(n_pads >= 0 && (n_pads == 0 || (pad_node && pad_g)), "bad pad arrays");
  REQUIRE(std::isfinite(vdd), "vdd must be finite");
  const int64_t n = (int64_t)layers * ny * nx;
  pg_grid *g = new pg_grid();
  GridGuard guard{g};
  g->kind = 0;
  g->n = n;
  g->vdd = vdd;
  g->md.L = layers;
  g->md.NY = ny;
  g->md.NX = nx;
  g->md.NXP = (nx + 63) / 64 * 64;
  g->md.HP = g->md.NXP / 2;
  g->md.layer_stride = (int64_t)ny * g->md.NXP;
  g->md.np = (int64_t)layers * g->md.layer_stride;
  g->np = g->md.np;
  int rc;
  PhaseTrace tr("pg_create_mesh");
  if ((rc = common_init(g))) return rc;
  tr.mark("common_init");
  const cudaMemcpyKind kind = mem == PG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  double *stage = nullptr;  // user-order staging buffer, scattered into the storage layout
  int32_t *d_bad = nullptr;  // value-check flags of the inputs (checked on the device)
  // the staging buffer stays with the grid as its user-order buffer
  // (pg_get_voltages / pg_set_voltages), so reading the result back allocates nothing
  if ((rc = dalloc(&stage, n))) return rc;
  g->user_buf = stage;
  if ((rc = dalloc(&d_bad, 1))) return rc;
  struct FlagGuard {
    int32_t *q;
    ~FlagGuard() { dfree(q); }
  } flag_guard{d_bad};
  CK(cudaMemset(d_bad, 0, sizeof(int32_t)));
  // which: 0 gx, 1 gy, 2 gz (>= 0, finite, zero on the open boundary), 3 cap, 4 lz (>= 0, finite)
  auto put = [&](double **dst, const double *src, int which) -> int {
    int r = dalloc(dst, g->np);
    if (r) return r;
    CK(cudaMemset(*dst, 0, sizeof(double) * g->np));
    tr.mark("alloc+memset");
    CK(cudaMemcpy(stage, src, sizeof(double) * n, kind));
    tr.mark("copy");
    CK(mesh_check_async(g, stage, which, d_bad));
    CK(launch_scatter_user(g, stage, *dst));
    tr.mark("check+scatter");
    return PG_OK;
  };
  if ((rc = put(&g->gx, gx, 0)) || (rc = put(&g->gy, gy, 1)) || (rc = put(&g->gz, gz, 2)) ||
      (rc = put(&g->cap, cap, 3)))
    return rc;
  if ((rc = dalloc(&g->gze, g->np))) return rc;
  CK(cudaMemcpy(g->gze, g->gz, sizeof(double) * g->np, cudaMemcpyDeviceToDevice));
  if (lz) {
    if ((rc = put(&g->lz, lz, 4)) || (rc = dalloc(&g->iz, g->np))) return rc;
    CK(cudaMemset(g->iz, 0, sizeof(double) * g->np));
    g->rlc = true;
  }
  int32_t bad = 0;
  CK(cudaMemcpy(&bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost));
  REQUIRE(!(bad & (1 << 0)), "gx must be finite, >= 0 and 0 in the last column");
  REQUIRE(!(bad & (1 << 1)), "gy must be finite, >= 0 and 0 in the last row");
  REQUIRE(!(bad & (1 << 2)), "gz must be finite, >= 0 and 0 in the top layer");
  REQUIRE(!(bad & (1 << 3)), "cap must be finite and >= 0");
  REQUIRE(!(bad & (1 << 4)), "lz must be finite and >= 0");
  tr.mark("gze+lz+flags");
  if ((rc = set_pads(g, n_pads, pad_node, pad_g, pad_l, mem, nullptr))) return rc;
  CK(cudaDeviceSynchronize());
  tr.mark("set_pads");
  guard.g = nullptr;
  *out = g;
  return PG_OK;
}

PG_API int pg_create_csr(int64_t n, int64_t m, const int64_t *bu, const int64_t *bv, const double *bg,
                         const double *cap, int64_t n_pads, const int64_t *pad_node,
                         const double *pad_g, double vdd, int mem, pg_grid **out) {
  if (out) *out = nullptr;
  REQUIRE(out != nullptr, "out is NULL");
  REQUIRE(n >= 1, "n must be >= 1");
  REQUIRE(n < (int64_t)INT32_MAX, "CSR grids are limited to 2^31-1 nodes");
  REQUIRE(m >= 0 && (m == 0 || (bu && bv && bg)), "bad branch arrays");
  REQUIRE(cap != nullptr, "cap is required");
  REQUIRE(mem == PG_MEM_HOST || mem == PG_MEM_DEVICE, "mem must be PG_MEM_HOST or PG_MEM_DEVICE");
  REQUIRE(n_pads >= 0 && (n_pads == 0 || (pad_node && pad_g)), "bad pad arrays");
  int rc;
  PhaseTrace tr("pg_create_csr");
  pg_grid *g = new pg_grid();
  GridGuard guard{g};
  g->kind = 1;
  g->n = n;
  g->np = n;
  g->vdd = vdd;
  if ((rc = common_init(g))) return rc;
  tr.mark("init");
  // The colour-permuted store is built on the device (pg_csr_device.cu) when
  // the graph is bipartite, else -- or with PGB200_CSR_HOST set
  // -- by the host builder (pg_csr_build.cpp); both give the same store.
  std::vector<int64_t> iperm_h;
  bool done = false;
  if (!std::getenv("PGB200_CSR_HOST")) {
    const int64_t *du = bu, *dv = bv;
    const double *dg = bg, *dc = cap;
    void *tmp[4] = {nullptr, nullptr, nullptr, nullptr};
    struct TmpGuard {
      void **p;
      ~TmpGuard() {
        for (int k = 0; k < 4; ++k)
          if (p[k]) dfree(p[k]);
      }
    } tg{tmp};
    if (mem == PG_MEM_HOST) {
      int64_t *a = nullptr, *b = nullptr;
      double *c = nullptr, *d = nullptr;
      if ((rc = dalloc(&a, m)) || (rc = dalloc(&b, m)) || (rc = dalloc(&c, m)) || (rc = dalloc(&d, n))) {
        for (void *q : {(void *)a, (void *)b, (void *)c, (void *)d})
          if (q) dfree(q);
        return rc;
      }
      tmp[0] = a, tmp[1] = b, tmp[2] = c, tmp[3] = d;
      if (m > 0) {
        CK(cudaMemcpyAsync(a, bu, sizeof(int64_t) * m, cudaMemcpyHostToDevice, g->stream));
        CK(cudaMemcpyAsync(b, bv, sizeof(int64_t) * m, cudaMemcpyHostToDevice, g->stream));
        CK(cudaMemcpyAsync(c, bg, sizeof(double) * m, cudaMemcpyHostToDevice, g->stream));
      }
      CK(cudaMemcpyAsync(d, cap, sizeof(double) * n, cudaMemcpyHostToDevice, g->stream));
      du = a, dv = b, dg = c, dc = d;
    }
    std::string err;
    if ((rc = build_csr_device(g, n, m, du, dv, dg, dc, &done, err))) {
      set_error(err);
      return rc;
    }
    if (done) {
      iperm_h.resize((size_t)n);
      CK(cudaMemcpy(iperm_h.data(), g->iperm, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    }
    tr.mark(done ? "build (device)" : "device build declined (not bipartite)");
  }
  if (!done) {
    std::vector<int64_t> u, v;
    std::vector<double> gg, c;
    if ((rc = to_host(bu, m, mem, u)) || (rc = to_host(bv, m, mem, v)) || (rc = to_host(bg, m, mem, gg)) ||
        (rc = to_host(cap, n, mem, c)))
      return rc;
    for (int64_t k = 0; k < n; ++k) REQUIRE(c[k] >= 0 && std::isfinite(c[k]), "cap must be finite and >= 0");
    CsrHost H;
    std::string err;
    if (build_csr(n, m, u.data(), v.data(), gg.data(), H, err) != 0) {
      set_error(err);
      return PG_EINVAL;
    }
    g->ncolor = (int32_t)H.color_ptr.size() - 1;
    g->color_ptr = H.color_ptr;
    std::vector<double> cp((size_t)n);
    for (int64_t k = 0; k < n; ++k) cp[H.iperm[k]] = c[k];
    const int64_t nnz = (int64_t)H.col.size();
    REQUIRE(nnz < (int64_t)INT32_MAX - 64, "CSR grids are limited to 2^31 - 64 stored entries");
    // int32 row pointers (4 B per row) and 8 elements of zero slack after
    // rowptr / col / val: the staged sweep bulk-copies 16-byte-rounded ranges
    std::vector<int32_t> rp32((size_t)n + 1 + 8, (int32_t)nnz);
    for (int64_t k = 0; k <= n; ++k) rp32[k] = (int32_t)H.rowptr[k];
    std::vector<int32_t> col_p(H.col);
    col_p.resize((size_t)nnz + 8, 0);
    std::vector<double> val_p(H.val);
    val_p.resize((size_t)nnz + 8, 0.0);
    // every kCsrR-row tile of every colour must fit the staged sweep's entry buffer
    bool fits = true;
    for (int32_t c = 0; c + 1 < (int32_t)H.color_ptr.size() && fits; ++c)
      for (int64_t r0 = H.color_ptr[c]; r0 < H.color_ptr[c + 1]; r0 += kCsrR) {
        const int64_t r1 = std::min<int64_t>(H.color_ptr[c + 1], r0 + kCsrR);
        if (H.rowptr[r1] - H.rowptr[r0] > kCsrE) {
          fits = false;
          break;
        }
      }
    g->csr_staged_ok = fits;
    if ((rc = dalloc(&g->rowptr, (int64_t)rp32.size())) || (rc = dalloc(&g->col, (int64_t)col_p.size())) ||
        (rc = dalloc(&g->val, (int64_t)val_p.size())) || (rc = dalloc(&g->perm, n)) ||
        (rc = dalloc(&g->iperm, n)) || (rc = dalloc(&g->cap, n)))
      return rc;
    if ((rc = upload(g->rowptr, rp32)) || (rc = upload(g->col, col_p)) || (rc = upload(g->val, val_p)) ||
        (rc = upload(g->perm, H.perm)) || (rc = upload(g->iperm, H.iperm)) || (rc = upload(g->cap, cp)))
      return rc;
    iperm_h = std::move(H.iperm);
    tr.mark("build (host) + uploads");
  }
  if ((rc = set_pads(g, n_pads, pad_node, pad_g, nullptr, mem, &iperm_h))) return rc;
  CK(cudaDeviceSynchronize());
  tr.mark("set_pads");
  guard.g = nullptr;
  *out = g;
  return PG_OK;
}

PG_API void pg_destroy(pg_grid *g) { free_grid(g); }

PG_API int pg_release_memory(int32_t device) {
  REQUIRE(device >= -1 && device < 64, "device must be -1 (all) or a device index < 64");
  int cur = 0;
  CK(cudaGetDevice(&cur));
  for (int dv = device < 0 ? 0 : device; dv < (device < 0 ? 64 : device + 1); ++dv) {
    DevPool *d = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      if (g_pools[dv].init && g_pools[dv].pool) d = &g_pools[dv];
    }
    if (!d) continue;
    CK(cudaSetDevice(dv));
    CK(cudaDeviceSynchronize());  // blocks freed stream-ordered on the pool stream are returned
    CK(cudaMemPoolTrimTo(d->pool, 0));
    CK(cudaMemPoolTrimTo(d->small, 0));
  }
  CK(cudaSetDevice(cur));
  return PG_OK;
}

PG_API int pg_set_stream(pg_grid *g, void *stream) {
  REQUIRE(g != nullptr, "grid is NULL");
  g->stream = (cudaStream_t)stream;
  return PG_OK;
}

PG_API int pg_set_option(pg_grid *g, const char *key, int64_t value) {
  REQUIRE(g != nullptr && key != nullptr, "grid/key is NULL");
  const std::string k(key);
  if (k == "fuse") {
    REQUIRE(value >= 0 && value <= 4, "fuse must be 0 (auto) or 1..4");
    g->fuse = (int)value;
  } else if (k == "lag") {
    REQUIRE(value == 3 || value == 4, "lag must be 3 or 4");
    g->lag = (int)value;
  } else if (k == "batch") {
    REQUIRE(value >= 1 && value <= 1024, "batch must be in 1..1024");
    g->batch = (int)value;
  } else if (k == "resident") {
    g->resident = value != 0;
  } else if (k == "pipe") {
    g->pipe = value != 0;
  } else if (k == "pdl") {
    g->pdl = value != 0;
  } else if (k == "l2keep") {
    REQUIRE(value >= -1 && value < 64, "l2keep is a 6-bit mask (gx, gy, gz, b, 1/d, V) or -1 (auto)");
    g->l2keep = (int)value;
    if (value > 0 && (value & 31)) {
      // evict_last lines may only occupy the persisting L2 set-aside
      cudaDeviceProp prop;
      if (cudaGetDeviceProperties(&prop, g->dev) == cudaSuccess && prop.persistingL2CacheMaxSize > 0)
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)prop.persistingL2CacheMaxSize);
      cudaGetLastError();
    }
  } else if (k == "l2first") {
    REQUIRE(value >= -1 && value < 64, "l2first is a 6-bit mask (gx, gy, gz, b, 1/d, V) or -1 (auto)");
    g->l2first = (int)value;
  } else if (k == "l2promo") {
    REQUIRE(value == 0 || value == 64 || value == 128 || value == 256, "l2promo must be 0, 64, 128 or 256");
    g->l2promo = (int)value;
    g->tma_state = 0;  // re-encode the tensor maps
    if (g->slab && g->hx.G > 0 && !encode_halo_maps(g)) {
      set_error("re-encoding the slab halo tensor maps failed");
      return PG_ECUDA;
    }
  } else if (k == "colour") {
    g->colour = value != 0;
  } else if (k == "csr_stage") {
    g->csr_stage = value != 0;
  } else if (k == "graph") {
    g->use_graph = value != 0;
  } else if (k == "timing") {
    g->timing = value != 0;
  } else if (k == "rows") {
    REQUIRE(value >= 0 && value <= (1 << 20), "rows must be >= 0");
    g->rows = (int)value;
  } else if (k == "width") {
    REQUIRE(value == 0 || value == 32 || value == 64, "width must be 0 (auto), 32 or 64");
    g->width = (int)value;
  } else if (k == "stages") {
    REQUIRE(value == 0 || (value >= 6 && value <= 17), "stages must be 0 (auto) or 6..17");
    g->stages = (int)value;
  } else {
    set_error("unknown option: " + k);
    return PG_EINVAL;
  }
  // a captured sweep batch bakes in the launch configuration: recapture
  if (g->batch_exec) {
    cudaGraphExecDestroy(g->batch_exec);
    g->batch_exec = nullptr;
  }
  return PG_OK;
}

PG_API int pg_info(const pg_grid *g, int64_t *n, int32_t *layers, int32_t *ny, int32_t *nx,
                   int32_t *n_colors) {
  REQUIRE(g != nullptr, "grid is NULL");
  if (n) *n = g->n;
  if (layers) *layers = g->kind == 0 ? g->md.L : 0;
  if (ny) *ny = g->kind == 0 ? g->md.NY : 0;
  if (nx) *nx = g->kind == 0 ? g->md.NX : 0;
  if (n_colors) *n_colors = g->kind == 0 ? 2 : g->ncolor;
  return PG_OK;
}

PG_API int pg_set_sources(pg_grid *g, int64_t n_src, const int64_t *node, const int64_t *ptr,
                          const double *t, const double *i, int mem) {
  REQUIRE(g != nullptr, "grid is NULL");
  REQUIRE(n_src >= 0, "n_src must be >= 0");
  REQUIRE(mem == PG_MEM_HOST || mem == PG_MEM_DEVICE, "bad mem");
  REQUIRE(n_src == 0 || (node && ptr && t && i), "source arrays are NULL");
  int64_t npts = 0;
  if (n_src > 0) {
    if (mem == PG_MEM_HOST)
      npts = ptr[n_src];
    else
      CK(cudaMemcpy(&npts, ptr + n_src, sizeof(int64_t), cudaMemcpyDeviceToHost));
    REQUIRE(npts >= n_src, "ptr[n_src] must be >= n_src (every source needs at least one breakpoint)");
  }
  // the store is built on the device (pg_store.cu): host inputs are copied
  // there first (pinned host buffers at full PCIe / C2C speed)
  const int64_t *d_node = node, *d_ptr = ptr;
  const double *d_t = t, *d_i = i;
  void *tmp[4] = {nullptr, nullptr, nullptr, nullptr};
  struct TmpGuard {
    void **p;
    ~TmpGuard() {
      for (int k = 0; k < 4; ++k)
        if (p[k]) dfree(p[k]);
    }
  } tg{tmp};
  int rc;
  PhaseTrace tr("pg_set_sources");
  if (n_src > 0 && mem == PG_MEM_HOST) {
    int64_t *a = nullptr, *b = nullptr;
    double *c = nullptr, *d = nullptr;
    if ((rc = dalloc(&a, n_src)) || (rc = dalloc(&b, n_src + 1)) || (rc = dalloc(&c, npts)) ||
        (rc = dalloc(&d, npts))) {
      for (void *p : {(void *)a, (void *)b, (void *)c, (void *)d})
        if (p) dfree(p);
      return rc;
    }
    tmp[0] = a, tmp[1] = b, tmp[2] = c, tmp[3] = d;
    CK(cudaMemcpyAsync(a, node, sizeof(int64_t) * n_src, cudaMemcpyHostToDevice, g->stream));
    CK(cudaMemcpyAsync(b, ptr, sizeof(int64_t) * (n_src + 1), cudaMemcpyHostToDevice, g->stream));
    CK(cudaMemcpyAsync(c, t, sizeof(double) * npts, cudaMemcpyHostToDevice, g->stream));
    CK(cudaMemcpyAsync(d, i, sizeof(double) * npts, cudaMemcpyHostToDevice, g->stream));
    d_node = a, d_ptr = b, d_t = c, d_i = d;
    tr.mark("alloc+copy");
  }
  int64_t *old_i64[4] = {g->src_idx, g->src_grp, g->src_ptr, g->src_tile};
  double *old_d[2] = {g->pwl_t, g->pwl_i};
  if (n_src > 0) {
    int32_t bad = 0;
    std::string err;
    if ((rc = build_sources_device(g, n_src, d_node, d_ptr, d_t, d_i, npts, &bad, err))) {
      set_error("pg_set_sources: " + err);
      return rc;
    }
    REQUIRE(!(bad & 1), "ptr[0] must be 0 and every ptr[k] in [0, ptr[n_src]]");
    REQUIRE(!(bad & 2), "every source needs at least one breakpoint");
    REQUIRE(!(bad & 4), "source node index out of range");
    REQUIRE(!(bad & 8), "PWL breakpoint times must be strictly increasing");
    REQUIRE(!(bad & 16), "PWL breakpoints and values must be finite");
    tr.mark("build");
  } else {
    g->src_idx = g->src_grp = g->src_ptr = g->src_tile = nullptr;
    g->pwl_t = g->pwl_i = nullptr;
    g->nsrc = g->nsrc_grp = g->npts = 0;
  }
  // the new store is in place: release the previous one
  for (int64_t *p : old_i64)
    if (p) dfree(p);
  for (double *p : old_d)
    if (p) dfree(p);
  return PG_OK;
}

PG_API int pg_set_voltages(pg_grid *g, const double *v, int mem) {
  REQUIRE(g != nullptr && v != nullptr, "grid/v is NULL");
  REQUIRE(mem == PG_MEM_HOST || mem == PG_MEM_DEVICE, "bad mem");
  int rc;
  if (!g->user_buf && (rc = dalloc(&g->user_buf, g->n))) return rc;
  double *tmp = g->user_buf;
  // the values are checked on the device (host or device input) before the
  // grid's state changes
  int32_t *d_bad = nullptr;
  if ((rc = dalloc(&d_bad, 1))) return rc;
  struct FlagGuard {
    int32_t *q;
    ~FlagGuard() { dfree(q); }
  } flag_guard{d_bad};
  int32_t bad = 0;
  CK(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), g->stream));
  CK(cudaMemcpyAsync(tmp, v, sizeof(double) * g->n,
                     mem == PG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, g->stream));
  CK(finite_check_async(g, tmp, g->n, d_bad));
  CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  REQUIRE(!bad, "voltages must be finite");
  cudaError_t e = launch_scatter_user(g, tmp, g->x0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(g->V[0], g->x0, sizeof(double) * g->np, cudaMemcpyDeviceToDevice, g->stream);
  if (e == cudaSuccess) e = launch_reset_state(g);
  if (e == cudaSuccess && g->iz) e = cudaMemsetAsync(g->iz, 0, sizeof(double) * g->np, g->stream);
  if (e == cudaSuccess && g->pad_i) e = cudaMemsetAsync(g->pad_i, 0, sizeof(double) * g->npad, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return cuda_fail(e, "pg_set_voltages");
  g->traj_steps = 0;
  g->traj_h = 0.0;
  return PG_OK;
}

PG_API int pg_get_voltages(pg_grid *g, double *v, int mem) {
  REQUIRE(g != nullptr && v != nullptr, "grid/v is NULL");
  REQUIRE(mem == PG_MEM_HOST || mem == PG_MEM_DEVICE, "bad mem");
  if (mem == PG_MEM_DEVICE) {
    CK(launch_gather_user(g, v));
    CK(cudaStreamSynchronize(g->stream));
    return PG_OK;
  }
  // staged through a per-grid buffer kept until pg_destroy: no cudaMalloc /
  // cudaFree (a device-wide synchronisation) per read-back
  int rc;
  PhaseTrace tr("pg_get_voltages");
  if (!g->user_buf && (rc = dalloc(&g->user_buf, g->n))) return rc;
  double *tmp = g->user_buf;
  cudaError_t e = launch_gather_user(g, tmp);
  tr.mark("alloc+gather");
  if (e == cudaSuccess) e = cudaMemcpyAsync(v, tmp, sizeof(double) * g->n, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  tr.mark("copy");
  if (e != cudaSuccess) return cuda_fail(e, "pg_get_voltages");
  return PG_OK;
}

PG_API int pg_transient(pg_grid *g, double h, int64_t steps, double tol, double omega, int method,
                        int64_t max_sweeps, int64_t n_probe, const int64_t *probe_node,
                        double *probe_out, int mem, int64_t *sweeps_out, pg_stats *stats) {
  REQUIRE(g != nullptr, "grid is NULL");
  REQUIRE(!g->slab, "slab grids are driven through a pg_group (pg_group_transient)");
  pg_grid *gs[1] = {g};
  return pgb::run_transient(gs, 1, nullptr, h, steps, tol, omega, method, max_sweeps, n_probe,
                            probe_node, probe_out, mem, sweeps_out, stats);
}

PG_API int pg_transient_continue(pg_grid *g, double h, int64_t steps, double tol, double omega, int method,
                                 int64_t max_sweeps, int64_t n_probe, const int64_t *probe_node,
                                 double *probe_out, int mem, int64_t *sweeps_out, pg_stats *stats) {
  REQUIRE(g != nullptr, "grid is NULL");
  REQUIRE(!g->slab, "slab grids are driven through a pg_group (pg_group_transient_continue)");
  pg_grid *gs[1] = {g};
  return pgb::run_transient(gs, 1, nullptr, h, steps, tol, omega, method, max_sweeps, n_probe,
                            probe_node, probe_out, mem, sweeps_out, stats, 0.0, true);
}

PG_API int pg_dc(pg_grid *g, double t, double tol, double omega, int method, int64_t max_sweeps,
                 pg_stats *stats) {
  REQUIRE(g != nullptr, "grid is NULL");
  REQUIRE(!g->slab, "slab grids are driven through a pg_group");
  REQUIRE(std::isfinite(t), "t must be finite");
  pg_grid *gs[1] = {g};
  const int rc = pgb::run_transient(gs, 1, nullptr, INFINITY, 1, tol, omega, method, max_sweeps, 0, nullptr,
                                    nullptr, PG_MEM_HOST, nullptr, stats, t);
  // the DC point is the state a following pg_transient_continue starts from (t = 0)
  g->traj_steps = 0;
  g->traj_h = 0.0;
  return rc;
}

PG_API int pg_estimate_omega(pg_grid *g, double h, int64_t sweeps, double *rho, double *omega_opt) {
  REQUIRE(g != nullptr, "grid is NULL");
  REQUIRE(h > 0.0 && std::isfinite(h), "h must be finite and > 0");
  REQUIRE(sweeps >= 8, "need at least 8 Jacobi sweeps");
  cudaStream_t st = g->stream;
  int rc;
  const int nb = dnorm2_blocks(g);
  double *part = nullptr;
  if ((rc = dalloc(&part, 2 * (int64_t)nb))) return rc;
  struct Free {
    void *p;
    ~Free() { dfree(p); }
  } fr{part};
  // Jacobi (omega = 1) on the homogeneous system M e = 0 from the start vector
  // x(0) (b = 0): V^(k) = J^k x(0), J = I - D^{-1} M.  D^{1/2} J D^{-1/2} is
  // symmetric and D J^2 = J^T D J, so ||V^(N)||_D^2 / ||V^(N-1)||_D^2 is the
  // Rayleigh quotient of J^2 at V^(N-1): it tends to rho(J)^2 from below, with
  // an error that decays twice as fast (in the exponent) as the ratio of
  // successive norms, and it is not fooled by the +-rho pair of the 2-cyclic
  // (red-black) spectrum.  Young: omega_opt = 2 / (1 + sqrt(1 - rho^2)) for the
  // consistently ordered red-black numbering (§IV-D refers to Young).
  g->setup_ok = false;
  CK(launch_setup(g, h));
  CK(cudaMemsetAsync(g->b, 0, sizeof(double) * g->np, st));
  CK(cudaMemcpyAsync(g->V[0], g->x0, sizeof(double) * g->np, cudaMemcpyDeviceToDevice, st));
  CK(launch_reset_state(g));
  int64_t launches = 0;
  for (int64_t j = 0; j < sweeps; ++j) CK(launch_sweep(g, PG_METHOD_JACOBI, 1.0, 0.0, (int)j, 1, &launches));
  // launch j reads V[j & 1] and writes V[(j + 1) & 1]: V^(N) is in V[N & 1]
  CK(launch_dnorm2(g, part));
  std::vector<double> hp(2 * (size_t)nb);
  CK(cudaMemcpyAsync(hp.data(), part, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, st));
  CK(launch_reset_state(g));
  CK(cudaMemcpyAsync(g->V[0], g->x0, sizeof(double) * g->np, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  double s0 = 0.0, s1 = 0.0;
  for (int k = 0; k < nb; ++k) {
    s0 += hp[2 * k];
    s1 += hp[2 * k + 1];
  }
  const double sN = (sweeps & 1) ? s1 : s0, sN1 = (sweeps & 1) ? s0 : s1;
  double r = (sN1 > 0.0 && sN >= 0.0) ? std::sqrt(sN / sN1) : 0.0;
  if (!(r >= 0.0)) r = 0.0;
  if (r > 1.0) r = 1.0;
  if (rho) *rho = r;
  if (omega_opt) *omega_opt = std::min(2.0 / (1.0 + std::sqrt(std::max(0.0, 1.0 - r * r))), 1.999);
  return PG_OK;
}

PG_API int pg_tune_omega(pg_grid *g, double h, int64_t steps, double tol, int64_t n_cand, double d_omega,
                         double *omega_out, int64_t *sweeps_out) {
  REQUIRE(g != nullptr && omega_out != nullptr, "grid / omega_out is NULL");
  REQUIRE(!g->slab, "slab grids are tuned through their single-grid twin");
  REQUIRE(h > 0.0 && std::isfinite(h), "h must be finite and > 0");
  REQUIRE(steps >= 1 && n_cand >= 1 && n_cand <= 64, "steps >= 1 and 1 <= n_cand <= 64");
  REQUIRE(tol > 0.0 && d_omega >= 0.0 && std::isfinite(d_omega), "tol > 0 and d_omega >= 0");
  double rho = 0.0, omega_b = 1.0;
  int rc;
  if ((rc = pg_estimate_omega(g, h, 2000, &rho, &omega_b))) return rc;
  // Young: the SOR convergence rate falls steeply below omega_b and only
  // linearly above it (and omega_b itself has a Jordan block), so candidates
  // start at omega_b and go up; the first candidate with the fewest sweeps
  // over the first `steps` time steps from x(0) wins
  double best = omega_b;
  int64_t best_sw = -1;
  for (int64_t k = 0; k < n_cand; ++k) {
    const double om = std::min(omega_b + (double)k * d_omega, 1.999);
    pg_stats st;
    rc = pg_transient(g, h, steps, tol, om, PG_METHOD_RBSOR, 1000000, 0, nullptr, nullptr, PG_MEM_HOST, nullptr,
                      &st);
    if (rc != PG_OK && rc != PG_ENOCONV) return rc;
    const int64_t sw = rc == PG_OK ? st.sweeps_total : INT64_MAX;
    if (sweeps_out) sweeps_out[k] = sw;
    if (best_sw < 0 || sw < best_sw) {
      best_sw = sw;
      best = om;
    }
  }
  // leave the grid at x(0) (as after creation / pg_set_voltages)
  CK(cudaMemcpyAsync(g->V[0], g->x0, sizeof(double) * g->np, cudaMemcpyDeviceToDevice, g->stream));
  CK(launch_reset_state(g));
  if (g->iz) CK(cudaMemsetAsync(g->iz, 0, sizeof(double) * g->np, g->stream));
  if (g->pad_i) CK(cudaMemsetAsync(g->pad_i, 0, sizeof(double) * g->npad, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  g->traj_steps = 0;
  g->traj_h = 0.0;
  *omega_out = best;
  return PG_OK;
}

}  // extern "C"

namespace pgb {

// CUDA graph of one full batch of sweep launches (launch indices 0..batch-1
// relative to ctl->jbase, then jbase += batch), captured on a private stream
// and cached per (omega, tol, method, F, batch, stream).  Replaying it replaces
// `batch` + 1 host launches by one graph launch (small grids are launch-bound).
int batch_graph(pg_grid *g, int method, double omega, double tol, int F, Exchange *ex) {
  // ex: a host-driven exchange after every sweep launch (NCCL norm allreduce
  // + halo send/recv) captured into the same graph, so the host leaves the
  // per-launch loop; its per-launch buffers depend on the launch index only
  // modulo the norm ring (batch % kRing == 0), so one capture serves every batch
  const double key[7] = {omega, tol, (double)method, (double)F, (double)g->batch,
                         (double)(uintptr_t)g->stream, (double)(uintptr_t)ex};
  if (g->batch_exec && std::memcmp(key, g->graph_key, sizeof(key)) == 0) return PG_OK;
  if (g->batch_exec) {
    cudaGraphExecDestroy(g->batch_exec);
    g->batch_exec = nullptr;
  }
  if (!g->cap_stream) CK(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
  cudaStream_t user = g->stream;
  g->stream = g->cap_stream;
  cudaGraph_t graph = nullptr;
  int64_t dummy = 0;
  cudaError_t e = cudaStreamBeginCapture(g->cap_stream, cudaStreamCaptureModeThreadLocal);
  for (int b = 0; e == cudaSuccess && b < g->batch; ++b) {
    e = launch_sweep(g, method, omega, tol, b, F, &dummy);
    if (e == cudaSuccess && ex) e = ex->after_sweep(b, b, &dummy);
  }
  if (e == cudaSuccess) e = launch_batch_advance(g, g->batch);
  cudaError_t e2 = cudaStreamEndCapture(g->cap_stream, &graph);
  g->stream = user;
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&g->batch_exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    g->batch_exec = nullptr;
    return cuda_fail(e, "capturing the sweep batch graph");
  }
  std::memcpy(g->graph_key, key, sizeof(key));
  return PG_OK;
}

// Algorithm 1 over ng grids advanced in lockstep on grid 0's stream (ng > 1:
// the slabs of a partitioned mesh, `ex` refreshes their ghost rows and makes
// the convergence norm global after every sweep launch).
int run_transient(pg_grid **gs, int ng, Exchange *ex, double h, int64_t steps, double tol,
                  double omega, int method, int64_t max_sweeps, int64_t n_probe,
                  const int64_t *probe_node, double *probe_out, int mem, int64_t *sweeps_out,
                  pg_stats *stats, double t_dc, bool cont) {
  pg_grid *g = gs[0];
  const bool dc = std::isinf(h);  // DC analysis (pg_dc): one solve of G v = b(t_dc)
  REQUIRE(h > 0.0 && (std::isfinite(h) || dc), "h must be finite and > 0");
  REQUIRE(steps >= 0, "steps must be >= 0");
  REQUIRE(omega > 0.0 && omega < 2.0, "omega must be in (0, 2) (Eq. (15) convergence range)");
  REQUIRE(method == PG_METHOD_RBSOR || method == PG_METHOD_JACOBI, "unknown method");
  REQUIRE(max_sweeps >= 1, "max_sweeps must be >= 1");
  REQUIRE(!std::isnan(tol), "tol is NaN");
  REQUIRE(n_probe >= 0 && (n_probe == 0 || (probe_node && probe_out)), "bad probe arrays");
  REQUIRE(n_probe == 0 || ng == 1, "probes are recorded on single grids only");
  REQUIRE(mem == PG_MEM_HOST || mem == PG_MEM_DEVICE, "bad mem");
  for (int k = 0; k < ng; ++k) {
    REQUIRE(gs[k] != nullptr, "grid is NULL");
    REQUIRE(!gs[k]->slab || method == PG_METHOD_RBSOR, "slab grids support the red-black sweep only");
    REQUIRE(gs[k]->stream == g->stream, "grids of a group must share one stream");
    REQUIRE(!cont || gs[k]->traj_steps == 0 || gs[k]->traj_h == h,
            "pg_transient_continue: h differs from the h of the steps taken so far");
  }
  // first step index of this call: steps s0 + 1 .. s0 + steps at t = s h
  const int64_t s0 = cont ? g->traj_steps : 0;

  int rc;
  // ---- probes
  std::vector<int64_t> pn;
  if ((rc = to_host(probe_node, n_probe, mem, pn))) return rc;
  std::vector<int64_t> iperm_h;
  if (g->kind == 1 && n_probe > 0) {
    iperm_h.resize((size_t)g->n);
    CK(cudaMemcpy(iperm_h.data(), g->iperm, sizeof(int64_t) * g->n, cudaMemcpyDeviceToHost));
  }
  std::vector<int64_t> pidx((size_t)n_probe);
  for (int64_t k = 0; k < n_probe; ++k) {
    REQUIRE(pn[k] >= 0 && pn[k] < g->n, "probe node index out of range");
    pidx[k] = storage_index(g, pn[k], &iperm_h);
  }
  int64_t *d_pidx = nullptr;
  double *d_pout = nullptr;
  struct Tmp {
    int64_t **a;
    double **b;
    bool own_b;
    ~Tmp() {
      if (*a) dfree(*a);
      if (own_b && *b) dfree(*b);
    }
  } tmp{&d_pidx, &d_pout, mem == PG_MEM_HOST};
  if (n_probe > 0) {
    if ((rc = dalloc(&d_pidx, n_probe))) return rc;
    if ((rc = upload(d_pidx, pidx))) return rc;
    if (mem == PG_MEM_HOST) {
      if ((rc = dalloc(&d_pout, (steps + 1) * n_probe))) return rc;
    } else {
      d_pout = probe_out;
    }
  }
  for (int k = 0; k < ng; ++k) {
    pg_grid *q = gs[k];
    if (q->dev_sweeps_cap < steps + 1) {
      if (q->dev_sweeps) dfree(q->dev_sweeps);
      q->dev_sweeps = nullptr;
      q->dev_sweeps_cap = 0;
      if ((rc = dalloc(&q->dev_sweeps, steps + 1))) return rc;
      q->dev_sweeps_cap = steps + 1;
    }
  }
  cudaStream_t st = g->stream;
  cudaEvent_t ev0, ev1, poll[2];
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  CK(cudaEventCreateWithFlags(&poll[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&poll[1], cudaEventDisableTiming));
  struct Ev {
    cudaEvent_t *e;
    ~Ev() {
      for (int k = 0; k < 4; ++k) cudaEventDestroy(e[k]);
    }
  };
  cudaEvent_t evs[4] = {ev0, ev1, poll[0], poll[1]};
  Ev evguard{evs};

  int64_t launches = 0;
  // a single grid, or one slab per process whose exchange is fused into the
  // sweep kernels (peer memory), has nothing to do between sweep launches
  const bool quiet = ng == 1 && (ex == nullptr || ex->fused());
  // a host-driven exchange of one slab per process (NCCL) is captured into
  // the batch graph together with the sweeps (NCCL calls are capturable)
  const bool captured_ex = ng == 1 && ex != nullptr && !ex->fused() && ex->capturable() &&
                           g->batch % kRing == 0;
  const bool graph_ok = g->use_graph && (quiet || captured_ex);
  // consecutive sweep launches may overlap (PDL): launch j > 0 of a batch
  // directly follows launch j - 1 in the stream
  for (int k = 0; k < ng; ++k) gs[k]->pdl_ok = false;
  g->pdl_ok = g->pdl != 0 && quiet;
  const bool resident = ng == 1 && ex == nullptr && resident_ok(g, method);
  const int F = sweeps_per_launch(g, method);
  for (int k = 1; k < ng; ++k)
    REQUIRE(sweeps_per_launch(gs[k], method) == F, "grids of a group must use the same fuse option");
  const int flips = (g->kind == 0 || method == PG_METHOD_JACOBI) ? 1 : 0;
  const int64_t max_launch = (max_sweeps + F - 1) / F;

  CK(cudaEventRecord(ev0, st));
  for (int k = 0; k < ng; ++k) {
    pg_grid *q = gs[k];
    // a new transient starts from x(0) with zero inductor currents; a
    // continuation keeps V (ping-pong parity included) and the currents
    if (!cont) CK(cudaMemcpyAsync(q->V[0], q->x0, sizeof(double) * q->np, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(q->dev_sweeps, 0, sizeof(int64_t) * (steps + 1), st));
    if (!cont && q->iz) CK(cudaMemsetAsync(q->iz, 0, sizeof(double) * q->np, st));
    if (!cont && q->pad_i) CK(cudaMemsetAsync(q->pad_i, 0, sizeof(double) * q->npad, st));
    CK(launch_reset_state(q, cont));
    if (!(q->setup_ok && q->setup_h == h)) {  // h = +inf (DC) is a setup of its own
      q->setup_ok = false;
      CK(launch_setup(q, h));
      launches += 3;
    }
    launches += 1;
  }
  if (ex) CK(ex->begin());
  if (n_probe > 0) {
    CK(launch_probe(g, d_pidx, n_probe, d_pout));
    ++launches;
  }
  double sweep_ms = 0.0;
  int64_t sweep_launches = 0;
  auto tev = [&](int64_t k) -> cudaEvent_t {
    while ((int64_t)g->tev.size() <= k) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      g->tev.push_back(e);
    }
    return g->tev[(size_t)k];
  };
  for (int64_t s = 1; s <= steps; ++s) {
    for (int k = 0; k < ng; ++k) {
      CK(launch_rhs(gs[k], h, dc ? t_dc : (double)(s0 + s) * h));
      ++launches;
    }
    // option "timing": an event pair around the step's sweep launches (read
    // after the run, so timing adds no synchronisation and keeps the graphs)
    if (g->timing && !tev(2 * (s - 1) + 1)) return cuda_fail(cudaErrorMemoryAllocation, "timing events");
    if (resident) {
      // the whole sweep loop of the step in one launch (small meshes)
      if (g->timing) CK(cudaEventRecord(tev(2 * (s - 1)), st));
      CK(launch_rb_resident(g, omega, tol, max_sweeps, s));
      ++launches;
      if (g->timing) CK(cudaEventRecord(tev(2 * (s - 1) + 1), st));
      if (g->rlc) {
        CK(launch_inductor_update(g, h));
        launches += 2;
      }
      if (n_probe > 0) {
        CK(launch_probe(g, d_pidx, n_probe, d_pout + s * n_probe));
        ++launches;
      }
      continue;
    }
    int64_t j = 0;
    int pending = -1;  // poll slot of the previous batch
    int slot = 0;
    if (g->timing) CK(cudaEventRecord(tev(2 * (s - 1)), st));
    while (j < max_launch) {
      const int64_t nb = std::min<int64_t>(g->batch, max_launch - j);
      // a full batch (batch launches of F sweeps) of a single grid replays the
      // captured CUDA graph; launch indices are relative to ctl->jbase
      const bool full = nb == g->batch && (j + nb) * F <= max_sweeps;
      if (full && graph_ok && (j > 0 || g->batch_exec != nullptr)) {
        if ((rc = batch_graph(g, method, omega, tol, F, captured_ex ? ex : nullptr))) return rc;
        CK(cudaGraphLaunch(g->batch_exec, st));
        launches += nb + 1;
      } else {
        for (int64_t b = 0; b < nb; ++b) {
          const int nsw = (int)std::min<int64_t>(F, max_sweeps - (j + b) * F);
          for (int k = 0; k < ng; ++k) CK(launch_sweep(gs[k], method, omega, tol, (int)b, nsw, &launches));
          if (ex) CK(ex->after_sweep((int)(j + b), (int)b, &launches));
        }
        for (int k = 0; k < ng; ++k) CK(launch_batch_advance(gs[k], (int)nb));
        launches += ng;
      }
      j += nb;
      if (!(tol > 0.0) || j >= max_launch) continue;
      CK(cudaMemcpyAsync(&g->done_host[slot], &g->ctl->done, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaEventRecord(poll[slot], st));
      if (pending >= 0) {
        CK(cudaEventSynchronize(poll[pending]));
        if (g->done_host[pending]) break;
      }
      pending = slot;
      slot ^= 1;
    }
    if (g->timing) CK(cudaEventRecord(tev(2 * (s - 1) + 1), st));
    if (ex) CK(ex->end_step(&launches));
    for (int k = 0; k < ng; ++k) {
      CK(launch_step_end(gs[k], s, (int)j, flips, F, max_sweeps, tol));
      ++launches;
    }
    for (int k = 0; k < ng; ++k) {
      if (gs[k]->rlc) {
        CK(launch_inductor_update(gs[k], h));
        launches += 2;
      }
    }
    if (n_probe > 0) {
      CK(launch_probe(g, d_pidx, n_probe, d_pout + s * n_probe));
      ++launches;
    }
  }
  for (int k = 0; k < ng; ++k) {
    CK(launch_check_finite(gs[k]));
    ++launches;
  }
  CK(cudaEventRecord(ev1, st));
  for (int k = 1; k < ng; ++k)
    CK(cudaMemcpyAsync(gs[k]->ctl_host, gs[k]->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(g->ctl_host, g->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
  if (n_probe > 0 && mem == PG_MEM_HOST)
    CK(cudaMemcpyAsync(probe_out, d_pout, sizeof(double) * (steps + 1) * n_probe, cudaMemcpyDeviceToHost, st));
  if (sweeps_out)
    CK(cudaMemcpyAsync(sweeps_out, g->dev_sweeps, sizeof(int64_t) * (steps + 1), cudaMemcpyDeviceToHost, st));
  std::vector<int64_t> step_sweeps;
  if (g->timing) {
    step_sweeps.resize(steps + 1);
    CK(cudaMemcpyAsync(step_sweeps.data(), g->dev_sweeps, sizeof(int64_t) * (steps + 1), cudaMemcpyDeviceToHost,
                       st));
  }
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ev0, ev1));
  if (g->timing) {
    // sweep-phase time of every step; launches that did work = ceil(sweeps / F)
    // (the resident sweep: one launch per step)
    for (int64_t s = 1; s <= steps; ++s) {
      float m = 0.f;
      CK(cudaEventElapsedTime(&m, tev(2 * (s - 1)), tev(2 * (s - 1) + 1)));
      sweep_ms += m;
      sweep_launches += resident ? 1 : (step_sweeps[s] + F - 1) / F;
    }
  }
  const DevCtl &c = *g->ctl_host;
  if (stats) {
    stats->steps_done = steps;
    stats->sweeps_total = c.sweeps_total;
    stats->sweeps_max = c.sweeps_max;
    stats->failed_step = c.failed;
    stats->kernel_launches = launches;
    stats->last_delta = c.last_delta;
    stats->device_ms = ms;
    stats->sweep_ms = sweep_ms;
    stats->sweep_launches = sweep_launches;
    stats->sweeps_per_launch = F;
  }
  for (int k = 0; k < ng; ++k) {
    gs[k]->traj_steps = dc ? 0 : s0 + steps;
    gs[k]->traj_h = dc ? 0.0 : h;
  }
  for (int k = 0; k < ng; ++k) {
    if (gs[k]->ctl_host->diag_bad) {
      set_error("a node has a non-positive diagonal d_i (no capacitance and no conductive path; Lemma 1)");
      return PG_EINVAL;
    }
  }
  for (int k = 0; k < ng; ++k) {  // the setup for h is valid (diagonal checked)
    gs[k]->setup_ok = true;
    gs[k]->setup_h = h;
  }
  for (int k = 0; k < ng; ++k) {
    if (gs[k]->ctl_host->nonfinite) {
      set_error("an iterate became non-finite (NaN or Inf); results are invalid");
      return PG_ENONFINITE;
    }
  }
  if (c.failed) {
    set_error("step " + std::to_string(c.failed) + " did not reach tol within max_sweeps");
    return PG_ENOCONV;
  }
  return PG_OK;
}

}  // namespace pgb
