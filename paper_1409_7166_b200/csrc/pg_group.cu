// Multi-GPU slab partition of a mesh (include/pgrid.h "pg_group", DESIGN.md
// §10): every slab grid owns a contiguous block of rows and keeps G ghost rows
// of each neighbour.  After every sweep launch (F fused red-black sweeps) the
// group
//   1. max-reduces the launch's convergence norm max|dV| over all slabs, so the
//      device-side stopping test of the next launch is global (ncclAllReduce on
//      the 8-byte norm slot; bit pattern of a non-negative double, so the
//      unsigned max is the double max);
//   2. sends the G owned rows next to each boundary to the neighbour: the
//      sweep kernel itself writes them to a send buffer as it finishes them,
//      ncclSend/ncclRecv move them, and the next sweep launch reads its ghost
//      rows straight from the receive buffer through a TMA tensor map (no pack
//      or unpack kernel per launch; one unpack into V per time step).
// A fused launch with F sweeps recomputes the 2F rows next to its owned range
// from ghost data (pg_sweep_fused.cu), so G >= 2F ghost rows exchanged every
// launch reproduce the single-grid red-black iterates exactly.
//
// Transports: NCCL (one slab per process, NCCL loaded at run time with dlopen
// so the library has no link-time NCCL dependency) or "local" (n slabs on one
// device in one process, exchanged by device-to-device copies: the same
// protocol, pack/unpack kernels and ordering, used to test the partition on a
// single GPU).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "pg_internal.h"

using namespace pgb;

namespace {

#define CKR(call)                                        \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

#define REQ(cond, msg)    \
  do {                    \
    if (!(cond)) {        \
      set_error(msg);     \
      return PG_EINVAL;   \
    }                     \
  } while (0)

// ------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  // an NCCL already loaded into the process (e.g. by torch) is reused
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
    return api;
  }
  auto sym = [&](const char *name) -> void * { return dlsym(h, name); };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Send &&
           api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
  if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  return api;
}

// ------------------------------------------------------------------ kernels
// V buffer holding the current iterate after sweep launch j of the step: the
// launch wrote V[(base + j + 1) & 1] unless the step had already converged
// (then launches_done launches ran).
__device__ __forceinline__ const double *current_v(const DevCtl *c, int j, const double *V0,
                                                   const double *V1) {
  j += c->jbase;  // j is relative to the current batch
  const int64_t ran = c->done ? c->launches_done : (int64_t)j + 1;
  return ((c->base + ran) & 1) ? V1 : V0;
}

// rows [row0, row0 + G) of all layers <-> buf[(l * G + r) * NXP + x]
__global__ void k_halo_pack(MeshDims d, const double *V0, const double *V1, const DevCtl *c, int j,
                            int lo_row, int hi_row, int G, double *lo_buf, double *hi_buf) {
  const double *V = current_v(c, j, V0, V1);
  const int64_t per = (int64_t)d.L * G * d.NXP;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 2 * per;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int side = k >= per;
    const int64_t q = side ? k - per : k;
    const int row0 = side ? hi_row : lo_row;
    double *buf = side ? hi_buf : lo_buf;
    if (row0 < 0 || buf == nullptr) continue;
    const int64_t x = q % d.NXP, lr = q / d.NXP;
    const int64_t l = lr / G, r = lr % G;
    buf[q] = V[l * d.layer_stride + (row0 + r) * d.NXP + x];
  }
}

__global__ void k_halo_unpack(MeshDims d, double *V0, double *V1, const DevCtl *c, int j, int lo_row,
                              int hi_row, int G, const double *lo_buf, const double *hi_buf) {
  double *V = const_cast<double *>(current_v(c, j, V0, V1));
  const int64_t per = (int64_t)d.L * G * d.NXP;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 2 * per;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int side = k >= per;
    const int64_t q = side ? k - per : k;
    const int row0 = side ? hi_row : lo_row;
    const double *buf = side ? hi_buf : lo_buf;
    if (row0 < 0 || buf == nullptr) continue;
    const int64_t x = q % d.NXP, lr = q / d.NXP;
    const int64_t l = lr / G, r = lr % G;
    V[l * d.layer_stride + (row0 + r) * d.NXP + x] = buf[q];
  }
}

// local transport: max of the launch's norm slot over all slabs, written back
__global__ void k_group_max(DevCtl **ctls, int n, int slot) {
  unsigned long long m = 0ull;
  for (int k = 0; k < n; ++k) m = max(m, ctls[k]->dmax[slot]);
  for (int k = 0; k < n; ++k) ctls[k]->dmax[slot] = m;
}

int grid_for(int64_t work, int num_sms) {
  int64_t g = (work + 255) / 256;
  g = std::min<int64_t>(g, (int64_t)num_sms * 8);
  return (int)std::max<int64_t>(g, 1);
}

}  // namespace

struct pg_group : public pgb::Exchange {
  int kind = 0;  // 0 local, 1 nccl
  std::vector<pg_grid *> slabs;
  int rank = 0, nranks = 1, G = 0;
  int64_t halo = 0;  // doubles per side per slab
  std::vector<double *> send_lo, send_hi, recv_lo, recv_hi;
  DevCtl **d_ctls = nullptr;
  ncclComm_t comm = nullptr;
  std::string err;

  bool has_lo(int k) const { return (kind == 0 ? k : rank) > 0; }
  bool has_hi(int k) const { return (kind == 0 ? k : rank) < nranks - 1; }

  cudaError_t after_sweep(int j, int jr, int64_t *launches) override {
    cudaStream_t st = slabs[0]->stream;
    const int slot = j & (kRing - 1);
    cudaError_t e;
    // 1. global convergence norm
    if (kind == 0) {
      k_group_max<<<1, 1, 0, st>>>(d_ctls, (int)slabs.size(), slot);
      ++*launches;
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else {
      const NcclApi &N = nccl();
      unsigned long long *p = &slabs[0]->ctl->dmax[slot];
      if (N.AllReduce(p, p, 1, ncclUint64, ncclMax, comm, st) != ncclSuccess) return cudaErrorUnknown;
    }
    // 2. the sweep kernel already wrote the G owned rows next to each
    //    boundary into the send buffers; the next launch reads its ghost rows
    //    from the receive buffers (no pack / unpack per launch)
    // 3. transport
    const size_t bytes = sizeof(double) * (size_t)halo;
    if (kind == 0) {
      for (size_t k = 0; k + 1 < slabs.size(); ++k) {
        if ((e = cudaMemcpyAsync(recv_lo[k + 1], send_hi[k], bytes, cudaMemcpyDeviceToDevice, st))) return e;
        if ((e = cudaMemcpyAsync(recv_hi[k], send_lo[k + 1], bytes, cudaMemcpyDeviceToDevice, st))) return e;
      }
    } else {
      const NcclApi &N = nccl();
      bool ok = N.GroupStart() == ncclSuccess;
      if (ok && has_lo(0)) {
        ok = N.Send(send_lo[0], (size_t)halo, ncclFloat64, rank - 1, comm, st) == ncclSuccess &&
             N.Recv(recv_lo[0], (size_t)halo, ncclFloat64, rank - 1, comm, st) == ncclSuccess;
      }
      if (ok && has_hi(0)) {
        ok = N.Send(send_hi[0], (size_t)halo, ncclFloat64, rank + 1, comm, st) == ncclSuccess &&
             N.Recv(recv_hi[0], (size_t)halo, ncclFloat64, rank + 1, comm, st) == ncclSuccess;
      }
      if (N.GroupEnd() != ncclSuccess || !ok) return cudaErrorUnknown;
    }
    return cudaGetLastError();
  }

  // initial state: the ghost rows of V[0] (x(0)) seed the receive buffers
  cudaError_t begin() override {
    cudaStream_t st = slabs[0]->stream;
    for (size_t k = 0; k < slabs.size(); ++k) {
      pg_grid *g = slabs[k];
      k_halo_pack<<<grid_for(2 * halo, g->num_sms), 256, 0, st>>>(
          g->md, g->V[0], g->V[1], g->ctl, -1, has_lo((int)k) ? g->y_begin - G : -1,
          has_hi((int)k) ? g->y_end : -1, G, recv_lo[k], recv_hi[k]);
    }
    return cudaGetLastError();
  }

  // end of a step: the received ghost rows go into V (the right-hand side and
  // the inductor update of the next step read them there)
  cudaError_t end_step(int64_t *launches) override {
    cudaStream_t st = slabs[0]->stream;
    for (size_t k = 0; k < slabs.size(); ++k) {
      pg_grid *g = slabs[k];
      k_halo_unpack<<<grid_for(2 * halo, g->num_sms), 256, 0, st>>>(
          g->md, g->V[0], g->V[1], g->ctl, -1, has_lo((int)k) ? g->y_begin - G : -1,
          has_hi((int)k) ? g->y_end : -1, G, recv_lo[k], recv_hi[k]);
      ++*launches;
    }
    return cudaGetLastError();
  }

  void release() {
    for (pg_grid *g : slabs)
      if (g) g->hx = SlabHalo{};
    for (auto *v : {&send_lo, &send_hi, &recv_lo, &recv_hi})
      for (double *p : *v)
        if (p) cudaFree(p);
    if (d_ctls) cudaFree(d_ctls);
    if (comm) nccl().CommDestroy(comm);
    d_ctls = nullptr;
    comm = nullptr;
  }
};

namespace {

int check_slab(const pg_grid *g, int G, bool lo, bool hi) {
  REQ(g != nullptr, "slab grid is NULL");
  REQ(g->kind == 0 && g->slab, "group members must be mesh grids marked with pg_set_slab");
  REQ(!lo || g->y_begin >= G, "a slab with a lower neighbour needs G ghost rows below its owned rows");
  REQ(!hi || g->y_end + G <= g->md.NY, "a slab with an upper neighbour needs G ghost rows above its owned rows");
  REQ(lo || g->y_begin == 0, "the first slab owns its lowest row (no ghost rows below the grid)");
  REQ(hi || g->y_end == g->md.NY, "the last slab owns its highest row");
  return PG_OK;
}

int alloc_bufs(pg_group *grp);

// hand the exchange buffers to the slab grids' sweeps
int attach_halo(pg_group *grp) {
  for (size_t k = 0; k < grp->slabs.size(); ++k) {
    pg_grid *g = grp->slabs[k];
    SlabHalo &h = g->hx;
    h.G = grp->G;
    h.has_lo = grp->has_lo((int)k);
    h.has_hi = grp->has_hi((int)k);
    h.send_lo = grp->send_lo[k];
    h.send_hi = grp->send_hi[k];
    h.recv_lo = grp->recv_lo[k];
    h.recv_hi = grp->recv_hi[k];
    if (!encode_halo_maps(g)) {
      set_error("encoding the ghost-row tensor maps failed");
      return PG_ECUDA;
    }
  }
  return PG_OK;
}

int alloc_bufs(pg_group *grp) {
  const pg_grid *g0 = grp->slabs[0];
  for (pg_grid *g : grp->slabs)
    REQ(g->md.L == g0->md.L && g->md.NXP == g0->md.NXP && g->md.NX == g0->md.NX,
        "slabs must share layers and columns");
  grp->halo = (int64_t)g0->md.L * grp->G * g0->md.NXP;
  const size_t n = grp->slabs.size();
  for (auto *v : {&grp->send_lo, &grp->send_hi, &grp->recv_lo, &grp->recv_hi}) v->assign(n, nullptr);
  for (size_t k = 0; k < n; ++k) {
    for (auto *v : {&grp->send_lo, &grp->send_hi, &grp->recv_lo, &grp->recv_hi}) {
      cudaError_t e = cudaMalloc((void **)&(*v)[k], sizeof(double) * (size_t)grp->halo);
      if (e != cudaSuccess) {
        set_error(std::string("halo buffer allocation failed: ") + cudaGetErrorString(e));
        return PG_ENOMEM;
      }
      cudaMemset((*v)[k], 0, sizeof(double) * (size_t)grp->halo);
    }
  }
  return PG_OK;
}

}  // namespace

extern "C" {

PG_API int pg_set_slab(pg_grid *g, int32_t y_begin, int32_t y_end, int32_t y0_parity) {
  REQ(g != nullptr, "grid is NULL");
  if (g->kind != 0) {
    set_error("slabs are defined for mesh grids only");
    return PG_ESTATE;
  }
  REQ(0 <= y_begin && y_begin < y_end && y_end <= g->md.NY, "need 0 <= y_begin < y_end <= ny");
  g->slab = true;
  g->y_begin = y_begin;
  g->y_end = y_end;
  g->ypar = y0_parity & 1;
  return PG_OK;
}

PG_API int pg_nccl_unique_id(void *id128) {
  REQ(id128 != nullptr, "id buffer is NULL");
  const NcclApi &N = nccl();
  if (!N.ok) {
    set_error(N.why);
    return PG_ESTATE;
  }
  ncclUniqueId id;
  ncclResult_t r = N.GetUniqueId(&id);
  if (r != ncclSuccess) {
    set_error(std::string("ncclGetUniqueId: ") + N.GetErrorString(r));
    return PG_ECUDA;
  }
  std::memcpy(id128, &id, sizeof(id));
  return PG_OK;
}

PG_API int pg_group_nccl(pg_grid *slab, const void *id128, int32_t nranks, int32_t rank, int32_t ghost,
                         pg_group **out) {
  if (out) *out = nullptr;
  REQ(out != nullptr && id128 != nullptr, "out/id is NULL");
  REQ(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
  REQ(ghost >= 1 && ghost <= 64, "ghost rows must be in 1..64");
  int rc;
  if ((rc = check_slab(slab, ghost, rank > 0, rank < nranks - 1))) return rc;
  const NcclApi &N = nccl();
  if (!N.ok) {
    set_error(N.why);
    return PG_ESTATE;
  }
  pg_group *grp = new pg_group();
  grp->kind = 1;
  grp->slabs = {slab};
  grp->rank = rank;
  grp->nranks = nranks;
  grp->G = ghost;
  if ((rc = alloc_bufs(grp)) || (rc = attach_halo(grp))) {
    grp->release();
    delete grp;
    return rc;
  }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclResult_t r = N.CommInitRank(&grp->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    set_error(std::string("ncclCommInitRank: ") + N.GetErrorString(r));
    grp->comm = nullptr;
    grp->release();
    delete grp;
    return PG_ECUDA;
  }
  *out = grp;
  return PG_OK;
}

PG_API int pg_group_local(int32_t n, pg_grid *const *slabs, int32_t ghost, pg_group **out) {
  if (out) *out = nullptr;
  REQ(out != nullptr && slabs != nullptr, "out/slabs is NULL");
  REQ(n >= 1, "need at least one slab");
  REQ(ghost >= 1 && ghost <= 64, "ghost rows must be in 1..64");
  int rc;
  for (int k = 0; k < n; ++k)
    if ((rc = check_slab(slabs[k], ghost, k > 0, k < n - 1))) return rc;
  pg_group *grp = new pg_group();
  grp->kind = 0;
  grp->slabs.assign(slabs, slabs + n);
  grp->nranks = n;
  grp->G = ghost;
  if ((rc = alloc_bufs(grp)) || (rc = attach_halo(grp))) {
    grp->release();
    delete grp;
    return rc;
  }
  std::vector<DevCtl *> ctls(n);
  for (int k = 0; k < n; ++k) ctls[k] = slabs[k]->ctl;
  cudaError_t e = cudaMalloc((void **)&grp->d_ctls, sizeof(DevCtl *) * n);
  if (e == cudaSuccess)
    e = cudaMemcpy(grp->d_ctls, ctls.data(), sizeof(DevCtl *) * n, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    grp->release();
    delete grp;
    return cuda_fail(e, "pg_group_local");
  }
  *out = grp;
  return PG_OK;
}

PG_API int pg_group_transient(pg_group *grp, double h, int64_t steps, double tol, double omega,
                              int64_t max_sweeps, int64_t *sweeps_out, pg_stats *stats) {
  REQ(grp != nullptr, "group is NULL");
  for (pg_grid *g : grp->slabs)
    REQ(2 * sweeps_per_launch(g, PG_METHOD_RBSOR) <= grp->G,
        "ghost rows must cover 2 F rows (F = fuse option): lower fuse or rebuild the slabs");
  return run_transient(grp->slabs.data(), (int)grp->slabs.size(), grp, h, steps, tol, omega,
                       PG_METHOD_RBSOR, max_sweeps, 0, nullptr, nullptr, PG_MEM_HOST, sweeps_out, stats);
}

PG_API void pg_group_destroy(pg_group *grp) {
  if (!grp) return;
  grp->release();
  delete grp;
}

}  // extern "C"
