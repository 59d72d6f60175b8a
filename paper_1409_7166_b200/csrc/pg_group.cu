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
#include <cstddef>
#include <cstring>
#include <mutex>
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

void load_nccl(NcclApi &api) {
  // an NCCL already loaded into the process (e.g. by torch) is reused
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
    return;
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
}

const NcclApi &nccl() {  // loaded once per process (thread-safe)
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] { load_nccl(api); });
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

// ------------------------------------------------ peer-memory exchange kernels
// wait (thread 0 of each block) until `sig` reaches `target`, with a watchdog
__device__ __forceinline__ void wait_sig(DevCtl *c, unsigned long long target) {
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    while (*(volatile unsigned long long *)&c->sig < target && !*(volatile int32_t *)&c->p2p_timeout) {
      if (clock64() - t0 > (1ll << 33)) {
        c->p2p_timeout = 1;
        break;
      }
      __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// transient start: this slab's ghost rows of x(0) (V[base]) seed the receive
// buffers of parity epoch & 1, which the first sweep launch reads
__global__ void k_halo_seed_p2p(MeshDims d, const double *V0, const double *V1, const DevCtl *c, int lo_row,
                                int hi_row, int G, double *lo_a, double *lo_b, double *hi_a, double *hi_b) {
  const double *V = c->base ? V1 : V0;
  const int par = (int)(c->epoch & 1);
  double *lo_buf = par ? lo_b : lo_a, *hi_buf = par ? hi_b : hi_a;
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

// end of a step: once every slab finished the step's last working launch, the
// ghost rows it stored into this slab's receive buffers go into V
__global__ void k_halo_unpack_p2p(MeshDims d, double *V0, double *V1, DevCtl *c, int lo_row, int hi_row, int G,
                                  const double *lo_a, const double *lo_b, const double *hi_a, const double *hi_b,
                                  int32_t nranks) {
  const int64_t ran = c->done ? c->launches_done : c->jbase;
  const int64_t en = c->epoch + ran;
  wait_sig(c, (unsigned long long)en * (unsigned long long)nranks);
  double *V = ((c->base + ran) & 1) ? V1 : V0;
  const int par = (int)(en & 1);
  const double *lo_buf = par ? lo_b : lo_a, *hi_buf = par ? hi_b : hi_a;
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

// pg_group_p2p_selftest: phase 0 marks this rank's control block and stores the
// mark into element 0 of the neighbours' receive buffers through the mapped
// pointers; phase 1 reads every rank's mark through its mapped control block
// and the neighbours' marks from this rank's own receive buffers (no waiting:
// the caller orders the phases with a host barrier)
__global__ void k_p2p_mark(DevCtl *own, int64_t token, double *peer_lo, double *peer_hi) {
  own->ipc_token = token;
  if (peer_lo) peer_lo[0] = (double)token;
  if (peer_hi) peer_hi[0] = (double)token;
  __threadfence_system();
}
__global__ void k_p2p_read(unsigned long long *const *sig_all, int n, const double *recv_lo,
                           const double *recv_hi, int64_t *out) {
  for (int r = 0; r < n; ++r) {
    const DevCtl *c = reinterpret_cast<const DevCtl *>(reinterpret_cast<const char *>(sig_all[r]) -
                                                       offsetof(DevCtl, sig));
    out[r] = *(volatile const int64_t *)&c->ipc_token;
  }
  out[n] = recv_lo ? (int64_t)*(volatile const double *)recv_lo : -1;
  out[n + 1] = recv_hi ? (int64_t)*(volatile const double *)recv_hi : -1;
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
  int kind = 0;  // 0 local (copies), 1 nccl, 2 local peer-memory, 3 ipc peer-memory
  std::vector<pg_grid *> slabs;
  int rank = 0, nranks = 1, G = 0;
  int64_t halo = 0;  // doubles per side per slab
  std::vector<double *> send_lo, send_hi, recv_lo, recv_hi, recv_lo_b, recv_hi_b;
  std::vector<void *> opened;  // peers' buffers mapped with cudaIpcOpenMemHandle
  int64_t my_ctas = 0;         // ipc: this slab's CTAs per launch (exported)
  bool p2p() const { return kind >= 2; }
  DevCtl **d_ctls = nullptr;
  ncclComm_t comm = nullptr;
  std::string err;

  bool local() const { return kind == 0 || kind == 2; }
  bool has_lo(int k) const { return (local() ? k : rank) > 0; }
  bool has_hi(int k) const { return (local() ? k : rank) < nranks - 1; }

  bool fused() const override { return p2p(); }
  // NCCL: one 8-byte allreduce and grouped send/recv of fixed buffers per
  // launch -- captured into the sweep-batch graph (the local copy transport
  // and its k_group_max over a device pointer table are capturable too)
  bool capturable() const override { return kind == 0 || kind == 1; }

  cudaError_t after_sweep(int j, int jr, int64_t *launches) override {
    // peer-memory exchange: the sweep kernel itself stored the boundary rows
    // into the neighbours' buffers and max-reduced the norm into every slab
    if (p2p()) return cudaSuccess;
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
    if (p2p()) {
      for (size_t k = 0; k < slabs.size(); ++k) {
        pg_grid *g = slabs[k];
        k_halo_seed_p2p<<<grid_for(2 * halo, g->num_sms), 256, 0, st>>>(
            g->md, g->V[0], g->V[1], g->ctl, has_lo((int)k) ? g->y_begin - G : -1,
            has_hi((int)k) ? g->y_end : -1, G, recv_lo[k], recv_lo_b[k], recv_hi[k], recv_hi_b[k]);
      }
      return cudaGetLastError();
    }
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
    if (p2p()) {
      for (size_t k = 0; k < slabs.size(); ++k) {
        pg_grid *g = slabs[k];
        k_halo_unpack_p2p<<<grid_for(2 * halo, g->num_sms), 256, 0, st>>>(
            g->md, g->V[0], g->V[1], g->ctl, has_lo((int)k) ? g->y_begin - G : -1,
            has_hi((int)k) ? g->y_end : -1, G, recv_lo[k], recv_lo_b[k], recv_hi[k], recv_hi_b[k],
            g->hx.nranks);
        ++*launches;
      }
      return cudaGetLastError();
    }
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
    for (void *p : opened) cudaIpcCloseMemHandle(p);
    opened.clear();
    for (auto *v : {&send_lo, &send_hi, &recv_lo, &recv_hi, &recv_lo_b, &recv_hi_b})
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
    h.p2p = grp->p2p();
    h.recv_lo_b = grp->recv_lo_b[k];
    h.recv_hi_b = grp->recv_hi_b[k];
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
  for (auto *v : {&grp->send_lo, &grp->send_hi, &grp->recv_lo, &grp->recv_hi, &grp->recv_lo_b, &grp->recv_hi_b})
    v->assign(n, nullptr);
  std::vector<std::vector<double *> *> bufs = {&grp->recv_lo, &grp->recv_hi};
  if (grp->p2p()) {
    bufs.push_back(&grp->recv_lo_b);
    bufs.push_back(&grp->recv_hi_b);
  } else {
    bufs.push_back(&grp->send_lo);
    bufs.push_back(&grp->send_hi);
  }
  for (size_t k = 0; k < n; ++k) {
    for (auto *v : bufs) {
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

// peer-memory exchange: every launch must be a full two-sweep launch of the
// pipeline kernel (its CTA count is part of the arrival target)
int check_p2p(const pg_grid *g) {
  REQ(g->pipe && sweep2_width(g->md.L) != 0 && sweeps_per_launch(const_cast<pg_grid *>(g), PG_METHOD_RBSOR) == 2,
      "the peer-memory exchange needs the two-sweep pipeline kernel (options fuse = 0 or 2, pipe = 1)");
  return PG_OK;
}

// fresh exchange state: epochs, arrival counter, norm ring, watchdog flag
int reset_p2p_state(pg_grid *g) {
  const size_t off = offsetof(DevCtl, epoch);
  CKR(cudaMemset(reinterpret_cast<char *>(g->ctl) + off, 0, sizeof(DevCtl) - off));
  return PG_OK;
}

// Serialised per-slab description exchanged between ranks (ipc transport)
struct P2pBlob {
  uint32_t magic, version;
  int32_t rank, nranks;
  int64_t ctas;  // informational: CTAs of one sweep launch of this slab
  cudaIpcMemHandle_t recv_lo, recv_lo_b, recv_hi, recv_hi_b, ctl;
};
constexpr uint32_t kBlobMagic = 0x50473250u;  // "PG2P"

}  // namespace

extern "C" {

PG_API int pg_set_slab(pg_grid *g, int32_t y_begin, int32_t y_end, int32_t y0_parity) {
  REQ(g != nullptr, "grid is NULL");
  if (g->kind != 0) {
    set_error("slabs are defined for mesh grids only");
    return PG_ESTATE;
  }
  REQ(0 <= y_begin && y_begin < y_end && y_end <= g->md.NY, "need 0 <= y_begin < y_end <= ny");
  if (g->md.L > kMaxLayers) {
    set_error("slab grids need the streaming sweep: at most 8 layers");
    return PG_ESTATE;
  }
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

PG_API int pg_group_local_p2p(int32_t n, pg_grid *const *slabs, int32_t ghost, pg_group **out) {
  if (out) *out = nullptr;
  REQ(out != nullptr && slabs != nullptr, "out/slabs is NULL");
  REQ(n >= 1 && n <= kMaxPeers, "peer-memory groups have 1..8 slabs");
  REQ(ghost >= 4 && ghost <= 64, "ghost rows must be in 4..64 (2 F, F = 2)");
  int rc;
  for (int k = 0; k < n; ++k) {
    if ((rc = check_slab(slabs[k], ghost, k > 0, k < n - 1))) return rc;
    if ((rc = check_p2p(slabs[k]))) return rc;
  }
  pg_group *grp = new pg_group();
  grp->kind = 2;
  grp->slabs.assign(slabs, slabs + n);
  grp->nranks = n;
  grp->G = ghost;
  if ((rc = alloc_bufs(grp))) {
    grp->release();
    delete grp;
    return rc;
  }
  // "peers" are the other slabs on this device: the kernels see exactly the
  // pointers a multi-GPU group maps from its neighbours
  for (int k = 0; k < n; ++k) {
    SlabHalo &h = slabs[k]->hx;
    h = SlabHalo{};
    h.nranks = n;
    for (int r = 0; r < n; ++r) {
      h.sig_all[r] = &slabs[r]->ctl->sig;
      h.pnorm_all[r] = slabs[r]->ctl->pnorm;
    }
    if (k > 0) {
      h.peer_lo[0] = grp->recv_hi[k - 1];
      h.peer_lo[1] = grp->recv_hi_b[k - 1];
    }
    if (k < n - 1) {
      h.peer_hi[0] = grp->recv_lo[k + 1];
      h.peer_hi[1] = grp->recv_lo_b[k + 1];
    }
    if ((rc = reset_p2p_state(slabs[k]))) {
      grp->release();
      delete grp;
      return rc;
    }
  }
  if ((rc = attach_halo(grp))) {
    grp->release();
    delete grp;
    return rc;
  }
  *out = grp;
  return PG_OK;
}

PG_API int pg_group_p2p_create(pg_grid *slab, int32_t nranks, int32_t rank, int32_t ghost, pg_group **out) {
  if (out) *out = nullptr;
  REQ(out != nullptr, "out is NULL");
  REQ(nranks >= 1 && nranks <= kMaxPeers && rank >= 0 && rank < nranks, "bad rank / nranks (1..8 ranks)");
  REQ(ghost >= 4 && ghost <= 64, "ghost rows must be in 4..64 (2 F, F = 2)");
  int rc;
  if ((rc = check_slab(slab, ghost, rank > 0, rank < nranks - 1)) || (rc = check_p2p(slab))) return rc;
  pg_group *grp = new pg_group();
  grp->kind = 3;
  grp->slabs = {slab};
  grp->rank = rank;
  grp->nranks = nranks;
  grp->G = ghost;
  slab->hx.G = ghost;  // the slab variant's grid (occupancy) decides the CTA count
  grp->my_ctas = sweep2_grid_ctas(slab);
  if ((rc = alloc_bufs(grp)) || (rc = reset_p2p_state(slab))) {
    grp->release();
    delete grp;
    return rc;
  }
  cudaDeviceSynchronize();
  *out = grp;
  return PG_OK;
}

PG_API int pg_group_p2p_export(pg_group *grp, void *blob, int64_t cap, int64_t *len) {
  REQ(grp != nullptr && grp->kind == 3, "not an ipc peer-memory group");
  REQ(len != nullptr, "len is NULL");
  *len = (int64_t)sizeof(P2pBlob);
  if (blob == nullptr) return PG_OK;
  REQ(cap >= (int64_t)sizeof(P2pBlob), "blob buffer too small");
  P2pBlob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = kBlobMagic;
  b.version = 1;
  b.rank = grp->rank;
  b.nranks = grp->nranks;
  b.ctas = grp->my_ctas;
  CKR(cudaIpcGetMemHandle(&b.recv_lo, grp->recv_lo[0]));
  CKR(cudaIpcGetMemHandle(&b.recv_lo_b, grp->recv_lo_b[0]));
  CKR(cudaIpcGetMemHandle(&b.recv_hi, grp->recv_hi[0]));
  CKR(cudaIpcGetMemHandle(&b.recv_hi_b, grp->recv_hi_b[0]));
  CKR(cudaIpcGetMemHandle(&b.ctl, grp->slabs[0]->ctl));
  std::memcpy(blob, &b, sizeof(b));
  return PG_OK;
}

PG_API int pg_group_p2p_connect(pg_group *grp, const void *blobs, int64_t blob_len) {
  REQ(grp != nullptr && grp->kind == 3, "not an ipc peer-memory group");
  REQ(blobs != nullptr && blob_len == (int64_t)sizeof(P2pBlob), "blobs: nranks records from pg_group_p2p_export");
  std::vector<P2pBlob> all((size_t)grp->nranks);
  std::memcpy(all.data(), blobs, sizeof(P2pBlob) * all.size());
  for (int r = 0; r < grp->nranks; ++r)
    REQ(all[r].magic == kBlobMagic && all[r].version == 1 && all[r].rank == r && all[r].nranks == grp->nranks,
        "inconsistent peer records (order them by rank)");
  pg_grid *g = grp->slabs[0];
  SlabHalo h;
  h.nranks = grp->nranks;
  auto open = [&](const cudaIpcMemHandle_t &hd, void **p) -> int {
    CKR(cudaIpcOpenMemHandle(p, hd, cudaIpcMemLazyEnablePeerAccess));
    grp->opened.push_back(*p);
    return PG_OK;
  };
  int rc;
  for (int r = 0; r < grp->nranks; ++r) {
    DevCtl *c = g->ctl;
    if (r != grp->rank) {
      void *p = nullptr;
      if ((rc = open(all[r].ctl, &p))) return rc;
      c = reinterpret_cast<DevCtl *>(p);
    }
    h.sig_all[r] = &c->sig;
    h.pnorm_all[r] = c->pnorm;
  }
  void *p[2];
  if (grp->rank > 0) {
    if ((rc = open(all[grp->rank - 1].recv_hi, &p[0])) || (rc = open(all[grp->rank - 1].recv_hi_b, &p[1])))
      return rc;
    h.peer_lo[0] = reinterpret_cast<double *>(p[0]);
    h.peer_lo[1] = reinterpret_cast<double *>(p[1]);
  }
  if (grp->rank < grp->nranks - 1) {
    if ((rc = open(all[grp->rank + 1].recv_lo, &p[0])) || (rc = open(all[grp->rank + 1].recv_lo_b, &p[1])))
      return rc;
    h.peer_hi[0] = reinterpret_cast<double *>(p[0]);
    h.peer_hi[1] = reinterpret_cast<double *>(p[1]);
  }
  g->hx = h;
  return attach_halo(grp);
}

PG_API int pg_group_p2p_selftest(pg_group *grp, int32_t phase, int64_t *out) {
  REQ(grp != nullptr && grp->kind == 3, "not an ipc peer-memory group");
  REQ(phase == 0 || phase == 1, "phase must be 0 (mark) or 1 (read)");
  REQ(phase == 0 || out != nullptr, "out is NULL");
  pg_grid *g = grp->slabs[0];
  REQ(g->hx.p2p, "pg_group_p2p_connect has not run");
  const int64_t token = 0x5EED0000ll + grp->rank;
  if (phase == 0) {
    k_p2p_mark<<<1, 1, 0, g->stream>>>(g->ctl, token, g->hx.peer_lo[0], g->hx.peer_hi[0]);
    CKR(cudaGetLastError());
    CKR(cudaStreamSynchronize(g->stream));
    return PG_OK;
  }
  const int n = grp->nranks;
  unsigned long long **d_sig = nullptr;
  int64_t *d_out = nullptr;
  CKR(cudaMalloc(&d_sig, sizeof(void *) * n));
  CKR(cudaMalloc(&d_out, sizeof(int64_t) * (n + 2)));
  cudaError_t e = cudaMemcpy(d_sig, g->hx.sig_all, sizeof(void *) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_p2p_read<<<1, 1, 0, g->stream>>>(d_sig, n, g->hx.has_lo ? grp->recv_lo[0] : nullptr,
                                       g->hx.has_hi ? grp->recv_hi[0] : nullptr, d_out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e == cudaSuccess) e = cudaMemcpy(out, d_out, sizeof(int64_t) * (n + 2), cudaMemcpyDeviceToHost);
  cudaFree(d_sig);
  cudaFree(d_out);
  if (e != cudaSuccess) return cuda_fail(e, "pg_group_p2p_selftest");
  return PG_OK;
}

static int group_transient(pg_group *grp, double h, int64_t steps, double tol, double omega,
                           int64_t max_sweeps, int64_t *sweeps_out, pg_stats *stats, bool cont) {
  REQ(grp != nullptr, "group is NULL");
  for (pg_grid *g : grp->slabs)
    REQ(2 * sweeps_per_launch(g, PG_METHOD_RBSOR) <= grp->G,
        "ghost rows must cover 2 F rows (F = fuse option): lower fuse or rebuild the slabs");
  if (grp->p2p()) {
    REQ(max_sweeps % 2 == 0, "the peer-memory exchange runs full two-sweep launches: max_sweeps must be even");
    int rc;
    for (pg_grid *g : grp->slabs)
      if ((rc = check_p2p(g))) return rc;
  }
  // a sweep-batch graph captured inside the group bakes the armed peer
  // protocol in (and one captured outside does not): recapture on entry / exit
  auto drop_graphs = [&] {
    for (pg_grid *g : grp->slabs)
      if (g->batch_exec) {
        cudaGraphExecDestroy(g->batch_exec);
        g->batch_exec = nullptr;
      }
  };
  for (pg_grid *g : grp->slabs) g->group_active = true;
  drop_graphs();
  const int rc = run_transient(grp->slabs.data(), (int)grp->slabs.size(), grp, h, steps, tol, omega,
                               PG_METHOD_RBSOR, max_sweeps, 0, nullptr, nullptr, PG_MEM_HOST, sweeps_out, stats,
                               0.0, cont);
  for (pg_grid *g : grp->slabs) g->group_active = false;
  drop_graphs();
  if (grp->p2p())
    for (pg_grid *g : grp->slabs)
      if (g->ctl_host->p2p_timeout) {
        set_error("peer-memory exchange: a wait for the other slabs timed out (results invalid)");
        return PG_ECUDA;
      }
  return rc;
}

PG_API int pg_group_transient(pg_group *grp, double h, int64_t steps, double tol, double omega,
                              int64_t max_sweeps, int64_t *sweeps_out, pg_stats *stats) {
  return group_transient(grp, h, steps, tol, omega, max_sweeps, sweeps_out, stats, false);
}

PG_API int pg_group_transient_continue(pg_group *grp, double h, int64_t steps, double tol, double omega,
                                       int64_t max_sweeps, int64_t *sweeps_out, pg_stats *stats) {
  return group_transient(grp, h, steps, tol, omega, max_sweeps, sweeps_out, stats, true);
}

PG_API void pg_group_destroy(pg_group *grp) {
  if (!grp) return;
  grp->release();
  delete grp;
}

}  // extern "C"
