// Device-side construction of the load store (pg_set_sources) and value
// checks of mesh inputs (pg_create_mesh), so that building a grid from host
// buffers costs the copies and a few kernels instead of single-threaded host
// loops over every node and source (the end-to-end path of bench.py: 134M
// nodes and 5M loads for config 4).
//
// Load store (§II-A: PWL current sources at the nodes; the fused RHS
// kernel of pg_kernels.cu sums each node's loads in a fixed order): sources
// sorted by storage index -- ties in input order (a stable LSD radix sort of
// (storage index, input position)) -- with their breakpoints gathered into
// that order, one group per node (equal storage indices), and the first group
// of every RHS tile of kRhsTile storage elements.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <string>
#include <vector>

#include "pg_internal.h"

namespace pgb {

namespace {

enum : int32_t {
  kBadPtr0 = 1,       // ptr[0] != 0 or an offset outside [0, npts]
  kBadCount = 2,      // a source with no breakpoint
  kBadNode = 4,       // node index out of range
  kBadOrder = 8,      // breakpoint times not strictly increasing
  kBadValue = 16,     // non-finite time or value
};

__device__ __forceinline__ bool finite(double x) { return fabs(x) <= 1.7976931348623157e308; }

// the breakpoint offsets alone first (0 = ptr[0] < ptr[1] < ... <= npts), so
// that the next kernel never reads outside t / v
__global__ void k_src_ptr_check(int64_t n_src, const int64_t *ptr, int64_t npts, int32_t *err) {
  int32_t e = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_src; k += (int64_t)gridDim.x * blockDim.x) {
    if (k == 0 && ptr[0] != 0) e |= kBadPtr0;
    const int64_t a = ptr[k], b = ptr[k + 1];
    if (!(b > a)) e |= kBadCount;
    if (a < 0 || b > npts) e |= kBadPtr0;
  }
  if (e) atomicOr(err, e);
}

// validation + storage index of every source (key) and its input position (value)
__global__ void k_src_keys(int64_t n_src, const int64_t *node, const int64_t *ptr, const double *t,
                           const double *v, int64_t n, int32_t mesh, MeshDims md, const int64_t *iperm,
                           int64_t *key, int64_t *pos, int64_t *len, int32_t *err) {
  int32_t e = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_src; k += (int64_t)gridDim.x * blockDim.x) {
    if (k == 0 && ptr[0] != 0) e |= kBadPtr0;
    const int64_t a = ptr[k], b = ptr[k + 1];
    if (!(b > a)) e |= kBadCount;
    const int64_t nd = node[k];
    int64_t s = 0;
    if (nd < 0 || nd >= n) {
      e |= kBadNode;
    } else if (mesh) {
      const int64_t per = (int64_t)md.NY * md.NX;
      const int64_t l = nd / per, r = nd - l * per, y = r / md.NX, x = r - y * md.NX;
      s = mesh_index(md, l, y, x);
    } else {
      s = iperm[nd];
    }
    for (int64_t q = a; q < b; ++q) {
      if (!finite(t[q]) || !finite(v[q])) e |= kBadValue;
      if (q > a && !(t[q] > t[q - 1])) e |= kBadOrder;
    }
    key[k] = s;
    pos[k] = k;
    len[k] = b > a ? b - a : 0;
  }
  if (e) atomicOr(err, e);
}

// breakpoints of source pos[q] to out_ptr[q] .. ; group heads
__global__ void k_src_gather(int64_t n_src, const int64_t *skey, const int64_t *spos, const int64_t *ptr,
                             const double *t, const double *v, const int64_t *optr, double *ot, double *ov,
                             int64_t *head) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_src; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = spos[q];
    int64_t o = optr[q];
    for (int64_t p = ptr[k]; p < ptr[k + 1]; ++p, ++o) {
      ot[o] = t[p];
      ov[o] = v[p];
    }
    head[q] = (q == 0 || skey[q] != skey[q - 1]) ? 1 : 0;
  }
}

__global__ void k_src_sorted_len(int64_t n_src, const int64_t *spos, const int64_t *len, int64_t *out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_src; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = len[spos[q]];
}

// o_ptr[n_src] = o_ptr[n_src - 1] + last length (the exclusive scan's total)
__global__ void k_src_total(int64_t n_src, const int64_t *slen, int64_t *optr) {
  optr[n_src] = optr[n_src - 1] + slen[n_src - 1];
}

// group starts: grp[gidx[q]] = q at heads (gidx = exclusive scan of head); grp[ngrp] = n_src
__global__ void k_src_groups(int64_t n_src, const int64_t *head, const int64_t *gidx, int64_t *grp) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_src; q += (int64_t)gridDim.x * blockDim.x)
    if (head[q]) grp[gidx[q]] = q;
  if (blockIdx.x == 0 && threadIdx.x == 0) grp[gidx[n_src - 1] + head[n_src - 1]] = n_src;
}

// first group of every RHS tile (lower bound of t * kRhsTile over the group nodes)
__global__ void k_src_tiles(int64_t ntile, int64_t ngrp, const int64_t *grp, const int64_t *skey, int64_t *tiles) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntile; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo_key = t * (int64_t)kRhsTile;
    int64_t lo = 0, hi = ngrp;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (skey[grp[mid]] < lo_key)
        lo = mid + 1;
      else
        hi = mid;
    }
    tiles[t] = lo;
  }
}

// mesh input checks in user layout (pg_create_mesh): values >= 0 and finite,
// gx = 0 in the last column, gy = 0 in the last row, gz = 0 in the top layer
__global__ void k_mesh_check(int64_t n, int32_t L, int32_t NY, int32_t NX, const double *a, int32_t which,
                             int32_t *err) {
  bool bad = false;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const double v = a[k];
    bad |= !(v >= 0.0) || !finite(v);
    if (which == 0) bad |= (k % NX == NX - 1) && v != 0.0;
    if (which == 1) bad |= ((k / NX) % NY == NY - 1) && v != 0.0;
    if (which == 2) bad |= (k / ((int64_t)NX * NY) == L - 1) && v != 0.0;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1 << which);
}

__global__ void k_finite_check(int64_t n, const double *a, int32_t *err) {
  bool bad = false;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    bad |= !finite(a[k]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1);
}

int grid_of(int64_t work, int num_sms) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)num_sms * 8));
}

}  // namespace

cudaError_t mesh_check_async(pg_grid *g, const double *user_array, int which, int32_t *d_err) {
  k_mesh_check<<<grid_of(g->n, g->num_sms), 256>>>(g->n, g->md.L, g->md.NY, g->md.NX, user_array, which, d_err);
  return cudaGetLastError();
}

cudaError_t finite_check_async(pg_grid *g, const double *a, int64_t n, int32_t *d_err) {
  k_finite_check<<<grid_of(n, g->num_sms), 256, 0, g->stream>>>(n, a, d_err);
  return cudaGetLastError();
}

// The load store from source arrays in device memory (node[n_src],
// ptr[n_src+1], t/v[npts]).  On success the grid's src_* arrays are replaced;
// on bad input *bad_bits is non-zero (see the enum) and the grid is unchanged.
int build_sources_device(pg_grid *g, int64_t n_src, const int64_t *node, const int64_t *ptr, const double *t,
                         const double *v, int64_t npts, int32_t *bad_bits, std::string &err) {
  *bad_bits = 0;
  cudaStream_t st = g->stream;
  const int B = 256, grid = grid_of(n_src, g->num_sms);
  // scratch: keys, positions (in / out), lengths, heads, group indices, error word
  int64_t *key = nullptr, *pos = nullptr, *skey = nullptr, *spos = nullptr, *len = nullptr, *head = nullptr,
          *gidx = nullptr;
  int32_t *d_err = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  // outputs come from the library's allocator (pg_api.cu: pool, freed with the grid)
  int64_t *o_ptr = nullptr, *o_grp = nullptr, *o_tiles = nullptr, *o_idx = nullptr;
  double *o_t = nullptr, *o_v = nullptr;
  auto out_alloc = [&](void **p, size_t bytes) -> cudaError_t {
    return dalloc_bytes(p, bytes) == PG_OK ? cudaSuccess : cudaErrorMemoryAllocation;
  };
  // scratch from the library's pool too (pg_api.cu): cudaMallocAsync on the
  // device's default pool returned its ~300 MB (config 4) to the device at
  // every synchronisation and re-mapped it on the next call (5-260 ms per
  // pg_set_sources, PGB200_TRACE)
  auto scratch = [&](void **p, size_t bytes) -> cudaError_t { return out_alloc(p, bytes); };
  auto cleanup = [&]() {
    cudaStreamSynchronize(st);
    for (void *p : {(void *)key, (void *)pos, (void *)skey, (void *)spos, (void *)len, (void *)head, (void *)gidx,
                    (void *)d_err, tmp})
      if (p) dfree_bytes(p);
  };
  auto fail = [&](cudaError_t e, const char *what) {
    cleanup();
    for (void *p : {(void *)o_ptr, (void *)o_grp, (void *)o_tiles, (void *)o_t, (void *)o_v, (void *)o_idx})
      if (p) dfree_bytes(p);
    err = std::string(what) + ": " + cudaGetErrorString(e);
    return PG_ECUDA;
  };
#define SCK(call, what)                          \
  do {                                           \
    cudaError_t _e = (call);                     \
    if (_e != cudaSuccess) return fail(_e, what); \
  } while (0)
  const size_t nb = sizeof(int64_t) * (size_t)n_src;
  SCK(scratch((void **)&key, nb), "alloc");
  SCK(scratch((void **)&pos, nb), "alloc");
  SCK(scratch((void **)&skey, nb), "alloc");
  SCK(scratch((void **)&spos, nb), "alloc");
  SCK(scratch((void **)&len, nb), "alloc");
  SCK(scratch((void **)&head, nb), "alloc");
  SCK(scratch((void **)&gidx, nb), "alloc");
  SCK(scratch((void **)&d_err, sizeof(int32_t)), "alloc");
  SCK(cudaMemsetAsync(d_err, 0, sizeof(int32_t), st), "memset");
  k_src_ptr_check<<<grid, B, 0, st>>>(n_src, ptr, npts, d_err);
  SCK(cudaGetLastError(), "k_src_ptr_check");
  int32_t p_err = 0;
  SCK(cudaMemcpyAsync(&p_err, d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
  SCK(cudaStreamSynchronize(st), "sync");
  if (p_err) {
    cleanup();
    *bad_bits = p_err;
    return PG_OK;
  }
  k_src_keys<<<grid, B, 0, st>>>(n_src, node, ptr, t, v, g->n, g->kind == 0, g->md, g->iperm, key, pos, len, d_err);
  SCK(cudaGetLastError(), "k_src_keys");
  int32_t h_err = 0;
  SCK(cudaMemcpyAsync(&h_err, d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
  SCK(cudaStreamSynchronize(st), "sync");
  if (h_err) {
    cleanup();
    *bad_bits = h_err;
    return PG_OK;
  }
  // stable sort by storage index (ties keep the input order)
  int end_bit = 1;
  while (end_bit < 63 && ((int64_t)1 << end_bit) <= g->np) ++end_bit;
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key, skey, pos, spos, n_src, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, len, len, n_src, st);
  tmp_bytes = std::max(sort_bytes, scan_bytes);
  SCK(scratch(&tmp, tmp_bytes), "alloc");
  SCK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, skey, pos, spos, n_src, 0, end_bit, st), "sort");
  // breakpoint offsets in sorted order: the sorted sources' lengths (key is
  // free after the sort), exclusively scanned, the total in o_ptr[n_src]
  k_src_sorted_len<<<grid, B, 0, st>>>(n_src, spos, len, key);
  SCK(cudaGetLastError(), "k_src_sorted_len");
  SCK(out_alloc((void **)&o_ptr, sizeof(int64_t) * (size_t)(n_src + 1)), "alloc");
  SCK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, key, o_ptr, n_src, st), "scan");
  k_src_total<<<1, 1, 0, st>>>(n_src, key, o_ptr);
  SCK(cudaGetLastError(), "k_src_total");
  SCK(out_alloc((void **)&o_t, sizeof(double) * (size_t)npts), "alloc");
  SCK(out_alloc((void **)&o_v, sizeof(double) * (size_t)npts), "alloc");
  k_src_gather<<<grid, B, 0, st>>>(n_src, skey, spos, ptr, t, v, o_ptr, o_t, o_v, head);
  SCK(cudaGetLastError(), "k_src_gather");
  SCK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, head, gidx, n_src, st), "scan");
  int64_t last[2] = {0, 0};
  SCK(cudaMemcpyAsync(&last[0], gidx + n_src - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "copy");
  SCK(cudaMemcpyAsync(&last[1], head + n_src - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "copy");
  SCK(cudaStreamSynchronize(st), "sync");
  const int64_t ngrp = last[0] + last[1];
  SCK(out_alloc((void **)&o_grp, sizeof(int64_t) * (size_t)(ngrp + 1)), "alloc");
  k_src_groups<<<grid, B, 0, st>>>(n_src, head, gidx, o_grp);
  SCK(cudaGetLastError(), "k_src_groups");
  SCK(out_alloc((void **)&o_tiles, sizeof(int64_t) * (size_t)(g->ntile + 1)), "alloc");
  SCK(out_alloc((void **)&o_idx, nb), "alloc");
  SCK(cudaMemcpyAsync(o_idx, skey, nb, cudaMemcpyDeviceToDevice, st), "copy");
  k_src_tiles<<<grid_of(g->ntile + 1, g->num_sms), B, 0, st>>>(g->ntile, ngrp, o_grp, skey, o_tiles);
  SCK(cudaGetLastError(), "k_src_tiles");
  SCK(cudaStreamSynchronize(st), "sync");
#undef SCK
  cleanup();
  g->src_idx = o_idx;
  g->src_grp = o_grp;
  g->src_ptr = o_ptr;
  g->src_tile = o_tiles;
  g->pwl_t = o_t;
  g->pwl_i = o_v;
  g->nsrc = n_src;
  g->nsrc_grp = ngrp;
  g->npts = npts;
  return PG_OK;
}

}  // namespace pgb
