// Device-side construction of the colour-permuted CSR store (pg_create_csr)
// for bipartite graphs -- the same store pg_csr_build.cpp builds on the host,
// element for element, in a few kernels instead of single-threaded passes over
// every node and branch (config 2: 8.4M nodes, 21M branches, ~1.7 s on the
// host).
//
// Eq. (13) sweeps the nodes in index order; the numbering "colour by colour,
// natural order inside a colour" with a colouring in which no two adjacent
// nodes share a colour makes the sweep of one colour parallel (§IV,
// DESIGN.md R12).  Here:
//   1. branch checks and node degrees (branches that carry no current --
//      self loops, zero conductance -- are dropped, as on the host);
//   2. adjacency rows: the 2 m (row, branch) entries stable-sorted by row, so a
//      row lists its branches in branch order (the host's fill order);
//   3. 2-colouring by BFS parity: a level-synchronous BFS from node 0, colour =
//      distance parity (the 2-colouring of a connected bipartite graph is unique
//      once one node's colour is fixed, so it equals the host's) --
//      with several components, every component from its smallest node (found
//      by minimum-label propagation), as the host's sequential BFS seeds them;
//   4. an edge with equal colours on both ends (not bipartite): *done = false
//      and the caller builds the store on the host (greedy colouring);
//   5. permutation (colour-major, stable), permuted row pointers, columns,
//      values and capacitances.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <string>
#include <vector>

#include "pg_internal.h"

namespace pgb {

namespace {

__device__ __forceinline__ bool fin(double x) { return fabs(x) <= 1.7976931348623157e308; }

int gridn(int64_t work, int num_sms) {
  int64_t g = (work + 255) / 256;
  if (g > (int64_t)num_sms * 16) g = (int64_t)num_sms * 16;
  return (int)(g < 1 ? 1 : g);
}

#define GSTRIDE(k, n) \
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (n); k += (int64_t)gridDim.x * blockDim.x)

// bad[0]: first branch with an endpoint out of range, bad[1]: first branch with
// a non-finite or negative conductance, bad[2]: first node with a bad cap
__global__ void k_branch_check(int64_t m, int64_t n, const int64_t *bu, const int64_t *bv, const double *bg,
                               const double *cap, unsigned long long *bad, int64_t *key, int64_t *val,
                               int64_t *deg) {
  GSTRIDE(k, m) {
    const int64_t a = bu[k], b = bv[k];
    const double gk = bg[k];
    if (a < 0 || a >= n || b < 0 || b >= n) atomicMin(&bad[0], (unsigned long long)k);
    if (!(gk >= 0.0) || !fin(gk)) atomicMin(&bad[1], (unsigned long long)k);
    const bool live = a >= 0 && a < n && b >= 0 && b < n && a != b && gk > 0.0 && fin(gk);
    // entry 2k: row a, neighbour b; entry 2k + 1: row b, neighbour a (dropped rows sort to n)
    key[2 * k] = live ? a : n;
    key[2 * k + 1] = live ? b : n;
    val[2 * k] = 2 * k;
    val[2 * k + 1] = 2 * k + 1;
    if (live) {
      atomicAdd((unsigned long long *)&deg[a], 1ull);
      atomicAdd((unsigned long long *)&deg[b], 1ull);
    }
  }
  GSTRIDE(i, n) {
    if (!(cap[i] >= 0.0) || !fin(cap[i])) atomicMin(&bad[2], (unsigned long long)i);
  }
}

// adjacency in sorted order: entry e = 2k + s -> other endpoint, conductance
__global__ void k_adj(int64_t nent, const int64_t *sval, const int64_t *bu, const int64_t *bv, const double *bg,
                      int64_t *adj, double *w) {
  GSTRIDE(q, nent) {
    const int64_t e = sval[q], k = e >> 1;
    adj[q] = (e & 1) ? bu[k] : bv[k];
    w[q] = bg[k];
  }
}

// one BFS level: frontier nodes (distance lvl) claim their unvisited neighbours;
// the frontier size is read on the device (levels are launched in batches
// without a host round trip)
__global__ void k_bfs_level(const unsigned long long *nfp, const int64_t *front, const int64_t *ptr,
                            const int64_t *adj, int32_t lvl, int32_t *dist, int64_t *next,
                            unsigned long long *nnext) {
  const int64_t nf = (int64_t)*nfp;
  GSTRIDE(q, nf) {
    const int64_t i = front[q];
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      const int64_t j = adj[k];
      if (dist[j] < 0 && atomicCAS(&dist[j], -1, lvl + 1) == -1) next[atomicAdd(nnext, 1ull)] = j;
    }
  }
}

__global__ void k_first_unvisited(int64_t n, const int32_t *dist, unsigned long long *first) {
  GSTRIDE(i, n) {
    if (dist[i] < 0) atomicMin(first, (unsigned long long)i);
  }
}

__global__ void k_seed(int64_t s, int32_t *dist, int64_t *front, unsigned long long *nf) {  // source s, level 0
  dist[s] = 0;
  front[0] = s;
  *nf = 1ull;
}

__global__ void k_carry(unsigned long long *lc, int b) { lc[0] = lc[b]; }

// connected components by minimum-label propagation (labels only decrease; at
// the fixed point every node carries the smallest index of its component)
__global__ void k_lab_init(int64_t n, int64_t *lab) {
  GSTRIDE(i, n) lab[i] = i;
}
__global__ void k_lab_hook(int64_t n, const int64_t *ptr, const int64_t *adj, int64_t *lab, int32_t *changed) {
  GSTRIDE(i, n) {
    int64_t m = lab[i];
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) m = min(m, lab[adj[k]]);
    if (m < lab[i]) {
      atomicMin((unsigned long long *)&lab[i], (unsigned long long)m);
      *changed = 1;
    }
  }
}
__global__ void k_lab_jump(int64_t n, int64_t *lab) {
  GSTRIDE(i, n) lab[i] = lab[lab[i]];
}
// every component's smallest node starts the BFS at level 0
__global__ void k_seed_all(int64_t n, const int64_t *lab, int32_t *dist, int64_t *front, unsigned long long *nf) {
  GSTRIDE(i, n) {
    if (lab[i] == i) {
      dist[i] = 0;
      front[atomicAdd(nf, 1ull)] = i;
    } else {
      dist[i] = -1;
    }
  }
}

// colour = distance parity; an edge inside one colour class: not bipartite
__global__ void k_colour_check(int64_t n, const int64_t *ptr, const int64_t *adj, const int32_t *dist,
                               int64_t *black, int32_t *conflict) {
  GSTRIDE(i, n) {
    const int32_t c = dist[i] & 1;
    black[i] = c;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
      if ((dist[adj[k]] & 1) == c) *conflict = 1;
  }
}

// colour-major stable permutation from the exclusive scan of the black flags
__global__ void k_perm(int64_t n, const int64_t *black, const int64_t *sblack, int64_t n_red, int64_t *perm,
                       int64_t *iperm, const int64_t *ptr, int64_t *len_p, const double *cap, double *cap_p) {
  GSTRIDE(i, n) {
    const int64_t p = black[i] ? n_red + sblack[i] : i - sblack[i];
    perm[p] = i;
    iperm[i] = p;
    len_p[p] = ptr[i + 1] - ptr[i];
    cap_p[p] = cap[i];
  }
}

__global__ void k_rows(int64_t n, const int64_t *perm, const int64_t *iperm, const int64_t *ptr,
                       const int64_t *adj, const double *w, const int64_t *rp, int32_t *rp32, int32_t *col,
                       double *val) {
  GSTRIDE(p, n) {
    const int64_t i = perm[p];
    int64_t o = rp[p];
    rp32[p] = (int32_t)o;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k, ++o) {
      col[o] = (int32_t)iperm[adj[k]];
      val[o] = w[k];
    }
  }
}

// slack after the arrays (the staged sweep bulk-copies 16-byte-rounded ranges)
__global__ void k_slack(int64_t n, int64_t nnz, int32_t *rp32, int32_t *col, double *val) {
  if (threadIdx.x < 8) {
    rp32[n + 1 + threadIdx.x] = (int32_t)nnz;
    col[nnz + threadIdx.x] = 0;
    val[nnz + threadIdx.x] = 0.0;
  }
  if (threadIdx.x == 0) rp32[n] = (int32_t)nnz;
}

// tiles of kCsrR rows of one colour whose entries exceed the staged sweep's buffer
__global__ void k_tile_fit(int64_t c0, int64_t c1, const int32_t *rp32, int32_t *too_big) {
  const int64_t nt = (c1 - c0 + kCsrR - 1) / kCsrR;
  GSTRIDE(t, nt) {
    const int64_t r0 = c0 + t * kCsrR, r1 = min(c1, r0 + kCsrR);
    if ((int64_t)rp32[r1] - rp32[r0] > kCsrE) *too_big = 1;
  }
}

}  // namespace

int build_csr_device(pg_grid *g, int64_t n, int64_t m, const int64_t *bu, const int64_t *bv, const double *bg,
                     const double *cap, bool *done, std::string &err) {
  *done = false;
  int rc = PG_OK;
  cudaStream_t st = g->stream;
  const int nsm = g->num_sms;
  std::vector<void *> tmp;
  auto alloc = [&](void **p, size_t bytes) -> bool {
    if (dalloc_bytes(p, bytes < 16 ? 16 : bytes) != PG_OK) return false;
    tmp.push_back(*p);
    return true;
  };
  struct Free {
    std::vector<void *> *t;
    cudaStream_t s;
    ~Free() {
      cudaStreamSynchronize(s);
      for (void *p : *t) dfree_bytes(p);
    }
  } fr{&tmp, st};
#define DCK(call, what)                                            \
  do {                                                             \
    cudaError_t _e = (call);                                       \
    if (_e != cudaSuccess) {                                       \
      err = std::string(what) + ": " + cudaGetErrorString(_e);     \
      return PG_ECUDA;                                             \
    }                                                              \
  } while (0)
#define DAL(p, bytes)                                              \
  do {                                                             \
    if (!alloc((void **)&(p), (bytes))) {                          \
      err = "out of device memory building the CSR store";        \
      return PG_ENOMEM;                                            \
    }                                                              \
  } while (0)
  const int64_t nent = 2 * m;
  int64_t *key = nullptr, *val = nullptr, *skey = nullptr, *sval = nullptr, *deg = nullptr, *ptr = nullptr;
  unsigned long long *bad = nullptr;
  DAL(bad, 4 * sizeof(unsigned long long));
  DAL(deg, sizeof(int64_t) * (size_t)(n + 1));
  DAL(ptr, sizeof(int64_t) * (size_t)(n + 1));
  if (nent > 0) {
    DAL(key, sizeof(int64_t) * (size_t)nent);
    DAL(val, sizeof(int64_t) * (size_t)nent);
    DAL(skey, sizeof(int64_t) * (size_t)nent);
    DAL(sval, sizeof(int64_t) * (size_t)nent);
  }
  DCK(cudaMemsetAsync(bad, 0xff, 4 * sizeof(unsigned long long), st), "memset");
  DCK(cudaMemsetAsync(deg, 0, sizeof(int64_t) * (size_t)(n + 1), st), "memset");
  k_branch_check<<<gridn(m > n ? m : n, nsm), 256, 0, st>>>(m, n, bu, bv, bg, cap, bad, key, val, deg);
  DCK(cudaGetLastError(), "k_branch_check");
  unsigned long long hbad[4];
  DCK(cudaMemcpyAsync(hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, st), "copy");
  DCK(cudaStreamSynchronize(st), "sync");
  if (hbad[0] != ~0ull) {
    err = "branch endpoint out of range at branch " + std::to_string(hbad[0]);
    return PG_EINVAL;
  }
  if (hbad[1] != ~0ull) {
    err = "branch conductance must be finite and >= 0 at branch " + std::to_string(hbad[1]);
    return PG_EINVAL;
  }
  if (hbad[2] != ~0ull) {
    err = "cap must be finite and >= 0";
    return PG_EINVAL;
  }
  // row pointers of the natural-order adjacency, rows in branch order
  int end_bit = 1;
  while (end_bit < 63 && ((int64_t)1 << end_bit) <= n) ++end_bit;
  size_t sort_bytes = 0, scan_bytes = 0;
  if (nent > 0) cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key, skey, val, sval, nent, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, deg, ptr, n + 1, st);
  void *cubtmp = nullptr;
  const size_t cub_bytes = sort_bytes > scan_bytes ? sort_bytes : scan_bytes;
  DAL(cubtmp, cub_bytes);
  size_t tb = cub_bytes;
  DCK(cub::DeviceScan::ExclusiveSum(cubtmp, tb, deg, ptr, n + 1, st), "scan");
  int64_t nnz = 0;
  DCK(cudaMemcpyAsync(&nnz, ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "copy");
  if (nent > 0) {
    tb = cub_bytes;
    DCK(cub::DeviceRadixSort::SortPairs(cubtmp, tb, key, skey, val, sval, nent, 0, end_bit, st), "sort");
  }
  DCK(cudaStreamSynchronize(st), "sync");
  if (nnz >= (int64_t)INT32_MAX - 64) {
    err = "CSR grids are limited to 2^31 - 64 stored entries";
    return PG_EINVAL;
  }
  int64_t *adj = nullptr;
  double *w = nullptr;
  DAL(adj, sizeof(int64_t) * (size_t)(nnz + 1));
  DAL(w, sizeof(double) * (size_t)(nnz + 1));
  if (nnz > 0) {
    k_adj<<<gridn(nnz, nsm), 256, 0, st>>>(nnz, sval, bu, bv, bg, adj, w);
    DCK(cudaGetLastError(), "k_adj");
  }
  // BFS parity colouring from node 0 (colour 0)
  int32_t *dist = nullptr;
  int64_t *fa = nullptr, *fb = nullptr;
  DAL(dist, sizeof(int32_t) * (size_t)n);
  DAL(fa, sizeof(int64_t) * (size_t)n);
  DAL(fb, sizeof(int64_t) * (size_t)n);
  DCK(cudaMemsetAsync(dist, 0xff, sizeof(int32_t) * (size_t)n, st), "memset");
  unsigned long long *cnt = bad;  // reused: cnt[1] first unvisited node
  // levels in batches of kB launches; lc[t] = frontier size of the batch's level t
  constexpr int kB = 32;
  unsigned long long *lc = nullptr;
  DAL(lc, sizeof(unsigned long long) * (kB + 1));
  int64_t *buf[2] = {fa, fb};  // level l's frontier in buf[l & 1] (kB even)
  const int bfs_grid = nsm * 8;
  auto bfs = [&]() -> int {  // from the level-0 frontier in fa (size lc[0])
    for (int32_t lvl = 0;; lvl += kB) {
      DCK(cudaMemsetAsync(lc + 1, 0, sizeof(unsigned long long) * kB, st), "memset");
      for (int t = 0; t < kB; ++t)
        k_bfs_level<<<bfs_grid, 256, 0, st>>>(lc + t, buf[t & 1], ptr, adj, lvl + t, dist, buf[(t + 1) & 1],
                                              lc + t + 1);
      DCK(cudaGetLastError(), "k_bfs_level");
      unsigned long long hn = 0;
      DCK(cudaMemcpyAsync(&hn, lc + kB, sizeof(hn), cudaMemcpyDeviceToHost, st), "copy");
      DCK(cudaStreamSynchronize(st), "sync");
      if (hn == 0) return PG_OK;
      k_carry<<<1, 1, 0, st>>>(lc, kB);
    }
  };
  k_seed<<<1, 1, 0, st>>>(0, dist, fa, lc);
  if ((rc = bfs())) return rc;
  DCK(cudaMemsetAsync(cnt + 1, 0xff, sizeof(unsigned long long), st), "memset");
  k_first_unvisited<<<gridn(n, nsm), 256, 0, st>>>(n, dist, cnt + 1);
  unsigned long long first = 0;
  DCK(cudaMemcpyAsync(&first, cnt + 1, sizeof(first), cudaMemcpyDeviceToHost, st), "copy");
  DCK(cudaStreamSynchronize(st), "sync");
  if (first != ~0ull) {
    // several components: the host seeds each at its smallest node (colour 0);
    // find those by minimum-label propagation, then one multi-source BFS
    int64_t *lab = nullptr;
    int32_t *changed = nullptr;
    DAL(lab, sizeof(int64_t) * (size_t)n);
    DAL(changed, sizeof(int32_t));
    k_lab_init<<<gridn(n, nsm), 256, 0, st>>>(n, lab);
    for (int32_t hc = 1; hc;) {
      DCK(cudaMemsetAsync(changed, 0, sizeof(int32_t), st), "memset");
      k_lab_hook<<<gridn(n, nsm), 256, 0, st>>>(n, ptr, adj, lab, changed);
      for (int k = 0; k < 4; ++k) k_lab_jump<<<gridn(n, nsm), 256, 0, st>>>(n, lab);
      DCK(cudaGetLastError(), "labels");
      DCK(cudaMemcpyAsync(&hc, changed, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
      DCK(cudaStreamSynchronize(st), "sync");
    }
    DCK(cudaMemsetAsync(lc, 0, sizeof(unsigned long long), st), "memset");
    k_seed_all<<<gridn(n, nsm), 256, 0, st>>>(n, lab, dist, fa, lc);
    DCK(cudaGetLastError(), "k_seed_all");
    if ((rc = bfs())) return rc;
  }
  int64_t *black = deg, *sblack = nullptr;  // deg is free now
  int32_t *conflict = nullptr;
  DAL(sblack, sizeof(int64_t) * (size_t)(n + 1));
  DAL(conflict, sizeof(int32_t));
  DCK(cudaMemsetAsync(conflict, 0, sizeof(int32_t), st), "memset");
  k_colour_check<<<gridn(n, nsm), 256, 0, st>>>(n, ptr, adj, dist, black, conflict);
  DCK(cudaGetLastError(), "k_colour_check");
  DCK(cudaMemsetAsync(black + n, 0, sizeof(int64_t), st), "memset");
  tb = cub_bytes;
  DCK(cub::DeviceScan::ExclusiveSum(cubtmp, tb, black, sblack, n + 1, st), "scan");
  int32_t hconf = 0;
  int64_t n_black = 0;
  DCK(cudaMemcpyAsync(&hconf, conflict, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
  DCK(cudaMemcpyAsync(&n_black, sblack + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "copy");
  DCK(cudaStreamSynchronize(st), "sync");
  if (hconf) return PG_OK;  // not bipartite: the host's greedy colouring
  const int64_t n_red = n - n_black;
  // the store (library allocations, kept by the grid)
  if ((rc = dalloc_bytes((void **)&g->rowptr, sizeof(int32_t) * (size_t)(n + 1 + 8))) ||
      (rc = dalloc_bytes((void **)&g->col, sizeof(int32_t) * (size_t)(nnz + 8))) ||
      (rc = dalloc_bytes((void **)&g->val, sizeof(double) * (size_t)(nnz + 8))) ||
      (rc = dalloc_bytes((void **)&g->perm, sizeof(int64_t) * (size_t)n)) ||
      (rc = dalloc_bytes((void **)&g->iperm, sizeof(int64_t) * (size_t)n)) ||
      (rc = dalloc_bytes((void **)&g->cap, sizeof(double) * (size_t)n))) {
    err = "out of device memory for the CSR store";
    return rc;
  }
  int64_t *len_p = nullptr, *rp = nullptr;
  DAL(len_p, sizeof(int64_t) * (size_t)(n + 1));
  DAL(rp, sizeof(int64_t) * (size_t)(n + 1));
  DCK(cudaMemsetAsync(len_p + n, 0, sizeof(int64_t), st), "memset");
  k_perm<<<gridn(n, nsm), 256, 0, st>>>(n, black, sblack, n_red, g->perm, g->iperm, ptr, len_p, cap, g->cap);
  DCK(cudaGetLastError(), "k_perm");
  tb = cub_bytes;
  DCK(cub::DeviceScan::ExclusiveSum(cubtmp, tb, len_p, rp, n + 1, st), "scan");
  k_rows<<<gridn(n, nsm), 256, 0, st>>>(n, g->perm, g->iperm, ptr, adj, w, rp, g->rowptr, g->col, g->val);
  DCK(cudaGetLastError(), "k_rows");
  k_slack<<<1, 32, 0, st>>>(n, nnz, g->rowptr, g->col, g->val);
  DCK(cudaGetLastError(), "k_slack");
  g->color_ptr = {0, n_red, n};
  g->ncolor = 2;
  int32_t *too_big = conflict;
  DCK(cudaMemsetAsync(too_big, 0, sizeof(int32_t), st), "memset");
  for (int c = 0; c < 2; ++c)
    if (g->color_ptr[c + 1] > g->color_ptr[c])
      k_tile_fit<<<gridn((g->color_ptr[c + 1] - g->color_ptr[c]) / kCsrR + 1, nsm), 256, 0, st>>>(
          g->color_ptr[c], g->color_ptr[c + 1], g->rowptr, too_big);
  int32_t htb = 0;
  DCK(cudaMemcpyAsync(&htb, too_big, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
  DCK(cudaStreamSynchronize(st), "sync");
  g->csr_staged_ok = htb == 0;
  *done = true;
  return PG_OK;
#undef DCK
#undef DAL
}

}  // namespace pgb
