// Host-side construction of the colour-permuted CSR store for irregular grids.
//
// Eq. (13) sweeps the nodes in index order; a colouring in which no two
// adjacent nodes share a colour makes every colour class independent, so the
// nodes of one class can be updated concurrently and the sweep equals the
// sequential Gauss-Seidel sweep in the numbering "colour by colour, natural
// order inside a colour".  Bipartite grids (meshes with deleted segments) get
// the 2-colouring by BFS parity (the red-black numbering); other graphs a
// first-fit greedy colouring.
#include <algorithm>
#include <cmath>
#include <queue>
#include <string>
#include <vector>

#include "pg_internal.h"

namespace pgb {

int build_csr(int64_t n, int64_t m, const int64_t *bu, const int64_t *bv, const double *bg,
              CsrHost &out, std::string &err) {
  std::vector<int64_t> deg((size_t)n + 1, 0);
  for (int64_t k = 0; k < m; ++k) {
    if (bu[k] < 0 || bu[k] >= n || bv[k] < 0 || bv[k] >= n) {
      err = "branch endpoint out of range at branch " + std::to_string(k);
      return -1;
    }
    if (!(bg[k] >= 0.0) || !std::isfinite(bg[k])) {
      err = "branch conductance must be finite and >= 0 at branch " + std::to_string(k);
      return -1;
    }
    if (bu[k] == bv[k] || bg[k] == 0.0) continue;  // self-loop / open branch: no current
    ++deg[bu[k] + 1];
    ++deg[bv[k] + 1];
  }
  std::vector<int64_t> ptr((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + deg[i + 1];
  std::vector<int64_t> adj((size_t)ptr[n]);
  std::vector<double> w((size_t)ptr[n]);
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  for (int64_t k = 0; k < m; ++k) {
    if (bu[k] == bv[k] || bg[k] == 0.0) continue;
    adj[fill[bu[k]]] = bv[k];
    w[fill[bu[k]]++] = bg[k];
    adj[fill[bv[k]]] = bu[k];
    w[fill[bv[k]]++] = bg[k];
  }
  // --- colouring: BFS parity per component; greedy if not bipartite
  std::vector<int32_t> color((size_t)n, -1);
  bool bipartite = true;
  for (int64_t s = 0; s < n && bipartite; ++s) {
    if (color[s] >= 0) continue;
    color[s] = 0;
    std::queue<int64_t> q;
    q.push(s);
    while (!q.empty() && bipartite) {
      const int64_t i = q.front();
      q.pop();
      for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
        const int64_t j = adj[k];
        if (color[j] < 0) {
          color[j] = color[i] ^ 1;
          q.push(j);
        } else if (color[j] == color[i]) {
          bipartite = false;
          break;
        }
      }
    }
  }
  int32_t ncolor = 2;
  if (!bipartite) {
    std::fill(color.begin(), color.end(), -1);
    ncolor = 1;
    std::vector<int64_t> mark;
    for (int64_t i = 0; i < n; ++i) {
      mark.assign((size_t)ncolor + 1, -1);
      for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
        const int32_t c = color[adj[k]];
        if (c >= 0 && c <= ncolor) mark[c] = i;
      }
      int32_t c = 0;
      while (mark[c] == i) ++c;
      color[i] = c;
      ncolor = std::max(ncolor, c + 1);
    }
  }
  // --- permutation: colour-major, natural order inside a colour
  out.color_ptr.assign((size_t)ncolor + 1, 0);
  for (int64_t i = 0; i < n; ++i) ++out.color_ptr[color[i] + 1];
  for (int32_t c = 0; c < ncolor; ++c) out.color_ptr[c + 1] += out.color_ptr[c];
  out.perm.assign((size_t)n, 0);
  out.iperm.assign((size_t)n, 0);
  std::vector<int64_t> pos(out.color_ptr.begin(), out.color_ptr.end() - 1);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t p = pos[color[i]]++;
    out.perm[p] = i;
    out.iperm[i] = p;
  }
  out.rowptr.assign((size_t)n + 1, 0);
  for (int64_t p = 0; p < n; ++p) {
    const int64_t i = out.perm[p];
    out.rowptr[p + 1] = out.rowptr[p] + (ptr[i + 1] - ptr[i]);
  }
  out.col.resize((size_t)ptr[n]);
  out.val.resize((size_t)ptr[n]);
  for (int64_t p = 0; p < n; ++p) {
    const int64_t i = out.perm[p];
    int64_t o = out.rowptr[p];
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k, ++o) {
      out.col[o] = (int32_t)out.iperm[adj[k]];
      out.val[o] = w[k];
    }
  }
  return 0;
}

}  // namespace pgb
