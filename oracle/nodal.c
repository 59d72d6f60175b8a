/*
 * oracle/nodal.c -- TEST INFRASTRUCTURE ORACLE (see oracle/__init__.py).
 *
 * Plain, slow, sequential C implementation of the paper's topology-based
 * transient analysis (§IV "Topology-based Transient Analysis of Power
 * Grid"): the per-node update Eq. (12)-(13), the SOR variant Eq. (15)
 * ("Algorithm 2"), and the time loop of Algorithm 1.  fp64 throughout.  No
 * blocking, no reordering beyond the node visiting order the caller passes
 * (Eq. (13) defines L_i / U_i by that order).  Shares no code with the CUDA
 * product path.
 *
 * Endpoint encoding: j >= 0 trivial node, j == -1 ground, j <= -2 source node
 * (-j-2) held at vd[-j-2].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Per-node branch lists N_i of Eq. (12) from a branch list a[k] -> b[k]:
 * every branch appears in the list of each trivial endpoint (a >= 0, b >= 0).
 * Inside a node's list the entries are the a-ends in branch order, then the
 * b-ends in branch order (a stable counting sort of the concatenated end
 * list).  ptr[n+1] (caller-zeroed), nbr/val[2m upper bound]; br/sgn may be NULL.
 * Plain two-pass counting sort: count degrees, prefix-sum, fill.             */
void oracle_group(int64_t n, int64_t m, const int64_t *a, const int64_t *b, const double *val,
                  int64_t *ptr, int64_t *nbr, double *vout, int64_t *br, double *sgn) {
  for (int64_t k = 0; k < m; ++k) {
    if (a[k] >= 0) ptr[a[k] + 1] += 1;
    if (b[k] >= 0) ptr[b[k] + 1] += 1;
  }
  for (int64_t i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  memcpy(fill, ptr, sizeof(int64_t) * (size_t)n);
  for (int pass = 0; pass < 2; ++pass)
    for (int64_t k = 0; k < m; ++k) {
      const int64_t i = pass == 0 ? a[k] : b[k], j = pass == 0 ? b[k] : a[k];
      if (i < 0) continue;
      const int64_t q = fill[i]++;
      nbr[q] = j;
      vout[q] = val[k];
      if (br) br[q] = k;
      if (sgn) sgn[q] = pass == 0 ? 1.0 : -1.0;
    }
  free(fill);
}

static double v_of(int64_t j, const double *V, const double *vd) {
  if (j >= 0) return V[j];
  if (j == -1) return 0.0;
  return vd[-j - 2];
}

/* Companion conductance of an inductor branch over one backward-Euler step:
 * h/L (Eq. (14)); with a series resistance R (series R-L element, DESIGN.md
 * R7) backward Euler of R i + L di/dt = v gives i(t+h) = v(t+h)/(R + L/h) +
 * (L/h)/(R + L/h) i(t), i.e. conductance h/(L + R h) and history factor
 * L/(L + R h).  R = 0 reproduces h/L and 1 exactly.                           */
static double l_cond(double L, double R, double h) { return h / (L + R * h); }
static double l_hist(double L, double R, double h) { return L / (L + R * h); }

/* Diagonal coefficient of V_i(t+h) in Eq. (14):
 *   d_i = sum_{j in N_i^R} g_ij + h * sum_{j in N_i^L} 1/L_ij + C_i/h          */
void oracle_diag(int64_t n, const int64_t *rptr, const double *rg,
                 const int64_t *lptr, const double *lval, const double *lres,
                 const double *cap, double h, double *d) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t k = rptr[i]; k < rptr[i + 1]; ++k) s += rg[k];
    for (int64_t k = lptr[i]; k < lptr[i + 1]; ++k) s += l_cond(lval[k], lres[k], h);
    s += cap[i] / h;
    d[i] = s;
  }
}

/* Known part of the update (everything but the trivial-neighbour sums),
 * companion / undifferenced form: backward Euler applied to the KCL Eq. (12)
 * at t+h with the inductor branch currents carried as state (Eq. (10)):
 *   d_i K_i = sum_{R fixed j} g_ij V_j + sum_{L fixed j} (h/L_ij) V_j
 *             - sum_{L branches b at i} s_ib I_b(t) - I_i(t+h) + (C_i/h) V_i(t)
 * (s_ib = +1 when the branch current b leaves node i).                        */
void oracle_known_companion(int64_t n, const int64_t *rptr, const int64_t *rnbr,
                            const double *rg, const int64_t *lptr, const int64_t *lnbr,
                            const double *lval, const double *lres, const int64_t *lbr,
                            const double *lsgn, const double *cap, const double *vd, double h,
                            const double *Vt, const double *Iload_tph,
                            const double *il_t, double *known) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t k = rptr[i]; k < rptr[i + 1]; ++k)
      if (rnbr[k] < 0) s += rg[k] * v_of(rnbr[k], Vt, vd);
    for (int64_t k = lptr[i]; k < lptr[i + 1]; ++k) {
      if (lnbr[k] < 0) s += l_cond(lval[k], lres[k], h) * v_of(lnbr[k], Vt, vd);
      s -= lsgn[k] * (l_hist(lval[k], lres[k], h) * il_t[lbr[k]]);
    }
    s -= Iload_tph[i];
    s += (cap[i] / h) * Vt[i];
    known[i] = s;
  }
}

/* Known part, the paper's second-order form Eq. (14):
 *   d_i K_i = sum_{R fixed} g V_j(t+h) + sum_{L fixed} (h/L) V_j(t+h)
 *           + (2C_i/h + sum_R g_ij) V_i(t) - sum_R g_ij V_j(t)
 *           - I_i(t+h) + I_i(t) - (C_i/h) V_i(t-h)                              */
void oracle_known_second_order(int64_t n, const int64_t *rptr, const int64_t *rnbr,
                               const double *rg, const int64_t *lptr, const int64_t *lnbr,
                               const double *lval, const double *cap, const double *vd,
                               double h, const double *Vt, const double *Vtmh,
                               const double *Iload_tph, const double *Iload_t,
                               double *known) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0, gsum = 0.0;
    for (int64_t k = rptr[i]; k < rptr[i + 1]; ++k) {
      int64_t j = rnbr[k];
      if (j < 0) s += rg[k] * v_of(j, Vt, vd); /* fixed: V_j(t+h) = V_j(t) */
      gsum += rg[k];
      s -= rg[k] * v_of(j, Vt, vd);
    }
    for (int64_t k = lptr[i]; k < lptr[i + 1]; ++k)
      if (lnbr[k] < 0) s += (h / lval[k]) * v_of(lnbr[k], Vt, vd);
    s += (2.0 * cap[i] / h + gsum) * Vt[i];
    s -= Iload_tph[i];
    s += Iload_t[i];
    s -= (cap[i] / h) * Vtmh[i];
    known[i] = s;
  }
}

/* One Gauss-Seidel sweep of Eq. (13), with SOR Eq. (15) when omega != 1, over
 * the nodes in the order `order` (nodes earlier in the order are L_i and use
 * V^(k); later ones are U_i and use V^(k-1) -- in-place update).  Returns
 * max_i |V_i^(k) - V_i^(k-1)|.                                                */
double oracle_sweep(int64_t n, const int64_t *order, const int64_t *rptr,
                    const int64_t *rnbr, const double *rg, const int64_t *lptr,
                    const int64_t *lnbr, const double *lval, const double *lres, double h,
                    const double *d, const double *known, double omega, double *V) {
  double dmax = 0.0;
  for (int64_t q = 0; q < n; ++q) {
    int64_t i = order ? order[q] : q;
    double s = known[i];
    for (int64_t k = rptr[i]; k < rptr[i + 1]; ++k)
      if (rnbr[k] >= 0) s += rg[k] * V[rnbr[k]];
    for (int64_t k = lptr[i]; k < lptr[i + 1]; ++k)
      if (lnbr[k] >= 0) s += l_cond(lval[k], lres[k], h) * V[lnbr[k]];
    double vt = s / d[i];
    double vn = omega * vt + (1.0 - omega) * V[i];
    double dv = fabs(vn - V[i]);
    if (dv > dmax) dmax = dv;
    V[i] = vn;
  }
  return dmax;
}

/* One (weighted) Jacobi sweep: every node from the previous iterate. */
double oracle_jacobi(int64_t n, const int64_t *rptr, const int64_t *rnbr,
                     const double *rg, const int64_t *lptr, const int64_t *lnbr,
                     const double *lval, const double *lres, double h, const double *d,
                     const double *known, double omega, const double *Vold,
                     double *Vnew) {
  double dmax = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double s = known[i];
    for (int64_t k = rptr[i]; k < rptr[i + 1]; ++k)
      if (rnbr[k] >= 0) s += rg[k] * Vold[rnbr[k]];
    for (int64_t k = lptr[i]; k < lptr[i + 1]; ++k)
      if (lnbr[k] >= 0) s += l_cond(lval[k], lres[k], h) * Vold[lnbr[k]];
    double vt = s / d[i];
    double vn = omega * vt + (1.0 - omega) * Vold[i];
    double dv = fabs(vn - Vold[i]);
    if (dv > dmax) dmax = dv;
    Vnew[i] = vn;
  }
  return dmax;
}

/* Companion state update after a converged step (Eq. (10), second line):
 *   I_b(t+h) = I_b(t) + (h/L_b) (V_a(t+h) - V_c(t+h))   for branch b = a -> c
 * (series R-L element: I_b(t+h) = l_hist I_b(t) + l_cond (V_a - V_c)).       */
void oracle_inductor_update(int64_t nl, const int64_t *la, const int64_t *lb,
                            const double *lv, const double *lr, const double *vd, double h,
                            const double *V, double *il) {
  for (int64_t b = 0; b < nl; ++b)
    il[b] = l_hist(lv[b], lr[b], h) * il[b] +
            l_cond(lv[b], lr[b], h) * (v_of(la[b], V, vd) - v_of(lb[b], V, vd));
}

/* Algorithm 1 (method 0: Gauss-Seidel/SOR in `order`; method 1: Jacobi).
 * form 0: companion / Eq. (2) for RC (steps s = 1..steps from V(0), il(0));
 * form 1: second-order Eq. (14) (steps s = 2..steps from V(0), V(1)).
 * Iload: [(steps+1) * n] per-node load currents I_i(s h).
 * Vout:  [(steps+1) * n] nodal voltages V(s) (V(0) [and V(1)] copied in).
 * sweeps_out[s]: inner iterations k taken at step s.
 * dtrace (nullable, [(steps+1) * 6], Gauss-Seidel/SOR only): the stopping
 *   record of step s -- ||V^(k-1) - V^(k-2)|| (NAN if k = 1), ||V^(k) -
 *   V^(k-1)||, then the norms of 4 further sweeps continued on a scratch copy
 *   of V^(k) (diagnostic only: V(s) stays V^(k)).  The GPU tests its stopping
 *   criterion every F sweeps (R13); these let a test compute the
 *   sweep at which that criterion first holds.
 * check_every: Algorithm 1 line 8 is evaluated after every sweep (1, the
 *   paper) or only after sweeps k that are multiples of check_every (DESIGN.md
 *   R13: the GPU tests once per launch of F fused sweeps).
 * Returns 0, or -(s) if step s hit max_sweeps without meeting tol.          */
int64_t oracle_transient(int64_t n, const int64_t *order, const int64_t *rptr,
                         const int64_t *rnbr, const double *rg, const int64_t *lptr,
                         const int64_t *lnbr, const double *lval, const double *lres,
                         const int64_t *lbr, const double *lsgn, const double *cap, int64_t nind,
                         const int64_t *la, const int64_t *lb, const double *lv, const double *lr,
                         const double *vd, int form, int method, double h,
                         int64_t steps, double tol, double omega, int64_t max_sweeps,
                         const double *Iload, const double *V0, const double *V1,
                         double *il, double *Vout, int64_t *sweeps_out, double *dtrace,
                         int64_t check_every) {
  double *d = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double *known = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double *tmp = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int64_t status = 0;
  oracle_diag(n, rptr, rg, lptr, lval, lres, cap, h, d);
  memcpy(Vout, V0, sizeof(double) * (size_t)n);
  int64_t s0 = 1;
  sweeps_out[0] = 0;
  if (form == 1) {
    memcpy(Vout + n, V1, sizeof(double) * (size_t)n);
    sweeps_out[1] = 0;
    s0 = 2;
  }
  for (int64_t s = s0; s <= steps; ++s) {
    const double *Vt = Vout + (s - 1) * n;
    double *Vs = Vout + s * n;
    if (form == 0)
      oracle_known_companion(n, rptr, rnbr, rg, lptr, lnbr, lval, lres, lbr, lsgn, cap, vd, h,
                             Vt, Iload + s * n, il, known);
    else
      oracle_known_second_order(n, rptr, rnbr, rg, lptr, lnbr, lval, cap, vd, h, Vt,
                                Vout + (s - 2) * n, Iload + s * n, Iload + (s - 1) * n,
                                known);
    memcpy(Vs, Vt, sizeof(double) * (size_t)n); /* Algorithm 1 line 3: V^(0)(s) = V(s-1) */
    int64_t k = 0;
    double dmax = NAN, dprev = NAN;
    do {
      ++k;
      dprev = dmax;
      if (method == 0) {
        dmax = oracle_sweep(n, order, rptr, rnbr, rg, lptr, lnbr, lval, lres, h, d, known, omega, Vs);
      } else {
        dmax = oracle_jacobi(n, rptr, rnbr, rg, lptr, lnbr, lval, lres, h, d, known, omega, Vs, tmp);
        memcpy(Vs, tmp, sizeof(double) * (size_t)n);
      }
    } while (!(k % check_every == 0 && dmax < tol) && k < max_sweeps); /* line 8: until ||V^(k) - V^(k-1)|| < tol */
    sweeps_out[s] = k;
    if (dtrace) {
      double *r = dtrace + s * 6;
      r[0] = dprev;
      r[1] = dmax;
      for (int e = 2; e < 6; ++e) r[e] = NAN;
      if (method == 0) {
        memcpy(tmp, Vs, sizeof(double) * (size_t)n);
        for (int e = 2; e < 6; ++e)
          r[e] = oracle_sweep(n, order, rptr, rnbr, rg, lptr, lnbr, lval, lres, h, d, known, omega, tmp);
      }
    }
    if (!(dmax < tol) && status == 0) status = -s;
    if (form == 0 && nind > 0) oracle_inductor_update(nind, la, lb, lv, lr, vd, h, Vs, il);
  }
  free(d);
  free(known);
  free(tmp);
  return status;
}
