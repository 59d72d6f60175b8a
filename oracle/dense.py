"""Dense nodal-analysis matrices and direct solves (§III, Eqs. (4)-(11))
- TEST INFRASTRUCTURE, tiny circuits only.

Sign conventions (readings R2/R3): KVL Eq. (7) ``A v_n = v_b - A_s v_d``
gives branch voltages ``v_b = A v_n + A_s v_d``; with the branch equations
Eq. (8) and KCL ``A^T i_b = 0`` the trivial-node equations are

    C dv/dt + G v + G_s v_d + A_l^T i_l + A_i^T I_s = 0,
    𝓛 di_l/dt = A_l v + A_ls v_d,

i.e. Eq. (9) with the signs of its ``G_s v_d`` and ``A_ls v_d`` terms flipped
(the paper's printed signs contradict its own Eq. (7); they agree with Eq. (1),
``b = -i + G_0 V_dd``, only this way).  Differencing the backward-Euler form
Eq. (10) gives Eq. (11) with ``h L_s v_d`` where ``L_s = -A_l^T 𝓛^{-1} A_ls``
(the paper's ``A_l 𝓛^{-1} A_ls`` is not conformable; reading R3).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .netlist import Netlist


def incidence(nl: Netlist):
    """Modified incidence A (m x n, Eq. (4)) and source incidence A_s (m x p,
    Eq. (5)), rows grouped as [g; c; l; i] (Eq. (6))."""
    n, p = nl.n, nl.p
    groups = [(nl.ra, nl.rb), (nl.ca, nl.cb), (nl.la, nl.lb), (nl.ia, nl.ib)]
    out = []
    for a, b in groups:
        m = a.size
        A = np.zeros((m, n))
        As = np.zeros((m, p))
        for k in range(m):
            for node, sign in ((int(a[k]), 1.0), (int(b[k]), -1.0)):
                if node >= 0:
                    A[k, node] = sign          # "+1 if trivial node j is the source of branch i"
                elif node <= -2:
                    As[k, -node - 2] = sign    # same for source nodes, Eq. (5)
        out.append((A, As))
    return out


def system(nl: Netlist, h: float):
    """G = A_g^T 𝒢 A_g, C = A_c^T 𝒞 A_c, L = A_l^T 𝓛^{-1} A_l, G_s = A_g^T 𝒢 A_gs,
    L_s = -A_l^T 𝓛^{-1} A_ls, and the system matrix M = C/h + G + hL (Eq. (11))."""
    if np.any(np.asarray(nl.lr) != 0):
        raise ValueError("dense solves model series R-L with internal nodes (series_rl='node')")
    (Ag, Ags), (Ac, Acs), (Al, Als), (Ai, Ais) = incidence(nl)
    G = Ag.T @ np.diag(nl.rg) @ Ag
    C = Ac.T @ np.diag(nl.cv) @ Ac
    Linv = np.diag(1.0 / nl.lv) if nl.lv.size else np.zeros((0, 0))
    L = Al.T @ Linv @ Al if nl.lv.size else np.zeros((nl.n, nl.n))
    Gs = Ag.T @ np.diag(nl.rg) @ Ags
    Ls = -(Al.T @ Linv @ Als) if nl.lv.size else np.zeros((nl.n, nl.p))
    M = C / h + G + h * L
    return dict(G=G, C=C, L=L, Gs=Gs, Ls=Ls, M=M, Al=Al, Als=Als, Ai=Ai, Ais=Ais, Linv=Linv)


def check_pd(M: np.ndarray, tol: float = 1e-12):
    """Lemma 1 checks: symmetry, weak diagonal dominance with nonnegative
    diagonal, irreducibility (connected coupling graph), and positive
    definiteness by Cholesky (all pivots > 0)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    n = M.shape[0]
    sym = bool(np.array_equal(M, M.T))
    off = np.abs(M).sum(axis=1) - np.abs(np.diag(M))
    diag = np.diag(M)
    wdd = bool(np.all(diag >= 0) and np.all(diag >= off * (1 - 1e-14)))
    strict = diag > off * (1 + 1e-14)
    adj = (np.abs(M) > 0) & ~np.eye(n, dtype=bool)
    ncomp, _ = connected_components(csr_matrix(adj), directed=False)
    try:
        c = np.linalg.cholesky(M)
        pd = bool(np.all(np.diag(c) > tol * np.max(np.abs(diag))))
    except np.linalg.LinAlgError:
        pd = False
    return dict(symmetric=sym, weakly_dd=wdd, n_strict=int(strict.sum()),
                irreducible=(ncomp == 1), n_components=int(ncomp), pd=pd)


def _chol(M):
    return sla.cho_factor(M, lower=True)


def direct_companion(nl: Netlist, h: float, steps: int, Itab: np.ndarray,
                     v0: np.ndarray, il0: np.ndarray | None = None):
    """Backward-Euler Eq. (10) solved directly (Cholesky of M) with the
    inductor currents carried as state ("companion" form):

        M v(t+h) = (C/h) v(t) - A_l^T i_l(t) + h L_s v_d - A_i^T I_s(t+h) - G_s v_d
        i_l(t+h) = i_l(t) + h 𝓛^{-1} (A_l v(t+h) + A_ls v_d)

    ``Itab[s]`` is the per-node load i(s h) (= A_i^T I_s for ground-terminated
    sources).  For an inductor-free grid this is exactly Eq. (2)."""
    S = system(nl, h)
    cf = _chol(S["M"])
    V = np.zeros((steps + 1, nl.n))
    V[0] = v0
    il = np.zeros(nl.la.size) if il0 is None else il0.copy()
    const = h * (S["Ls"] @ nl.vd) - S["Gs"] @ nl.vd
    for s in range(1, steps + 1):
        rhs = (S["C"] / h) @ V[s - 1] - S["Al"].T @ il + const - Itab[s]
        V[s] = sla.cho_solve(cf, rhs)
        if il.size:
            il = il + h * (S["Linv"] @ (S["Al"] @ V[s] + S["Als"] @ nl.vd))
    return V, il


def direct_second_order(nl: Netlist, h: float, steps: int, Itab: np.ndarray,
                        v0: np.ndarray, v1: np.ndarray):
    """Eq. (11) solved directly: the paper's second-order recurrence

        M v(t+h) = (2C/h + G) v(t) - (C/h) v(t-h) + h L_s v_d - A_i^T (I_s(t+h) - I_s(t))

    from the two initial states v(0), v(h) (Algorithm 1 line 1)."""
    S = system(nl, h)
    cf = _chol(S["M"])
    V = np.zeros((steps + 1, nl.n))
    V[0] = v0
    V[1] = v1
    A2 = 2 * S["C"] / h + S["G"]
    const = h * (S["Ls"] @ nl.vd)
    for s in range(2, steps + 1):
        rhs = A2 @ V[s - 1] - (S["C"] / h) @ V[s - 2] + const - (Itab[s] - Itab[s - 1])
        V[s] = sla.cho_solve(cf, rhs)
    return V


def dc_solve(nl: Netlist, I: np.ndarray):
    """DC operating point G v = -i - G_s v_d with inductors as shorts: solved on
    the netlist where each inductor is replaced by a large conductance is NOT
    exact, so DC here is only defined for inductor-free netlists (§II-A "In DC
    analysis, A = G")."""
    if nl.lv.size:
        raise ValueError("dc_solve: inductor-free netlists only")
    S = system(nl, 1.0)
    return np.linalg.solve(S["G"], -I - S["Gs"] @ nl.vd)
