"""Piecewise-linear current sources (§II-A: "the current pattern of the
gates and devices should be obtained and modeled as piecewise linear ideal
current sources").  Linear interpolation between breakpoints, first/last value
held outside them (reading R8)."""
from __future__ import annotations

import numpy as np


def eval_source(t_pts: np.ndarray, i_pts: np.ndarray, t: float) -> float:
    """Value of one PWL waveform at time t (np.interp holds the end values)."""
    return float(np.interp(t, t_pts, i_pts))


def node_currents(nl, t: float) -> np.ndarray:
    """I_i(t): total load current drawn from each trivial node at time t
    (the vector i(t) of Eq. (1); A_i^T I_s(t) of Eq. (9) for ground-terminated
    sources)."""
    out = np.zeros(nl.n)
    for k in range(nl.ia.size):
        a, b = int(nl.ia[k]), int(nl.ib[k])
        s, e = int(nl.iptr[k]), int(nl.iptr[k + 1])
        v = eval_source(nl.it[s:e], nl.ii[s:e], t)
        if a >= 0:
            out[a] += v
        if b >= 0:
            out[b] -= v
    return out


def node_currents_table(nl, h: float, steps: int) -> np.ndarray:
    """[steps+1, n] table of I_i(s*h), s = 0..steps."""
    tab = np.zeros((steps + 1, nl.n))
    for s in range(steps + 1):
        tab[s] = node_currents_at(nl, s * h)
    return tab


def node_currents_at(nl, t: float) -> np.ndarray:
    """I_i(t) for every trivial node (as ``node_currents``), vectorised over
    sources with the same breakpoint count; falls back to the loop otherwise."""
    out = np.zeros(nl.n)
    if nl.ia.size == 0:
        return out
    cnt = np.diff(nl.iptr)
    if not np.all(cnt == cnt[0]):
        return node_currents(nl, t)
    k = int(cnt[0])
    T = nl.it.reshape(-1, k)
    I = nl.ii.reshape(-1, k)
    v = _interp_rows(T, I, t)
    na = nl.ia >= 0
    np.add.at(out, nl.ia[na], v[na])
    nb = nl.ib >= 0
    if nb.any():
        np.add.at(out, nl.ib[nb], -v[nb])
    return out


def _interp_rows(T: np.ndarray, I: np.ndarray, t: float) -> np.ndarray:
    """Row-wise np.interp(t, T[r], I[r]) (same semantics: hold ends)."""
    k = T.shape[1]
    out = np.where(t <= T[:, 0], I[:, 0], I[:, k - 1])
    for j in range(k - 1):
        t0, t1 = T[:, j], T[:, j + 1]
        inside = (t > t0) & (t <= t1)
        if inside.any():
            w = (t - t0[inside]) / (t1[inside] - t0[inside])
            out[inside] = I[inside, j] + w * (I[inside, j + 1] - I[inside, j])
    return out
