"""Kirchhoff-current-law residual of one backward-Euler step - TEST
INFRASTRUCTURE (see oracle/__init__.py).

Evaluates, at every trivial node i, the sum of currents leaving it at t+h
(Eq. (12) before differentiation, discretised by backward Euler; the
KCL ``A^T i_b = 0`` of Eq. (7)):

    r_i = sum_R g_ij (V_i - V_j) + sum_L I_ij(t+h) + I_i(t+h) + C_i (V_i(t+h) - V_i(t)) / h

computed branch by branch (each branch current added to its source end and
subtracted at its sink end) - independent of the per-node stencils the nodal
iteration uses.  A converged solution has |r_i| bounded by the sweep
tolerance times the node's coupling.
"""
from __future__ import annotations

import numpy as np

from .netlist import Netlist


def _vals(V, vd, idx):
    out = np.zeros(idx.shape[0])
    t = idx >= 0
    out[t] = V[idx[t]]
    s = idx <= -2
    out[s] = vd[-idx[s] - 2]
    return out


def _scatter(r, a, b, cur):
    ma = a >= 0
    np.add.at(r, a[ma], cur[ma])
    mb = b >= 0
    np.add.at(r, b[mb], -cur[mb])


def inductor_currents_next(nl: Netlist, h: float, V_tph: np.ndarray, il_t: np.ndarray):
    """I_b(t+h) = I_b(t) + (h/L_b)(v_a - v_b)(t+h) (backward Euler, Eq. (10));
    for a series R-L element (R_b > 0) backward Euler of R i + L di/dt = v:
    I_b(t+h) = (v(t+h) + (L_b/h) I_b(t)) / (R_b + L_b/h)."""
    if nl.la.size == 0:
        return np.zeros(0)
    v = _vals(V_tph, nl.vd, nl.la) - _vals(V_tph, nl.vd, nl.lb)
    R = np.asarray(nl.lr, dtype=np.float64)
    return (v + (nl.lv / h) * il_t) / (R + nl.lv / h)


def residual(nl: Netlist, h: float, V_tph: np.ndarray, V_t: np.ndarray,
             I_tph: np.ndarray, il_t: np.ndarray | None = None) -> np.ndarray:
    """Per-node KCL residual (A) of the step t -> t+h; ``I_tph`` is the
    per-node load current i(t+h)."""
    r = np.zeros(nl.n)
    vr = _vals(V_tph, nl.vd, nl.ra) - _vals(V_tph, nl.vd, nl.rb)
    _scatter(r, nl.ra, nl.rb, nl.rg * vr)
    if nl.la.size:
        il = inductor_currents_next(nl, h, V_tph, np.zeros(nl.la.size) if il_t is None else il_t)
        _scatter(r, nl.la, nl.lb, il)
    vc_new = _vals(V_tph, nl.vd, nl.ca) - _vals(V_tph, nl.vd, nl.cb)
    vc_old = _vals(V_t, nl.vd, nl.ca) - _vals(V_t, nl.vd, nl.cb)
    _scatter(r, nl.ca, nl.cb, nl.cv * (vc_new - vc_old) / h)
    r += I_tph
    return r
