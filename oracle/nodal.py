"""ctypes front-end of the plain-C nodal oracle (``nodal.c``) - TEST
INFRASTRUCTURE (see oracle/__init__.py).

Implements PAPER.md §IV: Eq. (12)-(13) per-node update, SOR Eq. (15),
Algorithm 1 time loop.  ``form="companion"`` is backward Euler on the KCL with
inductor currents as state (Eq. (10); identical to Eq. (2) on RC grids);
``form="second_order"`` is the paper's Eq. (14).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from .netlist import Netlist, NodeLists, node_lists
from .pwl import node_currents_table

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nodal.c")
_LIB = os.path.join(_HERE, "liboracle_nodal.so")
_lib = None

_P64 = ctypes.POINTER(ctypes.c_int64)
_PD = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile nodal.c with gcc (plain -O2, no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_transient.restype = ctypes.c_int64
        L.oracle_sweep.restype = ctypes.c_double
        L.oracle_jacobi.restype = ctypes.c_double
        _lib = L
    return _lib


def _p64(a):
    return a.ctypes.data_as(_P64)


def _pd(a):
    return a.ctypes.data_as(_PD)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _cd(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class TransientResult:
    V: np.ndarray          # [steps+1, n]
    sweeps: np.ndarray     # [steps+1]
    il: np.ndarray         # inductor currents after the last step
    status: int
    dtrace: np.ndarray = None  # [steps+1, 6] stopping record (nodal.c oracle_transient), if asked


class NodalOracle:
    """The paper's matrix-free nodal iteration over one netlist."""

    def __init__(self, nl: Netlist):
        self.nl = nl
        self.L: NodeLists = node_lists(nl)
        a = self.L
        self._rptr, self._rnbr, self._rg = _c64(a.rptr), _c64(a.rnbr), _cd(a.rg)
        self._lptr, self._lnbr, self._lval = _c64(a.lptr), _c64(a.lnbr), _cd(a.lval)
        self._lbr, self._lsgn, self._cap = _c64(a.lbr), _cd(a.lsgn), _cd(a.cap)
        self._lres = _cd(a.lres if a.lres is not None else np.zeros(a.lval.size))
        self._la, self._lb, self._lv = _c64(nl.la), _c64(nl.lb), _cd(nl.lv)
        self._lr = _cd(nl.lr)
        # a dummy valid pointer for empty arrays
        if self._lres.size == 0:
            self._lres = np.zeros(1)
        if self._lr.size == 0:
            self._lr = np.zeros(1)
        self._vd = _cd(nl.vd)

    # -- pieces ---------------------------------------------------------------
    def diag(self, h: float) -> np.ndarray:
        d = np.zeros(self.nl.n)
        lib().oracle_diag(ctypes.c_int64(self.nl.n), _p64(self._rptr), _pd(self._rg),
                          _p64(self._lptr), _pd(self._lval), _pd(self._lres), _pd(self._cap),
                          ctypes.c_double(h), _pd(d))
        return d

    def known_companion(self, h, Vt, Iload_tph, il_t=None) -> np.ndarray:
        n = self.nl.n
        out = np.zeros(n)
        il = _cd(np.zeros(self.nl.la.size) if il_t is None else il_t)
        Vt, Ip = _cd(Vt), _cd(Iload_tph)
        lib().oracle_known_companion(
            ctypes.c_int64(n), _p64(self._rptr), _p64(self._rnbr), _pd(self._rg),
            _p64(self._lptr), _p64(self._lnbr), _pd(self._lval), _pd(self._lres), _p64(self._lbr),
            _pd(self._lsgn), _pd(self._cap), _pd(self._vd), ctypes.c_double(h),
            _pd(Vt), _pd(Ip), _pd(il), _pd(out))
        return out

    def sweep(self, h, d, known, V, omega=1.0, order=None, method="gs"):
        """One sweep in place (GS/SOR) or out of place (Jacobi); returns
        (V_new, max |delta|)."""
        n = self.nl.n
        known = _cd(known)
        d = _cd(d)
        if method == "gs":
            V = _cd(V).copy()
            o = None if order is None else _c64(order)
            dm = lib().oracle_sweep(ctypes.c_int64(n), _p64(o) if o is not None else None,
                                    _p64(self._rptr), _p64(self._rnbr), _pd(self._rg),
                                    _p64(self._lptr), _p64(self._lnbr), _pd(self._lval),
                                    _pd(self._lres), ctypes.c_double(h), _pd(d), _pd(known),
                                    ctypes.c_double(omega), _pd(V))
            return V, dm
        Vo = _cd(V)
        Vn = np.zeros(n)
        dm = lib().oracle_jacobi(ctypes.c_int64(n), _p64(self._rptr), _p64(self._rnbr),
                                 _pd(self._rg), _p64(self._lptr), _p64(self._lnbr),
                                 _pd(self._lval), _pd(self._lres), ctypes.c_double(h), _pd(d), _pd(known),
                                 ctypes.c_double(omega), _pd(Vo), _pd(Vn))
        return Vn, dm

    # -- Algorithm 1 ----------------------------------------------------------
    def transient(self, h: float, steps: int, tol: float = 1e-10, omega: float = 1.0,
                  form: str = "companion", method: str = "gs", order=None,
                  Itab=None, V0=None, V1=None, il0=None, max_sweeps: int = 1_000_000,
                  trace: bool = False, check_every: int = 1):
        nl = self.nl
        n = nl.n
        if Itab is None:
            Itab = node_currents_table(nl, h, steps)
        Itab = _cd(Itab)
        assert Itab.shape == (steps + 1, n)
        if V0 is None:
            V0 = np.full(n, float(nl.vd[0]) if nl.p else 0.0)
        V0 = _cd(V0)
        f = 0 if form == "companion" else 1
        if f == 1 and np.any(nl.lr != 0):
            raise ValueError("the second-order form Eq. (14) has no series R-L element; "
                             "use series_rl='node'")
        if f == 1:
            if V1 is None:
                raise ValueError("second-order form needs V(0) and V(1) (Algorithm 1 line 1)")
            V1 = _cd(V1)
        il = _cd(np.zeros(nl.la.size) if il0 is None else il0).copy()
        Vout = np.zeros((steps + 1, n))
        sw = np.zeros(steps + 1, dtype=np.int64)
        dt = np.full((steps + 1, 6), np.nan) if trace else None
        o = None if order is None else _c64(order)
        st = lib().oracle_transient(
            ctypes.c_int64(n), _p64(o) if o is not None else None,
            _p64(self._rptr), _p64(self._rnbr), _pd(self._rg),
            _p64(self._lptr), _p64(self._lnbr), _pd(self._lval), _pd(self._lres), _p64(self._lbr),
            _pd(self._lsgn), _pd(self._cap), ctypes.c_int64(nl.la.size),
            _p64(self._la), _p64(self._lb), _pd(self._lv), _pd(self._lr), _pd(self._vd),
            ctypes.c_int(f), ctypes.c_int(0 if method == "gs" else 1),
            ctypes.c_double(h), ctypes.c_int64(steps), ctypes.c_double(tol),
            ctypes.c_double(omega), ctypes.c_int64(max_sweeps), _pd(Itab), _pd(V0),
            _pd(V1) if f == 1 else None, _pd(il), _pd(Vout), _p64(sw),
            _pd(dt) if trace else None, ctypes.c_int64(max(1, int(check_every))))
        return TransientResult(V=Vout, sweeps=sw, il=il, status=int(st), dtrace=dt)


def red_black_order(layers: int, ny: int, nx: int) -> np.ndarray:
    """Node numbering that makes Eq. (13)'s sequential sweep a red-black sweep
    on the bipartite mesh: nodes with (l+y+x) even first, then odd, each in
    natural order."""
    l, y, x = np.meshgrid(np.arange(layers), np.arange(ny), np.arange(nx), indexing="ij")
    par = ((l + y + x) & 1).reshape(-1)
    idx = np.arange(layers * ny * nx, dtype=np.int64)
    return np.concatenate([idx[par == 0], idx[par == 1]])
