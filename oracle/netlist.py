"""Circuit model in the paper's notation (§III "System equation").

* trivial nodes 1..n (here 0..n-1): "nodes that are neither ground nor positive
  terminals of voltage sources";
* source nodes 1..p with constant voltages v_d (negative terminals at ground,
  topological assumption 1, §III-B);
* m branches not through voltage sources, grouped as resistors (g), capacitors
  (c), inductors (l) and current sources (i) - Eq. (6).

Endpoint encoding used throughout the oracle: ``j >= 0`` trivial node j,
``j == GROUND (-1)`` ground, ``j <= -2`` source node ``-j-2``.

A "series R-L" element (pads and vias of the RLC grid, reading R7) is modelled
by default exactly as the paper models inductors: an R branch and an L branch
joined at an extra trivial node with no capacitance (the paper's Fig. 2 node
model).  ``from_mesh(g, series_rl="element")`` instead keeps it as ONE inductor
branch with a series resistance ``lr`` (backward Euler of R i + L di/dt = v,
Eq. (8)'s inductor law with the resistor's voltage added; R7) -- the
exact elimination of that internal node, pinned equal to it in
tests/test_oracle_pins.py.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GROUND = -1


def src(k: int) -> int:
    """Encoding of source node k."""
    return -(k + 2)


@dataclass
class Netlist:
    n: int                      # trivial nodes
    vd: np.ndarray              # [p] source-node voltages (V)
    # resistor branches: a -> b, conductance g (the paper's 𝒢 holds conductances)
    ra: np.ndarray
    rb: np.ndarray
    rg: np.ndarray
    # capacitor branches a -> b, capacitance (F)
    ca: np.ndarray
    cb: np.ndarray
    cv: np.ndarray
    # inductor branches a -> b, inductance (H)
    la: np.ndarray
    lb: np.ndarray
    lv: np.ndarray
    # current-source branches a -> b (current flows a -> b through the source)
    ia: np.ndarray
    ib: np.ndarray
    # PWL waveform of current source k: t[ptr[k]:ptr[k+1]], i[...]
    iptr: np.ndarray
    it: np.ndarray
    ii: np.ndarray
    n_mesh: int = 0             # first n_mesh trivial nodes are the grid's nodes
    # series resistance (ohm) of each inductor branch (series R-L element); None = all 0
    lr: np.ndarray = None

    def __post_init__(self):
        if self.lr is None:
            self.lr = np.zeros(self.la.shape[0])

    @property
    def p(self) -> int:
        return int(self.vd.shape[0])

    @property
    def m(self) -> int:
        return int(self.ra.size + self.ca.size + self.la.size + self.ia.size)


def _i64(x):
    return np.asarray(x, dtype=np.int64)


def _f64(x):
    return np.asarray(x, dtype=np.float64)


def from_mesh(g, series_rl: str = "node") -> Netlist:
    """Netlist of a ``gridgen.MeshGrid`` (RC or RLC).  ``series_rl``: "node"
    (R branch + L branch through an internal node, the paper's element-wise
    model) or "element" (one inductor branch with series resistance)."""
    if series_rl not in ("node", "element"):
        raise ValueError("series_rl must be 'node' or 'element'")
    elem = series_rl == "element"
    lrs = []
    from gridgen import mesh_to_edges
    n = g.n
    eu, ev, eg = mesh_to_edges(g)
    is_via = (ev - eu) == g.ny * g.nx
    ra, rb, rg = [], [], []
    la, lb, lv = [], [], []
    nxt = n
    keep = eg > 0
    if g.lz is not None:
        lzf = g.lz.reshape(-1)
        via_l = lzf[eu]
        plain = keep & (~is_via | (via_l <= 0))
        ra.append(eu[plain]); rb.append(ev[plain]); rg.append(eg[plain])
        rl = keep & is_via & (via_l > 0)
        u, v, gg, ll = eu[rl], ev[rl], eg[rl], via_l[rl]
        if elem:
            la.append(u); lb.append(v); lv.append(ll); lrs.append(1.0 / gg)   # u -(R+L)- v
        else:
            mid = np.arange(nxt, nxt + u.size, dtype=np.int64)
            nxt += u.size
            ra.append(u); rb.append(mid); rg.append(gg)       # u -R- mid
            la.append(mid); lb.append(v); lv.append(ll)       # mid -L- v
            lrs.append(np.zeros(u.size))
    else:
        ra.append(eu[keep]); rb.append(ev[keep]); rg.append(eg[keep])
    # pads to the single Vdd source node (source node 0)
    pn = _i64(g.pad_node)
    if g.pad_l is not None:
        to_vdd = np.full(pn.size, src(0), dtype=np.int64)
        if elem:
            la.append(pn); lb.append(to_vdd); lv.append(_f64(g.pad_l)); lrs.append(1.0 / _f64(g.pad_g))
        else:
            mid = np.arange(nxt, nxt + pn.size, dtype=np.int64)
            nxt += pn.size
            ra.append(pn); rb.append(mid); rg.append(_f64(g.pad_g))
            la.append(mid); lb.append(to_vdd); lv.append(_f64(g.pad_l))
            lrs.append(np.zeros(pn.size))
    else:
        ra.append(pn); rb.append(np.full(pn.size, src(0), dtype=np.int64)); rg.append(_f64(g.pad_g))
    cap = g.cap.reshape(-1)
    s = g.sources
    return Netlist(
        n=int(nxt), vd=np.array([g.vdd], dtype=np.float64),
        ra=_i64(np.concatenate(ra)), rb=_i64(np.concatenate(rb)), rg=_f64(np.concatenate(rg)),
        ca=np.arange(n, dtype=np.int64), cb=np.full(n, GROUND, dtype=np.int64), cv=_f64(cap).copy(),
        la=_i64(np.concatenate(la)) if la else np.zeros(0, np.int64),
        lb=_i64(np.concatenate(lb)) if lb else np.zeros(0, np.int64),
        lv=_f64(np.concatenate(lv)) if lv else np.zeros(0),
        ia=_i64(s.node), ib=np.full(s.count, GROUND, dtype=np.int64),
        iptr=_i64(s.ptr), it=_f64(s.t), ii=_f64(s.i), n_mesh=n,
        lr=_f64(np.concatenate(lrs)) if lrs else None)


def from_edges(g) -> Netlist:
    """Netlist of a ``gridgen.EdgeGrid`` (irregular RC grid)."""
    n = g.n
    pn = _i64(g.pad_node)
    s = g.sources
    keep = g.eg > 0
    return Netlist(
        n=n, vd=np.array([g.vdd], dtype=np.float64),
        ra=_i64(np.concatenate([g.eu[keep], pn])),
        rb=_i64(np.concatenate([g.ev[keep], np.full(pn.size, src(0), dtype=np.int64)])),
        rg=_f64(np.concatenate([g.eg[keep], g.pad_g])),
        ca=np.arange(n, dtype=np.int64), cb=np.full(n, GROUND, dtype=np.int64), cv=_f64(g.cap).copy(),
        la=np.zeros(0, np.int64), lb=np.zeros(0, np.int64), lv=np.zeros(0),
        ia=_i64(s.node), ib=np.full(s.count, GROUND, dtype=np.int64),
        iptr=_i64(s.ptr), it=_f64(s.t), ii=_f64(s.i), n_mesh=n)


def from_grid(g, series_rl: str = "node") -> Netlist:
    return from_edges(g) if hasattr(g, "eu") else from_mesh(g, series_rl)


@dataclass
class NodeLists:
    """Per-trivial-node neighbour sets of Eq. (12): N_i^R with g_ij, N_i^L with
    L_ij (and the inductor branch id + orientation for the companion current),
    and the node-to-ground capacitance C_i.  CSR-style arrays."""
    rptr: np.ndarray
    rnbr: np.ndarray
    rg: np.ndarray
    lptr: np.ndarray
    lnbr: np.ndarray
    lval: np.ndarray
    lbr: np.ndarray       # inductor branch index
    lsgn: np.ndarray      # +1 if node i is the branch's a-end (current a->b leaves i), -1 else
    cap: np.ndarray       # C_i (ground capacitors only; assumption of Eq. (12))
    lres: np.ndarray = None  # series resistance of the inductor branch (0: pure inductor)


def _group_numpy(n, a, b, val):
    """Reference grouping (stable argsort of the concatenated end list); the
    oracle uses the equivalent plain-C counting sort ``oracle_group`` (memory:
    full-size grids), checked equal to this in tests/test_oracle_pins.py."""
    ends_i, ends_j, vals, br, sg = [], [], [], [], []
    idx = np.arange(a.size, dtype=np.int64)
    m = a >= 0
    ends_i.append(a[m]); ends_j.append(b[m]); vals.append(val[m]); br.append(idx[m]); sg.append(np.ones(m.sum()))
    m = b >= 0
    ends_i.append(b[m]); ends_j.append(a[m]); vals.append(val[m]); br.append(idx[m]); sg.append(-np.ones(m.sum()))
    ei = np.concatenate(ends_i); ej = np.concatenate(ends_j); ev = np.concatenate(vals)
    eb = np.concatenate(br); es = np.concatenate(sg)
    o = np.argsort(ei, kind="stable")
    ei, ej, ev, eb, es = ei[o], ej[o], ev[o], eb[o], es[o]
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(ptr, ei + 1, 1)
    ptr = np.cumsum(ptr)
    return ptr, ej.astype(np.int64), ev.astype(np.float64), eb.astype(np.int64), es.astype(np.float64)


def group(n, a, b, val, with_branch=True):
    """Each branch a[k] -> b[k] appears in the list of each trivial endpoint:
    (ptr, nbr, val, branch, sign), entries of node i in ptr[i]:ptr[i+1] (a-ends
    in branch order, then b-ends).  Plain-C counting sort (nodal.c)."""
    import ctypes
    from . import nodal
    a = np.ascontiguousarray(a, dtype=np.int64)
    b = np.ascontiguousarray(b, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    cnt = int(np.count_nonzero(a >= 0)) + int(np.count_nonzero(b >= 0))
    ptr = np.zeros(n + 1, dtype=np.int64)
    nbr = np.empty(cnt, dtype=np.int64)
    vo = np.empty(cnt, dtype=np.float64)
    br = np.empty(cnt, dtype=np.int64) if with_branch else None
    sg = np.empty(cnt, dtype=np.float64) if with_branch else None
    P64, PD = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)
    nodal.lib().oracle_group(ctypes.c_int64(n), ctypes.c_int64(a.size), a.ctypes.data_as(P64),
                             b.ctypes.data_as(P64), val.ctypes.data_as(PD), ptr.ctypes.data_as(P64),
                             nbr.ctypes.data_as(P64), vo.ctypes.data_as(PD),
                             br.ctypes.data_as(P64) if with_branch else None,
                             sg.ctypes.data_as(PD) if with_branch else None)
    return ptr, nbr, vo, br, sg


def node_lists(nl: Netlist) -> NodeLists:
    """Build N_i^R, N_i^L, C_i of Eq. (12) from the branch list."""
    n = nl.n
    rptr, rnbr, rg, _, _ = group(n, nl.ra, nl.rb, nl.rg, with_branch=False)
    lptr, lnbr, lval, lbr, lsgn = group(n, nl.la, nl.lb, nl.lv)
    lres = np.asarray(nl.lr, dtype=np.float64)[lbr] if lbr.size else np.zeros(0)
    cap = np.zeros(n)
    if np.any((nl.ca >= 0) & (nl.cb >= 0)) or np.any(nl.cb < -1) or np.any(nl.ca < 0):
        raise ValueError("nodal oracle supports node-to-ground capacitors only (Eq. (12))")
    np.add.at(cap, nl.ca, nl.cv)
    return NodeLists(rptr, rnbr, rg, lptr, lnbr, lval, lbr, lsgn, cap, lres)
