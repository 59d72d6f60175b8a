"""Seeded synthetic power-grid generators (shared INPUT module).

This module is the only code shared by the oracle (``oracle/``) and the CUDA
product path (``paper_1409_7166_b200/``).  It draws element values and topology
from seeded distributions and returns them as raw arrays.  It contains none of
the method's arithmetic: no conductance sums, no backward-Euler terms, no
companion models, no PWL evaluation.  Both sides consume the raw element values
and build their own stencils from them.

Workload recipes follow BASELINE.json ``configs`` (the paper, §II-A,
only says grids are RC/RLC meshes with PWL current loads, capacitors at the
nodes and inductors "at the vias ... and the metal layer connecting the power
grid to external power supply").  The readings taken where BASELINE.json is
ambiguous are listed in DESIGN.md §3 (R1–R12); the ones fixed here are:

* R5 pads: a top-layer node (l = L-1) is a pad iff ``x % pitch == 0`` and
  ``y % pitch == 0`` (a 2-D C4-bump lattice).
* R6 layer 0 is the bottom (device) layer that carries the current loads.
* R7 a via / pad "series R-L" is one branch of resistance R and inductance L in
  series; RC grids have L = 0.
* R8 PWL triangle: (start, 0) -> (start + width/2, peak) -> (start + width, 0),
  zero outside.

Arrays use the natural layout index = (l * ny + y) * nx + x.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "MeshGrid", "EdgeGrid", "Sources", "mesh_grid", "edge_grid", "CONFIGS",
    "config_grid", "mesh_to_edges", "scaled_config",
]


@dataclass
class Sources:
    """Piecewise-linear current loads (load convention: drawn from the node).

    ``node[k]`` is the flat node index of source k; its breakpoints are
    ``t[ptr[k]:ptr[k+1]]`` (seconds, strictly increasing) and
    ``i[ptr[k]:ptr[k+1]]`` (amperes).  Before the first / after the last
    breakpoint the first / last value is held.
    """
    node: np.ndarray      # int64 [S]
    ptr: np.ndarray       # int64 [S+1]
    t: np.ndarray         # float64 [ptr[-1]]
    i: np.ndarray         # float64 [ptr[-1]]

    @property
    def count(self) -> int:
        return int(self.node.shape[0])


@dataclass
class MeshGrid:
    """Layered rectangular mesh: ``layers`` metal layers of ny x nx nodes.

    gx[l,y,x]: conductance (S) of the segment (l,y,x)-(l,y,x+1); 0 at x = nx-1.
    gy[l,y,x]: conductance of (l,y,x)-(l,y+1,x); 0 at y = ny-1.
    gz[l,y,x]: series-resistor conductance (1/R) of the via (l,y,x)-(l+1,y,x);
               0 at l = layers-1.
    lz[l,y,x]: via series inductance (H) or None (RC grid).
    cap[l,y,x]: node-to-ground capacitance (F).
    pad_node/pad_g/pad_l: pads to Vdd (series R = 1/pad_g, series L or None).
    """
    layers: int
    ny: int
    nx: int
    gx: np.ndarray
    gy: np.ndarray
    gz: np.ndarray
    cap: np.ndarray
    pad_node: np.ndarray
    pad_g: np.ndarray
    vdd: float
    sources: Sources
    lz: Optional[np.ndarray] = None
    pad_l: Optional[np.ndarray] = None
    h: float = 5e-12
    steps: int = 10
    name: str = "mesh"

    @property
    def n(self) -> int:
        return self.layers * self.ny * self.nx

    @property
    def is_rlc(self) -> bool:
        return self.lz is not None or self.pad_l is not None


@dataclass
class EdgeGrid:
    """Irregular grid as an undirected branch list (for the CSR path).

    Branch k joins nodes ``eu[k]`` and ``ev[k]`` with conductance ``eg[k]``.
    Node indices are flat (l, y, x) indices of the mesh the grid came from
    (``layers, ny, nx`` are kept only for reference / partitioning).
    """
    n: int
    eu: np.ndarray
    ev: np.ndarray
    eg: np.ndarray
    cap: np.ndarray
    pad_node: np.ndarray
    pad_g: np.ndarray
    vdd: float
    sources: Sources
    layers: int = 0
    ny: int = 0
    nx: int = 0
    h: float = 5e-12
    steps: int = 10
    name: str = "edges"


def _triangle_sources(rng, nodes, peak_max, start_max, width):
    s = nodes.shape[0]
    peak = rng.uniform(0.0, peak_max, size=s)
    start = rng.uniform(0.0, start_max, size=s)
    t = np.empty((s, 3))
    t[:, 0] = start
    t[:, 1] = start + 0.5 * width
    t[:, 2] = start + width
    i = np.zeros((s, 3))
    i[:, 1] = peak
    ptr = np.arange(0, 3 * s + 1, 3, dtype=np.int64)
    return Sources(node=nodes.astype(np.int64), ptr=ptr, t=t.reshape(-1), i=i.reshape(-1))


def mesh_grid(layers: int, ny: int, nx: int, *, seed: int = 0,
              g_lo: float = 0.67, g_hi: float = 2.0, g_lognormal: Optional[tuple] = None,
              via_g: float = 5.0, pad_g: float = 10.0, pad_pitch: int = 16,
              cap_lo: float = 1e-15, cap_hi: float = 1e-14,
              src_frac: float = 0.2, src_peak: float = 1e-3, src_start: float = 500e-12,
              src_width: float = 100e-12, vdd: float = 1.0,
              rlc: bool = False, pad_r: float = 0.01, pad_l_range=(10e-12, 100e-12),
              via_l_range=(0.1e-12, 1e-12), h: float = 5e-12, steps: int = 10,
              name: str = "mesh") -> MeshGrid:
    """Seeded layered mesh following BASELINE.json config 0/1/3/4 recipes."""
    if layers < 1 or ny < 1 or nx < 1:
        raise ValueError("mesh dimensions must be >= 1")
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = (layers, ny, nx)

    def draw_g(size):
        if g_lognormal is not None:
            mu, sigma = g_lognormal
            return rng.lognormal(mu, sigma, size=size)
        return rng.uniform(g_lo, g_hi, size=size)

    gx = draw_g(shape)
    gx[:, :, nx - 1] = 0.0
    gy = draw_g(shape)
    gy[:, ny - 1, :] = 0.0
    gz = np.full(shape, via_g)
    gz[layers - 1] = 0.0
    cap = rng.uniform(cap_lo, cap_hi, size=shape)

    top = layers - 1
    ys = np.arange(0, ny, pad_pitch)
    xs = np.arange(0, nx, pad_pitch)
    yy, xx = np.meshgrid(ys, xs, indexing="ij")
    pad_node = ((top * ny + yy) * nx + xx).reshape(-1).astype(np.int64)
    npads = pad_node.shape[0]

    lz = None
    pad_l = None
    if rlc:
        lz = rng.uniform(via_l_range[0], via_l_range[1], size=shape)
        lz[layers - 1] = 0.0
        pad_l = rng.uniform(pad_l_range[0], pad_l_range[1], size=npads)
        pad_gv = np.full(npads, 1.0 / pad_r)
    else:
        pad_gv = np.full(npads, pad_g)

    nb = ny * nx
    nsrc = int(round(src_frac * nb))
    bottom = rng.permutation(nb)[:nsrc]
    bottom.sort()
    sources = _triangle_sources(rng, bottom.astype(np.int64), src_peak, src_start, src_width)
    return MeshGrid(layers=layers, ny=ny, nx=nx, gx=gx, gy=gy, gz=gz, cap=cap,
                    pad_node=pad_node, pad_g=pad_gv, vdd=vdd, sources=sources,
                    lz=lz, pad_l=pad_l, h=h, steps=steps, name=name)


def mesh_to_edges(m: MeshGrid):
    """Enumerate the mesh's branches as (u, v, g) with u < v (no arithmetic)."""
    L, NY, NX = m.layers, m.ny, m.nx
    idx = np.arange(m.n, dtype=np.int64).reshape(L, NY, NX)
    us, vs, gs = [], [], []
    if NX > 1:
        us.append(idx[:, :, :-1].reshape(-1)); vs.append(idx[:, :, 1:].reshape(-1))
        gs.append(m.gx[:, :, :-1].reshape(-1))
    if NY > 1:
        us.append(idx[:, :-1, :].reshape(-1)); vs.append(idx[:, 1:, :].reshape(-1))
        gs.append(m.gy[:, :-1, :].reshape(-1))
    if L > 1:
        us.append(idx[:-1].reshape(-1)); vs.append(idx[1:].reshape(-1))
        gs.append(m.gz[:-1].reshape(-1))
    if not us:
        z = np.zeros(0, dtype=np.int64)
        return z, z.copy(), np.zeros(0)
    return np.concatenate(us), np.concatenate(vs), np.concatenate(gs)


def edge_grid(layers: int, ny: int, nx: int, *, seed: int = 0, delete_frac: float = 0.2,
              lognormal=(0.0, 0.5), via_g: float = 5.0, pad_g: float = 10.0,
              pad_pitch: int = 32, src_frac: float = 0.3, h: float = 5e-12,
              steps: int = 10, name: str = "edges", **kw) -> EdgeGrid:
    """BASELINE.json config 2: irregular mesh with ``delete_frac`` of the in-layer
    segments removed while a random spanning tree of the whole grid is kept
    (so every node keeps a path to a pad).  Reading R9: the log-normal
    distribution applies to in-layer segments; vias stay at 5 S."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import minimum_spanning_tree

    m = mesh_grid(layers, ny, nx, seed=seed, g_lognormal=lognormal, via_g=via_g,
                  pad_g=pad_g, pad_pitch=pad_pitch, src_frac=src_frac, h=h,
                  steps=steps, **kw)
    eu, ev, eg = mesh_to_edges(m)
    n = m.n
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    is_via = (ev - eu) == ny * nx
    ne = eu.shape[0]
    keep = np.ones(ne, dtype=bool)
    if ne > 0 and delete_frac > 0:
        # random spanning tree: MST under i.i.d. random weights (Kruskal in scipy)
        w = rng.uniform(1.0, 2.0, size=ne)
        mst = minimum_spanning_tree(coo_matrix((w, (eu, ev)), shape=(n, n)).tocsr()).tocoo()
        tu = np.minimum(mst.row, mst.col).astype(np.int64)
        tv = np.maximum(mst.row, mst.col).astype(np.int64)
        key_all = eu * n + ev
        in_tree = np.isin(key_all, tu * n + tv)
        cand = np.flatnonzero(~in_tree & ~is_via)
        n_in_layer = int((~is_via).sum())
        n_del = min(int(round(delete_frac * n_in_layer)), cand.shape[0])
        dele = rng.choice(cand, size=n_del, replace=False)
        keep[dele] = False
    return EdgeGrid(n=n, eu=eu[keep], ev=ev[keep], eg=eg[keep], cap=m.cap.reshape(-1).copy(),
                    pad_node=m.pad_node, pad_g=m.pad_g, vdd=m.vdd, sources=m.sources,
                    layers=layers, ny=ny, nx=nx, h=h, steps=steps, name=name)


# BASELINE.json configs (index -> recipe).  ``dims`` are (layers, ny, nx).
CONFIGS = {
    0: dict(kind="mesh", dims=(2, 64, 64), pad_pitch=16, src_frac=0.2, h=10e-12, steps=100),
    1: dict(kind="mesh", dims=(4, 1024, 1024), pad_pitch=32, src_frac=0.3, h=5e-12, steps=500),
    2: dict(kind="edges", dims=(2, 2048, 2048), pad_pitch=32, src_frac=0.3, h=5e-12, steps=500),
    3: dict(kind="mesh", dims=(4, 2048, 2048), pad_pitch=32, src_frac=0.3, h=2e-12, steps=1000,
            rlc=True),
    4: dict(kind="mesh", dims=(8, 4096, 4096), pad_pitch=64, src_frac=0.3, h=5e-12, steps=200),
}


def config_grid(k: int, *, seed: int = 0, dims=None, steps=None):
    """Grid for BASELINE.json config ``k``; ``dims``/``steps`` override the size
    (same distributions) for the small parity cases."""
    c = dict(CONFIGS[k])
    kind = c.pop("kind")
    L, NY, NX = dims if dims is not None else c.pop("dims")
    c.pop("dims", None)
    if steps is not None:
        c["steps"] = steps
    name = f"config{k}" + ("" if dims is None else f"@{L}x{NY}x{NX}")
    if kind == "mesh":
        return mesh_grid(L, NY, NX, seed=seed, name=name, **c)
    return edge_grid(L, NY, NX, seed=seed, name=name, **c)


def scaled_config(k: int, L: int, NY: int, NX: int, *, seed: int = 0, steps=None):
    return config_grid(k, seed=seed, dims=(L, NY, NX), steps=steps)
