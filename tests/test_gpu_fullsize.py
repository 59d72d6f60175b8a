"""Full-size parity (-m gpu): BASELINE.json configs 1-4 at their full sizes, in
the launch configuration bench.py times (default options: fused red-black
sweep, F = 2, automatic rows per CTA), against the oracle.

* configs 1, 2, 3: fixed-sweep iterates (tol = 0, k sweeps per step) of the
  whole grid against the oracle's sequential sweep in the same numbering,
  |dV| <= 1e-12 V at every node (DESIGN.md §5 derivation);
* configs 1, 2: converged first steps (tol = 1e-10) at every node, <= 1e-8 V;
* config 4 (134M nodes, too large for the oracle as a whole): sampled outputs.
  After s steps of k sweeps from x(0) = Vdd a node's value depends only on
  nodes within 2 k s hops (one hop per half-sweep), so the oracle computes it
  exactly on a patch of radius R > 2 k s around the node (global red-black
  parity kept by even patch offsets); patches are centred on the earliest
  loads so the sampled values actually move.
"""
import numpy as np
import pytest

import gridgen
from oracle import netlist, nodal, pwl

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ATOL_ITER = 1e-12
ATOL_CONV = 1e-8


@pytest.fixture(scope="module")
def pgb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1409_7166_b200 as P
    from paper_1409_7166_b200 import build
    build.build()
    return P


def gpu_iterates(P, g, steps, k, omega, probes=None, tol=0.0):
    mk = P.Grid.from_mesh_grid if hasattr(g, "gx") else P.Grid.from_edge_grid
    G = mk(g, device=True)
    pr = None if probes is None else np.asarray(probes, dtype=np.int64)
    r = G.transient(g.h, steps, tol=tol, omega=omega, max_sweeps=k if tol <= 0 else 200000,
                    probes=pr)
    V = G.voltages()
    G.close()
    return r, V


def oracle_iterates(g, steps, k, omega, series_rl="node", tol=0.0):
    nl = netlist.from_grid(g, series_rl)
    It = pwl.node_currents_table(nl, g.h, steps)
    order = nodal.red_black_order(g.layers, g.ny, g.nx)
    return nodal.NodalOracle(nl).transient(g.h, steps, tol=tol, omega=omega, order=order, Itab=It,
                                           max_sweeps=k if tol <= 0 else 200000)


def _sample(n, count, seed):
    return np.sort(np.random.default_rng(seed).choice(n, size=count, replace=False))


@pytest.mark.parametrize("cfg,steps,k,omega,series_rl", [
    (1, 12, 6, 1.98, "node"),
    (2, 4, 6, 1.98, "node"),
    (3, 4, 4, 1.99, "element"),
])
def test_full_size_iterates(pgb, cfg, steps, k, omega, series_rl):
    g = gridgen.config_grid(cfg)
    pr = _sample(g.n, 4096, cfg)
    rg, V = gpu_iterates(pgb, g, steps, k, omega, probes=pr)
    ro = oracle_iterates(g, steps, k, omega, series_rl)
    assert np.all(rg.sweeps[1:] == k)
    assert np.abs(ro.V[-1, :g.n] - 1.0).max() > 1e-6          # the loads act
    np.testing.assert_allclose(V, ro.V[-1, :g.n], rtol=0, atol=ATOL_ITER)
    np.testing.assert_allclose(rg.probes, ro.V[:, pr], rtol=0, atol=ATOL_ITER)


def test_config1_full_size_converged(pgb):
    g = gridgen.config_grid(1)
    steps = 2
    pr = _sample(g.n, 4096, 11)
    rg, V = gpu_iterates(pgb, g, steps, 0, 1.98, probes=pr, tol=1e-10)
    ro = oracle_iterates(g, steps, 0, 1.98, tol=1e-10)
    assert rg.status == 0 and ro.status == 0
    np.testing.assert_allclose(V, ro.V[-1], rtol=0, atol=ATOL_CONV)
    np.testing.assert_allclose(rg.probes, ro.V[:, pr], rtol=0, atol=ATOL_CONV)
    F = int(rg.stats.sweeps_per_launch)
    assert np.all(rg.sweeps[1:] == -(-ro.sweeps[1:] // F) * F)


@pytest.mark.parametrize("cfg,steps,omega,series_rl", [(2, 1, 1.98, "node")])
def test_full_size_converged(pgb, cfg, steps, omega, series_rl):
    # converged transient steps (tol = 1e-10) of the irregular CSR grid at full
    # size: every node within 1e-8 V of the oracle (north_star bar), the same
    # sweep count.  (The RLC config 3 passed the same check for one step, but
    # its whole-grid oracle solve takes ~5 minutes: converged RLC parity is
    # kept at reduced sizes, test_gpu_parity.py, plus config 3's full-size
    # fixed-sweep iterates above.)
    g = gridgen.config_grid(cfg)
    pr = _sample(g.n, 4096, 20 + cfg)
    rg, V = gpu_iterates(pgb, g, steps, 0, omega, probes=pr, tol=1e-10)
    ro = oracle_iterates(g, steps, 0, omega, series_rl, tol=1e-10)
    assert rg.status == 0 and ro.status == 0
    assert np.abs(ro.V[-1, :g.n] - 1.0).max() > 1e-9          # the loads act
    np.testing.assert_allclose(V, ro.V[-1, :g.n], rtol=0, atol=ATOL_CONV)
    np.testing.assert_allclose(rg.probes, ro.V[:, pr], rtol=0, atol=ATOL_CONV)
    F = int(rg.stats.sweeps_per_launch)
    assert np.all(rg.sweeps[1:] == -(-ro.sweeps[1:] // F) * F)


def patch(g, y0, x0, R):
    """Sub-mesh rows [y0, y0+2R), columns [x0, x0+2R) of all layers (even
    offsets keep the global red-black parity), pads and loads inside it."""
    y1, x1 = min(y0 + 2 * R, g.ny), min(x0 + 2 * R, g.nx)
    sl = (slice(None), slice(y0, y1), slice(x0, x1))
    gx = g.gx[sl].copy(); gx[:, :, -1] = 0.0
    gy = g.gy[sl].copy(); gy[:, -1, :] = 0.0
    L, NY, NX = g.layers, y1 - y0, x1 - x0

    def local(idx):
        l, r = np.divmod(idx, g.ny * g.nx)
        y, x = np.divmod(r, g.nx)
        inside = (y >= y0) & (y < y1) & (x >= x0) & (x < x1)
        return inside, (l * NY + (y - y0)) * NX + (x - x0)

    pin, pidx = local(g.pad_node)
    s = g.sources
    sin, sidx = local(s.node)
    keep = np.flatnonzero(sin)
    ptr = [0]
    t, i = [], []
    for q in keep:
        t.append(s.t[s.ptr[q]:s.ptr[q + 1]]); i.append(s.i[s.ptr[q]:s.ptr[q + 1]])
        ptr.append(ptr[-1] + s.ptr[q + 1] - s.ptr[q])
    src = gridgen.Sources(node=sidx[keep].astype(np.int64), ptr=np.array(ptr, np.int64),
                          t=np.concatenate(t) if t else np.zeros(0),
                          i=np.concatenate(i) if i else np.zeros(0))
    sub = gridgen.MeshGrid(layers=L, ny=NY, nx=NX, gx=gx, gy=gy, gz=g.gz[sl].copy(),
                           cap=g.cap[sl].copy(), pad_node=pidx[pin].astype(np.int64),
                           pad_g=g.pad_g[pin], vdd=g.vdd, sources=src, h=g.h, steps=g.steps)
    return sub, (y0, x0)


def test_config4_sampled_patches(pgb):
    g = gridgen.config_grid(4)
    steps, k, omega = 6, 4, 1.99
    R = 2 * k * steps + 4                       # > 2 k s hops
    # centres: the nodes above the earliest-starting loads, plus random nodes
    s = g.sources
    early = s.node[np.argsort(s.t[s.ptr[:-1]])[:6]]
    rng = np.random.default_rng(4)
    centres = list(early) + list(rng.choice(g.n, size=2, replace=False))
    rg, V = gpu_iterates(pgb, g, steps, k, omega)
    moved = 0
    for c in centres:
        l, r = divmod(int(c), g.ny * g.nx)
        y, x = divmod(r, g.nx)
        y0 = max(0, (y - R) & ~1)
        x0 = max(0, (x - R) & ~1)
        sub, _ = patch(g, y0, x0, R)
        ro = oracle_iterates(sub, steps, k, omega)
        # the centre column (all layers) and its 3 x 3 neighbourhood
        for ll in range(g.layers):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    yy, xx = y + dy, x + dx
                    if not (0 <= yy < g.ny and 0 <= xx < g.nx):
                        continue
                    gi = (ll * g.ny + yy) * g.nx + xx
                    li = (ll * sub.ny + (yy - y0)) * sub.nx + (xx - x0)
                    assert abs(V[gi] - ro.V[-1, li]) <= ATOL_ITER, (c, ll, dy, dx)
                    moved += abs(V[gi] - 1.0) > 1e-7
    assert moved > 0
