"""GPU parity of the two-level pipeline sweep kernel (k_rb_sweep2, option "pipe").

Full launches of F = 2 red-black SOR sweeps run k_rb_sweep2 by default.  Its
arithmetic per node update is the same Eq. (13) + (15) expression as the
generic temporally blocked kernel (k_rb_sweep_fused), so the two must agree
bit for bit, and both must equal the oracle's sequential red-black SOR
iterates to 1e-12 V.  Shapes and "rows" (rows per CTA) are
chosen so that the warm-up (7 steps), the steady 12-step body and every tail
length occur, for every compiled layer count L = 1..8, ragged column counts
and strips.
"""
import numpy as np
import pytest

import gridgen
from oracle import netlist, nodal, pwl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pgb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1409_7166_b200 as P
    from paper_1409_7166_b200 import build
    build.build()
    return P


def mk(L, NY, NX, seed, rlc=False):
    return gridgen.mesh_grid(L, NY, NX, seed=seed, pad_pitch=5, src_frac=0.4, h=10e-12 if not rlc else 2e-12,
                             src_start=10e-12, src_width=40e-12, rlc=rlc)


def run(P, g, steps, k, omega, options, tol=0.0):
    G = P.Grid.from_mesh_grid(g, device=True)
    G.set_option("resident", 0)
    for key, v in options.items():
        G.set_option(key, v)
    r = G.transient(g.h, steps, tol=tol, omega=omega, max_sweeps=k, probes=np.arange(g.n, dtype=np.int64),
                    raise_on_noconv=False)
    G.close()
    return r


def oracle_iterates(g, steps, k, omega, series_rl="node"):
    nl = netlist.from_grid(g, series_rl)
    It = pwl.node_currents_table(nl, g.h, steps)
    o = nodal.NodalOracle(nl)
    r = o.transient(g.h, steps, tol=0.0, omega=omega, method="gs",
                    order=nodal.red_black_order(g.layers, g.ny, g.nx), Itab=It, max_sweeps=k)
    return r.V[:, :g.n]


CASES = [
    # (L, NY, NX, rows): rows per CTA -> steady blocks and tail lengths vary
    (1, 40, 131, 13),
    (2, 45, 70, 29),
    (3, 31, 128, 0),
    (4, 37, 130, 17),
    (4, 64, 250, 40),
    (5, 29, 65, 20),
    (6, 22, 40, 7),
    (7, 19, 33, 12),
    (8, 26, 64, 19),
    (4, 3, 9, 1),
    (2, 100, 5, 61),
]


@pytest.mark.parametrize("case", CASES)
def test_pipe_equals_fused_and_oracle(pgb, case):
    L, NY, NX, rows = case
    g = mk(L, NY, NX, seed=7 * L + NY)
    steps, k, omega = 3, 6, 1.8
    opts = {"fuse": 2, "rows": rows}
    rp = run(pgb, g, steps, k, omega, {**opts, "pipe": 1})
    rf = run(pgb, g, steps, k, omega, {**opts, "pipe": 0})
    assert np.all(rp.sweeps[1:] == k)
    assert np.array_equal(rp.probes, rf.probes), np.abs(rp.probes - rf.probes).max()
    Vo = oracle_iterates(g, steps, k, omega)
    np.testing.assert_allclose(rp.probes, Vo, rtol=0, atol=1e-12)


@pytest.mark.parametrize("L,NY,NX,rows", [(4, 40, 70, 11), (2, 33, 64, 0)])
def test_pipe_rlc_equals_fused(pgb, L, NY, NX, rows):
    # RLC meshes: the sweep sees the companion conductances g_e = 1/(R + L/h)
    g = mk(L, NY, NX, seed=3 + L, rlc=True)
    steps, k, omega = 3, 4, 1.6
    opts = {"fuse": 2, "rows": rows}
    rp = run(pgb, g, steps, k, omega, {**opts, "pipe": 1})
    rf = run(pgb, g, steps, k, omega, {**opts, "pipe": 0})
    assert np.array_equal(rp.probes, rf.probes)
    Vo = oracle_iterates(g, steps, k, omega, series_rl="element")
    np.testing.assert_allclose(rp.probes, Vo, rtol=0, atol=1e-12)


@pytest.mark.parametrize("opts", [{"pdl": 1}, {"pdl": 0}, {"pdl": 1, "timing": 1}, {"pdl": 1, "graph": 0},
                                  {"pdl": 1, "batch": 3}])
def test_pipe_converged_matches_fused(pgb, opts):
    # converged transient (tol 1e-10): identical sweep counts and voltages,
    # with and without programmatic dependent launch, graphs, timing events
    g = mk(4, 48, 96, seed=11)
    rp = run(pgb, g, 8, 100000, 1.9, {"pipe": 1, **opts}, tol=1e-10)
    rf = run(pgb, g, 8, 100000, 1.9, {"pipe": 0}, tol=1e-10)
    assert np.array_equal(rp.sweeps, rf.sweeps)
    assert np.array_equal(rp.probes, rf.probes)


def test_timing_option_accounts_sweep_launches(pgb):
    # option "timing": per-step event pairs around the sweep launches; the
    # launches that did work are ceil(sweeps / F) per step, the sweep time is
    # part of the device time
    g = mk(4, 48, 96, seed=5)
    G = pgb.Grid.from_mesh_grid(g, device=True)
    G.set_option("resident", 0)
    G.set_option("timing", 1)
    r = G.transient(g.h, 6, tol=1e-10, omega=1.9, max_sweeps=100000)
    G.close()
    F = int(r.stats.sweeps_per_launch)
    assert F == 2
    assert int(r.stats.sweep_launches) == int(sum((s + F - 1) // F for s in r.sweeps[1:]))
    assert 0.0 < float(r.stats.sweep_ms) <= float(r.stats.device_ms)
