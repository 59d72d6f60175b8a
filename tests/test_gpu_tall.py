"""Per-colour mesh sweep (-m gpu): meshes taller than the strip kernels' 8
layers, and option "colour" on any mesh.

k_rb_colour_mesh runs one red-black SOR sweep (Eq. (13) + (15) in the
red-black numbering, R12) as two launches, one per colour.  Bars as in
test_gpu_parity.py: fixed-sweep iterates within 1e-12 V of the
oracle's sequential sweep in the same numbering, converged results within
1e-8 V; the same operand order as the streaming kernels, so option "colour" on
a mesh of <= 8 layers gives their iterates bit for bit.
"""
import numpy as np
import pytest

import gridgen
from sweepcount import check_counts_same_stopping
from test_gpu_parity import ATOL_CONV, ATOL_ITER, gpu_run, mk, oracle_run

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


TALL = [(9, 5, 7), (12, 9, 17), (16, 3, 70), (10, 33, 31), (9, 1, 2), (256, 2, 3)]


@pytest.mark.parametrize("shape", TALL)
@pytest.mark.parametrize("resident", [0, 1])
def test_tall_mesh_iterates_equal_oracle(pgb, shape, resident):
    # > 8 layers: the per-colour sweep (resident 0) or, where the mesh fits a
    # cluster, the resident sweep loop (any layer count)
    g = mk(*shape, seed=7 * sum(shape))
    steps, k, omega = 5, 5, 1.7
    ro, _ = oracle_run(g, steps, tol=0.0, omega=omega, max_sweeps=k)
    rg, V = gpu_run(pgb, g, steps, tol=0.0, omega=omega, max_sweeps=k, options={"resident": resident})
    assert np.all(rg.sweeps[1:] == k)
    assert np.abs(ro.V - 1.0).max() > 1e-6                    # the loads act
    np.testing.assert_allclose(rg.probes, ro.V[:, :g.n], rtol=0, atol=ATOL_ITER)
    np.testing.assert_allclose(V, ro.V[-1, :g.n], rtol=0, atol=ATOL_ITER)


@pytest.mark.parametrize("shape", [(9, 5, 7), (12, 9, 17), (10, 33, 31)])
def test_tall_rlc_iterates_equal_oracle_series_element(pgb, shape):
    # series R-L vias and pads (R7: the oracle's element model is the GPU's
    # companion elimination)
    g = mk(*shape, seed=60 + sum(shape), rlc=True)
    steps, k = 6, 5
    ro, _ = oracle_run(g, steps, tol=0.0, omega=1.6, max_sweeps=k, series_rl="element")
    rg, _ = gpu_run(pgb, g, steps, tol=0.0, omega=1.6, max_sweeps=k, options={"resident": 0})
    assert np.abs(ro.V - 1.0).max() > 1e-6
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_ITER)


def test_tall_mesh_converged(pgb):
    # tol = 1e-10: within 1e-8 V of the oracle at every step, and the same
    # stopping sweep (the per-colour sweep tests after every sweep, F = 1)
    g = gridgen.mesh_grid(12, 24, 40, seed=5, pad_pitch=8, src_frac=0.3, h=5e-12, src_start=10e-12,
                          src_width=100e-12)
    steps, omega, tol = 12, 1.9, 1e-10
    ro, _ = oracle_run(g, steps, tol=tol, omega=omega, trace=True)
    rg, _ = gpu_run(pgb, g, steps, tol=tol, omega=omega, options={"resident": 0})
    assert ro.status == 0 and rg.status == 0
    assert np.abs(ro.V - 1.0).max() > 1e-6
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_CONV)
    check_counts_same_stopping(rg.sweeps, ro.sweeps, ro.dtrace, tol, 1)


@pytest.mark.parametrize("shape", [(2, 6, 5), (4, 9, 70), (8, 5, 3), (3, 23, 64), (1, 1, 1)])
@pytest.mark.parametrize("rlc", [False, True])
def test_colour_option_bit_identical_to_streaming(pgb, shape, rlc):
    # option "colour" on <= 8 layers: the same iterates as the streaming
    # two-sweep pipeline (k even: full F = 2 launches), bit for bit
    g = mk(*shape, seed=11 * sum(shape), rlc=rlc)
    steps, k, omega = 5, 6, 1.7
    ra, Va = gpu_run(pgb, g, steps, tol=0.0, omega=omega, max_sweeps=k, options={"resident": 0})
    rb, Vb = gpu_run(pgb, g, steps, tol=0.0, omega=omega, max_sweeps=k, options={"resident": 0, "colour": 1})
    assert int(ra.stats.sweeps_per_launch) == 2 and int(rb.stats.sweeps_per_launch) == 1
    assert np.array_equal(ra.probes, rb.probes)
    assert np.array_equal(Va, Vb)


def test_tall_mesh_continue_equals_one_call(pgb):
    # Algorithm 1 cut at step boundaries (R18) on the per-colour path
    g = mk(12, 9, 17, seed=3)
    G = pgb.Grid.from_mesh_grid(g)
    G.set_option("resident", 0)
    G.transient(g.h, 9, tol=1e-10, omega=1.8)
    V1 = G.voltages()
    G.close()
    G = pgb.Grid.from_mesh_grid(g)
    G.set_option("resident", 0)
    G.transient(g.h, 2, tol=1e-10, omega=1.8)
    G.transient(g.h, 3, tol=1e-10, omega=1.8, cont=True)
    G.transient(g.h, 4, tol=1e-10, omega=1.8, cont=True)
    V2 = G.voltages()
    G.close()
    assert np.array_equal(V1, V2)


def test_tall_mesh_limits(pgb):
    g = mk(9, 4, 4, seed=1)
    G = pgb.Grid.from_mesh_grid(g)
    with pytest.raises(pgb.PgError):                           # slabs need the strip kernels
        pgb._lib.check(G._lib.pg_set_slab(G._h, 0, 2, 0))
    G.close()
    g = mk(257, 1, 2, seed=1)
    with pytest.raises(pgb.PgError):
        pgb.Grid.from_mesh_grid(g)


def test_tall_mesh_dc_matches_dense_solve(pgb):
    # DC (A = G, §II-A) on a 12-layer mesh through the per-colour sweep
    from oracle import dense, netlist, pwl
    g = gridgen.mesh_grid(12, 5, 6, seed=9, pad_pitch=3, src_frac=0.5, h=10e-12, src_start=5e-12,
                          src_width=40e-12)
    t = 20e-12
    G = pgb.Grid.from_mesh_grid(g)
    G.set_option("resident", 0)
    G.dc(t=t, tol=1e-15, omega=1.7, max_sweeps=2_000_000)
    V = G.voltages()
    G.close()
    nl = netlist.from_mesh(g)
    Vd = dense.dc_solve(nl, pwl.node_currents(nl, t))
    assert np.abs(Vd - 1.0).max() > 1e-6
    np.testing.assert_allclose(V, Vd, rtol=0, atol=1e-9)
