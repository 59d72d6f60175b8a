"""GPU parity (-m gpu): the sm_100a path through the C ABI against the oracle.

Bars:
  * fixed-sweep iterates (tol <= 0): the GPU red-black sweep is Eq. (13)/(15) in
    the red-black numbering, so it must equal the oracle's sequential sweep in
    that numbering up to fp64 rounding: |dV| <= 1e-12 V;
  * converged transients at tol = 1e-10: |V_gpu - V_oracle| <= 1e-8 V per node
    per step (BASELINE.json north_star);
  * integer outputs (sweep counts) compared where both sides take the same
    decision.
"""
import numpy as np
import pytest

import gridgen
from oracle import netlist, nodal, pwl
from sweepcount import check_counts_same_stopping

pytestmark = pytest.mark.gpu

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


def oracle_run(g, steps, tol, omega, method="gs", order="redblack", max_sweeps=200000, form="companion",
               series_rl="node", trace=False, check_every=1):
    nl = netlist.from_grid(g, series_rl)
    It = pwl.node_currents_table(nl, g.h, steps)
    o = nodal.NodalOracle(nl)
    ordr = None
    if order == "redblack":
        ordr = nodal.red_black_order(g.layers, g.ny, g.nx)
    r = o.transient(g.h, steps, tol=tol, omega=omega, method=method, order=ordr, Itab=It,
                    max_sweeps=max_sweeps, form=form, trace=trace, check_every=check_every)
    return r, nl


def gpu_run(P, g, steps, tol, omega, method="rbsor", max_sweeps=200000, device=False, options=None):
    G = P.Grid.from_mesh_grid(g, device=device) if hasattr(g, "gx") else P.Grid.from_edge_grid(g, device=device)
    for k, v in (options or {}).items():
        G.set_option(k, v)
    n = g.n
    r = G.transient(g.h, steps, tol=tol, omega=omega, method=method, max_sweeps=max_sweeps,
                    probes=np.arange(n, dtype=np.int64), raise_on_noconv=False)
    V = G.voltages()
    G.close()
    return r, V


SHAPES = [(2, 6, 5), (1, 7, 9), (3, 4, 4), (2, 1, 9), (1, 1, 1), (4, 9, 70), (2, 33, 31), (8, 5, 3)]


def mk(L, NY, NX, seed, rlc=False):
    return gridgen.mesh_grid(L, NY, NX, seed=seed, pad_pitch=3, src_frac=0.5, h=10e-12 if not rlc else 2e-12,
                             src_start=20e-12, src_width=40e-12, rlc=rlc)


@pytest.mark.parametrize("F,resident", [(1, 0), (2, 0), (0, 1)])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("omega", [1.0, 1.7])
def test_rb_sweep_iterates_equal_oracle(pgb, shape, omega, F, resident):
    # the streaming mesh sweep with F = 1 (one sweep per launch) and F = 2, and
    # the one-CTA resident sweep loop that small meshes use by default
    g = mk(*shape, seed=sum(shape))
    steps, k = 6, 5
    ro, _ = oracle_run(g, steps, tol=0.0, omega=omega, max_sweeps=k)
    rg, V = gpu_run(pgb, g, steps, tol=0.0, omega=omega, max_sweeps=k,
                    options={"fuse": F, "resident": resident})
    assert np.all(rg.sweeps[1:] == k)
    np.testing.assert_allclose(rg.probes, ro.V[:, :g.n], rtol=0, atol=ATOL_ITER)
    np.testing.assert_allclose(V, ro.V[-1, :g.n], rtol=0, atol=ATOL_ITER)


FUSED_SHAPES = [(2, 6, 5), (1, 1, 1), (4, 9, 70), (2, 33, 31), (8, 5, 3), (4, 40, 150), (3, 23, 64)]


@pytest.mark.parametrize("shape", FUSED_SHAPES)
@pytest.mark.parametrize("F,lag,rows,width", [(1, 3, 0, 32), (2, 3, 0, 32), (3, 3, 0, 32), (4, 3, 0, 32),
                                              (2, 4, 0, 32), (2, 3, 7, 32), (3, 3, 4, 32), (4, 3, 64, 32),
                                              (1, 3, 0, 64), (2, 3, 0, 64), (3, 3, 0, 64), (2, 3, 5, 64)])
def test_fused_sweep_iterates_equal_oracle(pgb, shape, F, lag, rows, width):
    # F red-black SOR sweeps per streaming pass (temporal blocking);
    # k = 5 sweeps per step exercises the partial last launch (nsw < F)
    g = mk(*shape, seed=3 * sum(shape) + F)
    steps, k, omega = 4, 5, 1.6
    ro, _ = oracle_run(g, steps, tol=0.0, omega=omega, max_sweeps=k)
    rg, V = gpu_run(pgb, g, steps, tol=0.0, omega=omega, max_sweeps=k,
                    options={"fuse": F, "lag": lag, "rows": rows, "width": width, "resident": 0})
    assert np.all(rg.sweeps[1:] == k)
    np.testing.assert_allclose(rg.probes, ro.V[:, :g.n], rtol=0, atol=ATOL_ITER)
    np.testing.assert_allclose(V, ro.V[-1, :g.n], rtol=0, atol=ATOL_ITER)


@pytest.mark.parametrize("F", [2, 3, 4])
def test_fused_converged_sweep_counts(pgb, F):
    # convergence is tested after every launch (every F sweeps): the GPU stops
    # at the first multiple of F at or after the oracle's stopping sweep
    g = gridgen.config_grid(0, dims=(2, 40, 48), steps=15)
    ro, _ = oracle_run(g, 15, tol=1e-10, omega=1.9)
    rg, _ = gpu_run(pgb, g, 15, tol=1e-10, omega=1.9, options={"fuse": F, "resident": 0})
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_CONV)
    # the oracle with the GPU's stopping semantics (line 8 tested every F
    # sweeps, R13) runs the same iteration: same counts, iterates to rounding
    rf, _ = oracle_run(g, 15, tol=1e-10, omega=1.9, trace=True, check_every=F)
    np.testing.assert_allclose(rg.probes, rf.V, rtol=0, atol=ATOL_ITER)
    check_counts_same_stopping(rg.sweeps, rf.sweeps, rf.dtrace, 1e-10, F)


@pytest.mark.parametrize("shape", SHAPES[:5])
def test_jacobi_iterates_equal_oracle(pgb, shape):
    g = mk(*shape, seed=7 + sum(shape))
    steps, k = 4, 6
    ro, _ = oracle_run(g, steps, tol=0.0, omega=0.9, method="jacobi", order=None, max_sweeps=k)
    rg, _ = gpu_run(pgb, g, steps, tol=0.0, omega=0.9, method="jacobi", max_sweeps=k)
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_ITER)


@pytest.mark.parametrize("shape", [(2, 6, 5), (3, 4, 4), (2, 1, 6)])
def test_rlc_iterates_vs_converged(pgb, shape):
    # GPU eliminates the series R-L internal node (reading R7) so iterates differ
    # from the oracle's; converged solutions must agree.
    g = mk(*shape, seed=50 + sum(shape), rlc=True)
    steps = 12
    ro, nl = oracle_run(g, steps, tol=1e-14, omega=1.8, order=None)
    assert ro.status == 0
    rg, _ = gpu_run(pgb, g, steps, tol=1e-14, omega=1.8)
    assert rg.status == 0
    n = g.n
    assert np.abs(ro.V[:, :n] - 1.0).max() > 1e-6
    np.testing.assert_allclose(rg.probes, ro.V[:, :n], rtol=0, atol=ATOL_CONV)


@pytest.mark.parametrize("shape", [(2, 6, 5), (3, 4, 4), (2, 1, 6), (4, 9, 70), (8, 5, 3)])
@pytest.mark.parametrize("F", [1, 2, 3])
def test_rlc_iterates_equal_oracle_series_element(pgb, shape, F):
    # the oracle's series R-L element (one branch, R7) is the GPU's
    # companion model: fixed-sweep iterates agree to rounding
    g = mk(*shape, seed=60 + sum(shape), rlc=True)
    steps, k = 8, 5
    ro, _ = oracle_run(g, steps, tol=0.0, omega=1.6, max_sweeps=k, series_rl="element")
    rg, V = gpu_run(pgb, g, steps, tol=0.0, omega=1.6, max_sweeps=k, options={"fuse": F, "resident": 0})
    assert np.abs(ro.V - 1.0).max() > 1e-6
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_ITER)


@pytest.mark.parametrize("resident", [1, 0])
def test_config0_full_size_converged(pgb, resident):
    # BASELINE config 0 at full size: 2 x 64 x 64, h = 10 ps, 100 steps, tol 1e-10
    # (resident one-CTA sweep loop by default; the streaming sweep with F = 2)
    g = gridgen.config_grid(0)
    steps, omega = g.steps, 1.9
    ro, _ = oracle_run(g, steps, tol=1e-10, omega=omega)
    rg, _ = gpu_run(pgb, g, steps, tol=1e-10, omega=omega, options={"resident": resident})
    assert ro.status == 0 and rg.status == 0
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_CONV)
    # same numbering, same arithmetic up to rounding -> the same stopping
    # decisions outside the rounding band (the resident sweep tests after every
    # sweep, the streaming one every F = 2)
    F = int(rg.stats.sweeps_per_launch)
    assert F == (1 if resident else 2)
    rf, _ = oracle_run(g, steps, tol=1e-10, omega=omega, trace=True, check_every=F)
    np.testing.assert_allclose(rg.probes, rf.V, rtol=0, atol=ATOL_ITER)
    check_counts_same_stopping(rg.sweeps, rf.sweeps, rf.dtrace, 1e-10, F)


def test_redblack_vs_natural_order_tight(pgb):
    # the GPU's red-black numbering converges to the paper's natural-order solution
    g = gridgen.config_grid(0, dims=(2, 24, 24), steps=20)
    ro, _ = oracle_run(g, 20, tol=1e-13, omega=1.9, order="natural")
    rg, _ = gpu_run(pgb, g, 20, tol=1e-13, omega=1.9)
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_CONV)


def test_csr_grid(pgb):
    g = gridgen.edge_grid(2, 20, 18, seed=3, pad_pitch=6, h=5e-12, src_start=20e-12, src_width=40e-12)
    steps = 8
    nl = netlist.from_edges(g)
    It = pwl.node_currents_table(nl, g.h, steps)
    o = nodal.NodalOracle(nl)
    order = nodal.red_black_order(2, 20, 18)   # BFS parity of a connected mesh subgraph
    ro = o.transient(g.h, steps, tol=0.0, omega=1.5, order=order, Itab=It, max_sweeps=7)
    rg, _ = gpu_run(pgb, g, steps, tol=0.0, omega=1.5, max_sweeps=7)
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_ITER)
    ro = o.transient(g.h, steps, tol=1e-12, omega=1.7, Itab=It)
    rg, _ = gpu_run(pgb, g, steps, tol=1e-12, omega=1.7)
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_CONV)
    # weighted Jacobi on the CSR rows
    ro = o.transient(g.h, steps, tol=0.0, omega=0.9, method="jacobi", Itab=It, max_sweeps=5)
    rg, _ = gpu_run(pgb, g, steps, tol=0.0, omega=0.9, method="jacobi", max_sweeps=5)
    np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=ATOL_ITER)


def test_zero_current_settles_to_vdd(pgb):
    g = mk(3, 17, 40, seed=1)
    g.sources = gridgen.Sources(node=np.zeros(0, np.int64), ptr=np.zeros(1, np.int64), t=np.zeros(0), i=np.zeros(0))
    for F in (1, 2, 3):
        rg, V = gpu_run(pgb, g, 10, tol=1e-12, omega=1.5, options={"fuse": F, "resident": 0})
        assert np.abs(rg.probes - 1.0).max() <= 1e-13
        # one launch (F sweeps) per step: the first sweep already meets tol
        assert np.all(rg.sweeps[1:] == F)


def test_device_inputs_equal_host_inputs(pgb):
    import torch
    g = mk(4, 9, 70, seed=11)
    P = pgb
    G1 = P.Grid.from_mesh_grid(g, device=False)
    G2 = P.Grid.from_mesh_grid(g, device=True)
    pr = torch.arange(g.n, dtype=torch.int64, device="cuda")
    r1 = G1.transient(g.h, 5, tol=1e-11, omega=1.6, probes=np.arange(g.n))
    r2 = G2.transient(g.h, 5, tol=1e-11, omega=1.6, probes=pr)
    np.testing.assert_array_equal(r1.probes, r2.probes.cpu().numpy())
    out = torch.empty(g.n, dtype=torch.float64, device="cuda")
    G2.voltages(out)
    np.testing.assert_array_equal(G1.voltages(), out.cpu().numpy())


def test_errors_are_reported(pgb):
    P = pgb
    g = mk(2, 6, 5, seed=2)
    G = P.Grid.from_mesh_grid(g)
    with pytest.raises(P.PgError):
        G.transient(g.h, 3, omega=2.0)
    with pytest.raises(P.PgNoConvergence):
        G.transient(g.h, 3, tol=1e-30, omega=1.0, max_sweeps=3)
    with pytest.raises(P.PgError):
        G.transient(-1.0, 3)
    with pytest.raises(P.PgError):
        G.set_sources(np.array([10 ** 9]), np.array([0, 1]), np.array([0.0]), np.array([1.0]))
