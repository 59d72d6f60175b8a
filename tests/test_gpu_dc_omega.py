"""DC analysis (pg_dc) and Young's relaxation factor (pg_estimate_omega)
against the oracle (-m gpu).

* DC (§II-A "In DC analysis, A = G"): converged GPU solution vs the
  oracle's dense solve of G v = -i(t) - G_s v_d (RC), and vs the oracle's
  nodal iteration with the series R-L element at h = 1e300 (RLC; C/h -> 0,
  h/(L + R h) -> 1/R), <= 1e-9 V.
* omega: the GPU's power-iteration estimate of the Jacobi spectral radius vs
  the eigenvalues of J = I - D^{-1} M of the oracle's dense system matrix
  M = C/h + G (Eq. (11)), and Young's omega speeds up the transient.
"""
import numpy as np
import pytest

import gridgen
from oracle import dense, netlist, nodal, pwl

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


def grid(shape, seed, rlc=False):
    return gridgen.mesh_grid(*shape, seed=seed, pad_pitch=3, src_frac=0.5, h=10e-12, src_start=5e-12,
                             src_width=40e-12, rlc=rlc)


@pytest.mark.parametrize("shape", [(2, 6, 5), (3, 9, 8), (1, 7, 9), (4, 5, 70)])
def test_dc_matches_dense_solve(pgb, shape):
    g = grid(shape, sum(shape))
    t = 20e-12
    G = pgb.Grid.from_mesh_grid(g)
    st = G.dc(t=t, tol=1e-15, omega=1.7, max_sweeps=2_000_000)
    V = G.voltages()
    G.close()
    nl = netlist.from_mesh(g)
    Vd = dense.dc_solve(nl, pwl.node_currents(nl, t))
    assert np.abs(Vd - 1.0).max() > 1e-6
    np.testing.assert_allclose(V, Vd, rtol=0, atol=1e-9)
    assert st.sweeps_total > 0


def test_dc_rlc_matches_oracle_element(pgb):
    g = grid((3, 6, 7), 5, rlc=True)
    t = 20e-12
    G = pgb.Grid.from_mesh_grid(g)
    G.dc(t=t, tol=1e-15, omega=1.7, max_sweeps=2_000_000)
    V = G.voltages()
    G.close()
    nl = netlist.from_mesh(g, series_rl="element")
    It = np.stack([pwl.node_currents(nl, 0.0), pwl.node_currents(nl, t)])
    ro = nodal.NodalOracle(nl).transient(1e300, 1, tol=1e-15, omega=1.7, Itab=It)
    assert ro.status == 0
    np.testing.assert_allclose(V, ro.V[1], rtol=0, atol=1e-9)


def test_dc_needs_a_conductive_path(pgb):
    # node 1 of a 1 x 1 x 2 mesh is cut off (gx = 0) and has no pad: in DC its
    # diagonal sum of conductances is 0 (Lemma 1's irreducibility fails)
    P = pgb
    z = np.zeros((1, 1, 2))
    G = P.Grid.mesh(1, 1, 2, z.copy(), z.copy(), z.copy(), np.full((1, 1, 2), 1e-15),
                    np.array([0]), np.array([10.0]), 1.0)
    with pytest.raises(P.PgError):
        G.dc(t=0.0, tol=1e-12, omega=1.5, max_sweeps=10)
    # the transient is fine: C/h keeps the diagonal positive
    r = G.transient(1e-12, 2, tol=1e-12, omega=1.5)
    assert r.status == 0
    G.close()


@pytest.mark.parametrize("shape,h", [((2, 12, 10), 10e-12), ((3, 20, 16), 5e-12), ((1, 30, 30), 20e-12)])
def test_estimate_omega_matches_dense_spectrum(pgb, shape, h):
    g = grid(shape, 7 + sum(shape))
    nl = netlist.from_mesh(g)
    M = dense.system(nl, h)["M"]
    J = np.eye(M.shape[0]) - M / np.diag(M)[:, None]
    rho = float(np.max(np.abs(np.linalg.eigvals(J))))
    G = pgb.Grid.from_mesh_grid(g)
    r_est, om = G.estimate_omega(h, sweeps=4000)
    assert abs(r_est - rho) <= 2e-3 * max(1.0, 1 - rho) + 1e-4, (r_est, rho)
    assert abs(om - 2.0 / (1.0 + np.sqrt(1.0 - r_est ** 2))) < 1e-12 or om == 1.999
    # the estimate leaves the grid usable, and Young's omega beats Gauss-Seidel
    r1 = G.transient(h, 3, tol=1e-12, omega=1.0, max_sweeps=1_000_000)
    r2 = G.transient(h, 3, tol=1e-12, omega=om, max_sweeps=1_000_000)
    G.close()
    assert r2.stats.sweeps_total < r1.stats.sweeps_total


def test_tune_omega_picks_fewest_sweeps_and_resets(pgb):
    # pg_tune_omega: candidate 0 is Young's omega_b, the pick is the candidate
    # with the fewest sweeps over the first steps, and the grid is left at x(0)
    g = gridgen.config_grid(1, dims=(2, 96, 128), steps=6)
    G = pgb.Grid.from_mesh_grid(g, device=True)
    G.set_option("resident", 0)
    rho, omb = G.estimate_omega(g.h, 2000)
    om, sw = G.tune_omega(g.h, steps=4, tol=1e-10, n=5, d_omega=0.002)
    cands = [min(omb + k * 0.002, 1.999) for k in range(5)]
    assert min(abs(om - c) for c in cands) < 1e-15
    assert sw[cands.index(min(cands, key=lambda c: abs(c - om)))] == sw.min()
    r0 = G.transient(g.h, 4, tol=1e-10, omega=cands[0], max_sweeps=200000)
    assert int(r0.stats.sweeps_total) == sw[0]
    # left at x(0): a continuation from here equals a fresh transient
    G2 = pgb.Grid.from_mesh_grid(g, device=True)
    G2.set_option("resident", 0)
    G2.tune_omega(g.h, steps=2, tol=1e-10, n=2, d_omega=0.002)
    a = G2.transient(g.h, 3, tol=1e-10, omega=om, max_sweeps=200000, cont=True, probes=np.arange(g.n))
    b = G.transient(g.h, 3, tol=1e-10, omega=om, max_sweeps=200000, probes=np.arange(g.n))
    np.testing.assert_array_equal(a.probes, b.probes)
    G.close()
    G2.close()
