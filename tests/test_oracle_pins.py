"""Pins for the oracle (-m "not gpu"): the oracle checked against things other
than itself - closed forms, hand-evaluated fixtures (tests/golden), dense
Cholesky solves of the incidence-matrix assembly, Lemma 1's conditions,
textbook linear algebra definitions of a Gauss-Seidel / SOR / Jacobi sweep,
invariants, and brute force on tiny inputs."""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

import gridgen
from oracle import dense, kcl, netlist, nodal, pwl
from oracle.netlist import GROUND, Netlist, src

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def E(*a):
    return np.array(a, dtype=np.int64)


def F(*a):
    return np.array(a, dtype=np.float64)


def tiny_netlist(n, R=(), C=(), L=(), I=(), vd=(1.0,)):
    """R/C/L: tuples (a, b, value); I: (a, b, [(t, i), ...])."""
    def cols(lst, k):
        return [x[k] for x in lst]
    it, ii, ptr = [], [], [0]
    for a, b, pts in I:
        for t, v in pts:
            it.append(t); ii.append(v)
        ptr.append(len(it))
    return Netlist(
        n=n, vd=F(*vd),
        ra=E(*cols(R, 0)), rb=E(*cols(R, 1)), rg=F(*cols(R, 2)),
        ca=E(*cols(C, 0)), cb=E(*cols(C, 1)), cv=F(*cols(C, 2)),
        la=E(*cols(L, 0)), lb=E(*cols(L, 1)), lv=F(*cols(L, 2)),
        ia=E(*cols(I, 0)), ib=E(*cols(I, 1)), iptr=E(*ptr), it=F(*it), ii=F(*ii), n_mesh=n)


def small_grids():
    out = []
    for seed, (L, NY, NX) in enumerate([(2, 6, 5), (1, 7, 9), (3, 4, 4), (2, 1, 9), (1, 1, 1), (4, 3, 5)]):
        g = gridgen.mesh_grid(L, NY, NX, seed=seed, pad_pitch=2, src_frac=0.5, h=10e-12,
                              src_start=30e-12, src_width=40e-12)
        out.append(g)
    return out


def small_rlc_grids():
    out = []
    for seed, (L, NY, NX) in enumerate([(2, 4, 5), (3, 3, 3), (2, 1, 6)]):
        g = gridgen.mesh_grid(L, NY, NX, seed=100 + seed, pad_pitch=2, src_frac=0.5, rlc=True,
                              h=2e-12, src_start=10e-12, src_width=20e-12)
        out.append(g)
    return out


# --------------------------------------------------------------------- closed forms
def test_single_node_rc_golden():
    gd = gold("single_node_rc.json")
    nl = tiny_netlist(1, R=[(0, src(0), gd["g"])], C=[(0, GROUND, gd["C"])], vd=(gd["vdd"],))
    steps = len(gd["x_num"]) - 1
    It = np.zeros((steps + 1, 1))
    expect = np.array(gd["x_num"], float) / np.array(gd["x_den"], float)
    o = nodal.NodalOracle(nl)
    for method in ("gs", "jacobi"):
        r = o.transient(gd["h"], steps, tol=1e-15, Itab=It, V0=F(gd["x0"]), method=method)
        assert r.status == 0
        np.testing.assert_allclose(r.V[:, 0], expect, rtol=0, atol=1e-15)
    V, _ = dense.direct_companion(nl, gd["h"], steps, It, F(gd["x0"]))
    np.testing.assert_allclose(V[:, 0], expect, rtol=0, atol=1e-15)


def test_backward_euler_first_order_accuracy():
    # SPEC acceptance 6: analytic RC charging V(t) = Vdd (1 - exp(-g t / C));
    # BE error halves when h halves (first order).
    g, C = 2.0, 3e-12
    T = 5 * C / g
    nl = tiny_netlist(1, R=[(0, src(0), g)], C=[(0, GROUND, C)])
    errs = []
    for steps in (100, 200):
        h = T / steps
        r = nodal.NodalOracle(nl).transient(h, steps, tol=1e-15, Itab=np.zeros((steps + 1, 1)), V0=F(0.0))
        t = np.arange(steps + 1) * h
        errs.append(np.max(np.abs(r.V[:, 0] - (1 - np.exp(-g * t / C)))))
    assert 1.7 <= errs[0] / errs[1] <= 2.3


def test_chain_dc_golden():
    gd = gold("chain_dc.json")
    g = gd["g"]
    # DC = transient with no capacitance: (C/h + G) -> G (Eq. (2) with C = 0 is Eq. (3))
    nl = tiny_netlist(2, R=[(0, src(0), g), (0, 1, g)], C=[(0, GROUND, 0.0), (1, GROUND, 0.0)],
                      I=[(1, GROUND, [(0.0, gd["load"])])], vd=(gd["vdd"],))
    o = nodal.NodalOracle(nl)
    It = pwl.node_currents_table(nl, 1.0, 1)
    r = o.transient(1.0, 1, tol=1e-15, Itab=It, V0=F(1.0, 1.0))
    np.testing.assert_allclose(r.V[1], gd["V"], atol=1e-13)
    np.testing.assert_allclose(dense.dc_solve(nl, It[0]), gd["V"], atol=1e-13)


def test_stencil_diag_golden():
    gd = gold("stencil_diag.json")
    for c in gd["cases"]:
        R = [(0, src(0), c["g"])] if c["g"] else []
        L = [(0, src(0), c["L"])] if c["L"] else []
        nl = tiny_netlist(1, R=R, L=L, C=[(0, GROUND, c["C"])])
        d = nodal.NodalOracle(nl).diag(c["h"])
        assert d[0] == pytest.approx(c["d"], rel=1e-14)


def test_rlc_ringing_period():
    gd = gold("rlc_ringing.json")
    R, Lv, C, vdd = gd["R"], gd["L"], gd["C"], gd["vdd"]
    wd = math.sqrt(1 / (Lv * C) - (R / (2 * Lv)) ** 2)
    period = 2 * math.pi / wd
    h = period / 200
    steps = 800
    # nodes: 0 = m (between R and L), 1 = n (capacitor node)
    nl = tiny_netlist(2, R=[(src(0), 0, 1.0 / R)], L=[(0, 1, Lv)], C=[(1, GROUND, C)], vd=(vdd,))
    It = np.zeros((steps + 1, 2))
    r = nodal.NodalOracle(nl).transient(h, steps, tol=1e-14, Itab=It, V0=F(vdd, 0.0))
    assert r.status == 0
    x = r.V[:, 1] - vdd
    zc = np.flatnonzero(np.sign(x[1:]) != np.sign(x[:-1]))
    # linear interpolation of crossing times
    tz = [(k + x[k] / (x[k] - x[k + 1])) * h for k in zc]
    half = np.diff(tz)
    assert len(half) >= 4
    assert abs(np.mean(half) - period / 2) <= gd["period_tolerance"] * period / 2
    # and the dense Eq. (10) solve agrees with the nodal iteration
    V, _ = dense.direct_companion(nl, h, steps, It, F(vdd, 0.0))
    np.testing.assert_allclose(r.V, V, atol=1e-9)


def test_pwl_triangle():
    t = F(1.0, 2.0, 3.0)
    i = F(0.0, 5.0, 0.0)
    assert pwl.eval_source(t, i, 0.0) == 0.0
    assert pwl.eval_source(t, i, 1.5) == 2.5
    assert pwl.eval_source(t, i, 2.0) == 5.0
    assert pwl.eval_source(t, i, 2.5) == 2.5
    assert pwl.eval_source(t, i, 9.0) == 0.0
    g = gridgen.mesh_grid(1, 3, 3, seed=1, src_frac=1.0, pad_pitch=1)
    nl = netlist.from_mesh(g)
    tab = pwl.node_currents_table(nl, 7e-12, 100)
    for s in (0, 13, 57, 100):
        np.testing.assert_array_equal(tab[s], pwl.node_currents(nl, s * 7e-12))


# ------------------------------------------------------------ matrices / Lemma 1
@pytest.mark.parametrize("h", [1e-13, 1e-12, 1e-11])
def test_lemma1_pd(h):
    for g in small_grids()[:4] + small_rlc_grids():
        nl = netlist.from_mesh(g)
        rep = dense.check_pd(dense.system(nl, h)["M"])
        assert rep["symmetric"] and rep["weakly_dd"] and rep["irreducible"] and rep["pd"], rep
        assert rep["n_strict"] >= 1


def test_lemma1_detects_violations():
    # a node attached only through a current source: zero row -> not PD
    nl = tiny_netlist(2, R=[(0, src(0), 1.0)], C=[(0, GROUND, 1.0), (1, GROUND, 0.0)],
                      I=[(1, GROUND, [(0.0, 1.0)])])
    rep = dense.check_pd(dense.system(nl, 1.0)["M"])
    assert not rep["pd"]
    # Fig. 1: two clusters joined only through the source node -> reducible
    nl = tiny_netlist(2, R=[(0, src(0), 1.0), (1, src(0), 1.0)], C=[(0, GROUND, 1.0), (1, GROUND, 1.0)])
    rep = dense.check_pd(dense.system(nl, 1.0)["M"])
    assert rep["n_components"] == 2 and not rep["irreducible"] and rep["pd"]


def test_stencil_equals_system_matrix():
    # per-node Eq. (14) coefficients (oracle C code) == incidence-matrix M (Eq. (11))
    for g in small_grids() + small_rlc_grids():
        nl = netlist.from_mesh(g)
        h = g.h
        M = dense.system(nl, h)["M"]
        o = nodal.NodalOracle(nl)
        d = o.diag(h)
        Ls = o.L
        Ms = np.diag(d)
        for i in range(nl.n):
            for k in range(Ls.rptr[i], Ls.rptr[i + 1]):
                if Ls.rnbr[k] >= 0:
                    Ms[i, Ls.rnbr[k]] -= Ls.rg[k]
            for k in range(Ls.lptr[i], Ls.lptr[i + 1]):
                if Ls.lnbr[k] >= 0:
                    Ms[i, Ls.lnbr[k]] -= h / Ls.lval[k]
        np.testing.assert_allclose(Ms, M, rtol=1e-14, atol=1e-14 * np.abs(M).max())


def test_system_matrix_linear_in_h():
    g = small_rlc_grids()[0]
    nl = netlist.from_mesh(g)
    h1, h2 = 1e-12, 3e-12
    S1, S2 = dense.system(nl, h1), dense.system(nl, h2)
    np.testing.assert_allclose(S1["M"] - S2["M"], (1 / h1 - 1 / h2) * S1["C"] + (h1 - h2) * S1["L"],
                               atol=1e-9 * np.abs(S1["M"]).max())


# ---------------------------------------------------------------- sweep definitions
def _split(M, order):
    P = np.eye(M.shape[0])[order]
    Mp = P @ M @ P.T
    D = np.diag(np.diag(Mp))
    El = -np.tril(Mp, -1)
    Fu = -np.triu(Mp, 1)
    return P, D, El, Fu


@pytest.mark.parametrize("omega", [1.0, 0.7, 1.6])
@pytest.mark.parametrize("order_kind", ["natural", "redblack", "random"])
def test_sweep_is_sor_triangular_solve(omega, order_kind):
    g = small_grids()[0]
    nl = netlist.from_mesh(g)
    h = g.h
    o = nodal.NodalOracle(nl)
    n = nl.n
    rng = np.random.default_rng(3)
    order = {"natural": np.arange(n), "redblack": nodal.red_black_order(g.layers, g.ny, g.nx),
             "random": rng.permutation(n)}[order_kind]
    M = dense.system(nl, h)["M"]
    b = rng.normal(size=n)
    x0 = rng.normal(size=n)
    x1, _ = o.sweep(h, o.diag(h), b, x0, omega=omega, order=order)
    # textbook SOR: (D - w E) x1 = (w F + (1 - w) D) x0 + w b in the permuted numbering
    P, D, El, Fu = _split(M, order)
    y = sla.solve_triangular(D - omega * El, (omega * Fu + (1 - omega) * D) @ (P @ x0) + omega * (P @ b),
                             lower=True)
    np.testing.assert_allclose(P.T @ y, x1, rtol=1e-12, atol=1e-12)


def test_jacobi_sweep_definition():
    g = small_grids()[2]
    nl = netlist.from_mesh(g)
    h = g.h
    o = nodal.NodalOracle(nl)
    M = dense.system(nl, h)["M"]
    rng = np.random.default_rng(5)
    b, x0 = rng.normal(size=nl.n), rng.normal(size=nl.n)
    for w in (1.0, 0.8):
        x1, dm = o.sweep(h, o.diag(h), b, x0, omega=w, method="jacobi")
        D = np.diag(M)
        ref = w * (b - (M - np.diag(D)) @ x0) / D + (1 - w) * x0
        np.testing.assert_allclose(x1, ref, rtol=1e-12, atol=1e-12)
        assert dm == pytest.approx(np.abs(ref - x0).max(), rel=1e-12)


def test_omega_one_is_plain_gauss_seidel():
    g = small_grids()[1]
    nl = netlist.from_mesh(g)
    o = nodal.NodalOracle(nl)
    rng = np.random.default_rng(9)
    b, x0 = rng.normal(size=nl.n), rng.normal(size=nl.n)
    d = o.diag(g.h)
    x1, _ = o.sweep(g.h, d, b, x0, omega=1.0)
    # plain GS written out in Python (Eq. (13) literally)
    Ls = o.L
    x = x0.copy()
    for i in range(nl.n):
        s = b[i]
        for k in range(Ls.rptr[i], Ls.rptr[i + 1]):
            if Ls.rnbr[k] >= 0:
                s += Ls.rg[k] * x[Ls.rnbr[k]]
        x[i] = s / d[i]
    np.testing.assert_array_equal(x, x1)


# ------------------------------------------------------- transients vs direct solves
def _v0(nl):
    return np.full(nl.n, nl.vd[0])


@pytest.mark.parametrize("order_kind", ["natural", "redblack"])
def test_rc_nodal_matches_cholesky(order_kind):
    for g in small_grids():
        nl = netlist.from_mesh(g)
        steps = 12
        It = pwl.node_currents_table(nl, g.h, steps)
        V, _ = dense.direct_companion(nl, g.h, steps, It, _v0(nl))
        order = None if order_kind == "natural" else nodal.red_black_order(g.layers, g.ny, g.nx)
        r = nodal.NodalOracle(nl).transient(g.h, steps, tol=1e-13, omega=1.5, Itab=It, order=order)
        assert r.status == 0
        np.testing.assert_allclose(r.V, V, rtol=0, atol=1e-9)


def test_rlc_nodal_matches_cholesky():
    for g in small_rlc_grids():
        nl = netlist.from_mesh(g)
        steps = 15
        It = pwl.node_currents_table(nl, g.h, steps)
        V, il = dense.direct_companion(nl, g.h, steps, It, _v0(nl))
        assert np.abs(V - 1).max() > 1e-6      # the loads do something
        r = nodal.NodalOracle(nl).transient(g.h, steps, tol=1e-14, omega=1.8, Itab=It)
        assert r.status == 0
        np.testing.assert_allclose(r.V, V, rtol=0, atol=1e-9)
        np.testing.assert_allclose(r.il, il, rtol=0, atol=1e-7 * max(1.0, np.abs(il).max()))


def test_companion_equals_second_order_form():
    # Eq. (10) (inductor currents as state) and Eq. (11) (second-order
    # recurrence) are the same discretisation: equal under exact solves.
    for g in small_rlc_grids():
        nl = netlist.from_mesh(g)
        steps = 60
        It = pwl.node_currents_table(nl, g.h, steps)
        V, _ = dense.direct_companion(nl, g.h, steps, It, _v0(nl))
        V2 = dense.direct_second_order(nl, g.h, steps, It, V[0], V[1])
        np.testing.assert_allclose(V2, V, atol=1e-10)
        # the nodal Eq. (14) iteration agrees with the dense Eq. (11) solve
        r = nodal.NodalOracle(nl).transient(g.h, 20, tol=1e-15, omega=1.8, Itab=It[:21],
                                            form="second_order", V1=V[1], max_sweeps=200000)
        np.testing.assert_allclose(r.V, V2[:21], atol=1e-9)


def test_series_rl_is_eliminated_internal_node():
    # A series R-L branch (reading R7) modelled with an internal node m (the
    # paper's element-wise branches) equals the backward-Euler series element
    # i(t+h) = (v(t+h) + (L/h) i(t)) / (R + L/h) -- a Schur complement of M.
    R, Lv, C, h, g1 = 0.2, 0.5e-12, 5e-15, 2e-12, 1.3
    # nodes: 0 = a (layer node), 1 = m (internal), 2 = c (other layer node); pads keep M PD
    nl = tiny_netlist(3, R=[(0, 1, 1 / R), (0, src(0), g1), (2, src(0), g1)], L=[(1, 2, Lv)],
                      C=[(0, GROUND, C), (1, GROUND, 0.0), (2, GROUND, C)],
                      I=[(2, GROUND, [(0.0, 0.0), (10e-12, 1e-3)])])
    steps = 12
    It = pwl.node_currents_table(nl, h, steps)
    V, _ = dense.direct_companion(nl, h, steps, It, F(1.0, 1.0, 1.0))
    # eliminated two-node model
    ge = 1.0 / (R + Lv / h)
    alpha = (Lv / h) * ge
    va, vc, i = 1.0, 1.0, 0.0
    for s in range(1, steps + 1):
        A = np.array([[C / h + g1 + ge, -ge], [-ge, C / h + g1 + ge]])
        b = np.array([C / h * va + g1 - alpha * i, C / h * vc + g1 + alpha * i - It[s, 2]])
        va, vc = np.linalg.solve(A, b)
        i = ge * (va - vc) + alpha * i
        assert abs(va - V[s, 0]) < 1e-12 and abs(vc - V[s, 2]) < 1e-12


def test_series_rl_element_matches_internal_node_cholesky():
    # the oracle's series R-L element (netlist series_rl="element", one inductor
    # branch with series resistance) against the dense Cholesky solve of the
    # paper's element-wise model with internal nodes (series_rl="node"):
    # same voltages at the grid nodes, same branch currents
    for g in small_rlc_grids():
        nl_node = netlist.from_mesh(g, series_rl="node")
        nl_el = netlist.from_mesh(g, series_rl="element")
        assert nl_el.n == g.n and nl_node.n > g.n and np.all(nl_el.lr > 0)
        steps = 15
        V, il = dense.direct_companion(nl_node, g.h, steps,
                                       pwl.node_currents_table(nl_node, g.h, steps), _v0(nl_node))
        It = pwl.node_currents_table(nl_el, g.h, steps)
        for order in (None, nodal.red_black_order(g.layers, g.ny, g.nx)):
            r = nodal.NodalOracle(nl_el).transient(g.h, steps, tol=1e-15, omega=1.7, Itab=It,
                                                   order=order)
            assert r.status == 0
            np.testing.assert_allclose(r.V, V[:, :g.n], rtol=0, atol=1e-10)
            np.testing.assert_allclose(r.il, il, rtol=0, atol=1e-8 * max(1.0, np.abs(il).max()))
            # KCL at every grid node with the series element's companion current
            il_prev = np.zeros(nl_el.la.size)
            for s in range(1, steps + 1):
                res = kcl.residual(nl_el, g.h, r.V[s], r.V[s - 1], It[s], il_prev)
                assert np.abs(res).max() <= 1e-9
                il_prev = kcl.inductor_currents_next(nl_el, g.h, r.V[s], il_prev)


def test_series_rl_element_rejected_where_unsupported():
    g = small_rlc_grids()[0]
    nl = netlist.from_mesh(g, series_rl="element")
    with pytest.raises(ValueError):
        dense.system(nl, g.h)
    with pytest.raises(ValueError):
        nodal.NodalOracle(nl).transient(g.h, 3, form="second_order", V1=_v0(nl))
    with pytest.raises(ValueError):
        netlist.from_mesh(g, series_rl="bogus")


def test_zero_current_invariant():
    for g in small_grids()[:3] + small_rlc_grids()[:2]:
        g.sources = gridgen.Sources(node=np.zeros(0, np.int64), ptr=np.zeros(1, np.int64),
                                    t=np.zeros(0), i=np.zeros(0))
        nl = netlist.from_mesh(g)
        r = nodal.NodalOracle(nl).transient(g.h, 20, tol=1e-12, omega=1.3)
        assert np.abs(r.V - nl.vd[0]).max() <= 1e-13   # rounding of sum(g)/d only
        assert np.all(r.sweeps[1:] == 1)


def test_kcl_residual_converged():
    for g in small_grids()[:3] + small_rlc_grids()[:2]:
        nl = netlist.from_mesh(g)
        steps = 10
        It = pwl.node_currents_table(nl, g.h, steps)
        r = nodal.NodalOracle(nl).transient(g.h, steps, tol=1e-13, omega=1.5, Itab=It)
        il = np.zeros(nl.la.size)
        for s in range(1, steps + 1):
            res = kcl.residual(nl, g.h, r.V[s], r.V[s - 1], It[s], il)
            assert np.abs(res).max() <= 1e-9
            il = kcl.inductor_currents_next(nl, g.h, r.V[s], il)
        # an unconverged iterate violates it (the check has teeth)
        bad = r.V[5].copy()
        bad[nl.n // 2] += 1e-6
        assert np.abs(kcl.residual(nl, g.h, bad, r.V[4], It[5],
                                   None if nl.la.size == 0 else np.zeros(nl.la.size))).max() > 1e-9


@pytest.mark.parametrize("omega", [0.5, 1.0, 1.5, 1.9])
def test_sor_converges_for_omega_in_0_2(omega):
    g = small_grids()[0]
    nl = netlist.from_mesh(g)
    steps = 6
    It = pwl.node_currents_table(nl, g.h, steps)
    V, _ = dense.direct_companion(nl, g.h, steps, It, _v0(nl))
    r = nodal.NodalOracle(nl).transient(g.h, steps, tol=1e-14, omega=omega, Itab=It)
    assert r.status == 0
    np.testing.assert_allclose(r.V, V, atol=1e-9)


def test_jacobi_transient_matches():
    g = small_grids()[3]
    nl = netlist.from_mesh(g)
    steps = 6
    It = pwl.node_currents_table(nl, g.h, steps)
    V, _ = dense.direct_companion(nl, g.h, steps, It, _v0(nl))
    r = nodal.NodalOracle(nl).transient(g.h, steps, tol=1e-14, omega=1.0, Itab=It, method="jacobi")
    assert r.status == 0
    np.testing.assert_allclose(r.V, V, atol=1e-9)


def test_edge_grid_spanning_and_deletion():
    g = gridgen.edge_grid(2, 24, 20, seed=4, pad_pitch=8)
    nl = netlist.from_edges(g)
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    n = g.n
    A = coo_matrix((np.ones(g.eu.size), (g.eu, g.ev)), shape=(n, n))
    assert connected_components(A, directed=False)[0] == 1
    full = 2 * (24 * 19 + 23 * 20)
    in_layer = int(np.sum((g.ev - g.eu) != 24 * 20))
    assert abs(in_layer - 0.8 * full) <= 1
    steps = 5
    It = pwl.node_currents_table(nl, g.h, steps)
    V, _ = dense.direct_companion(nl, g.h, steps, It, _v0(nl))
    r = nodal.NodalOracle(nl).transient(g.h, steps, tol=1e-13, omega=1.6, Itab=It)
    np.testing.assert_allclose(r.V, V, atol=1e-9)


# ------------------------------------------------ round 2: oracle plumbing pins
def test_group_counting_sort_equals_stable_argsort():
    # oracle_group (plain-C counting sort used for full-size node lists) equals
    # the stable-argsort grouping on random branch lists with ground / source ends
    rng = np.random.default_rng(5)
    for n, m in [(1, 0), (1, 3), (5, 7), (60, 400), (300, 50)]:
        a = rng.integers(-4, n, m)
        b = rng.integers(-4, n, m)
        v = rng.random(m)
        want = netlist._group_numpy(n, a, b, v)
        got = netlist.group(n, a, b, v)
        for x, y in zip(want, got):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("cfg,series_rl", [(1, "node"), (3, "element"), (3, "node"), (2, "node")])
def test_transient_cut_at_step_boundaries_is_identical(cfg, series_rl):
    # Algorithm 1's time loop carries only V and the inductor currents: the
    # step-by-step chaining tools/make_golden_fullsize.py uses (V(s-1), i_L(s-1)
    # and the load rows I((s-1)h), I(sh) passed in) reproduces one call bit for bit
    g = gridgen.config_grid(cfg, dims=(2, 12, 14), steps=6)
    nl = netlist.from_grid(g, series_rl)
    o = nodal.NodalOracle(nl)
    order = nodal.red_black_order(g.layers, g.ny, g.nx) if nl.n == g.n else None
    It = pwl.node_currents_table(nl, g.h, 6)
    r = o.transient(g.h, 6, tol=1e-11, omega=1.6, order=order, Itab=It, trace=True)
    V, il = np.full(nl.n, 1.0), np.zeros(nl.la.size)
    for s in range(1, 7):
        It2 = np.stack([pwl.node_currents_at(nl, (s - 1) * g.h), pwl.node_currents_at(nl, s * g.h)])
        q = o.transient(g.h, 1, tol=1e-11, omega=1.6, order=order, Itab=It2, V0=V, il0=il, trace=True)
        V, il = q.V[1].copy(), q.il.copy()
        assert np.array_equal(V, r.V[s]) and q.sweeps[1] == r.sweeps[s]
        np.testing.assert_array_equal(q.dtrace[1], r.dtrace[s])
    np.testing.assert_array_equal(il, r.il)
    np.testing.assert_array_equal(It[3], pwl.node_currents(nl, 3 * g.h))


def test_stopping_record():
    # dtrace: the last sweep is the first below tol (Algorithm 1 line 8), the
    # sweep before it is not, and the continued sweeps are the sweeps the
    # oracle would have run next (checked by re-running with more sweeps)
    g = gridgen.config_grid(1, dims=(2, 10, 12), steps=3)
    nl = netlist.from_grid(g)
    o = nodal.NodalOracle(nl)
    It = pwl.node_currents_table(nl, g.h, 3)
    tol = 1e-9
    r = o.transient(g.h, 3, tol=tol, omega=1.5, Itab=It, trace=True)
    for s in range(1, 4):
        k = r.sweeps[s]
        assert r.dtrace[s, 1] < tol and (k == 1 or r.dtrace[s, 0] >= tol)
    # step 1 continued: fixed k + e sweeps reproduce the recorded norms
    k = int(r.sweeps[1])
    d = o.diag(g.h)
    kn = o.known_companion(g.h, np.full(nl.n, 1.0), It[1])
    V = np.full(nl.n, 1.0)
    norms = []
    for _ in range(k + 4):
        V, dm = o.sweep(g.h, d, kn, V, omega=1.5)
        norms.append(dm)
    np.testing.assert_array_equal(np.array(norms[k - 2:k + 4]) if k >= 2 else norms[k - 1:k + 4],
                                  r.dtrace[1] if k >= 2 else r.dtrace[1, 1:])


def test_check_every_is_line8_tested_every_f_sweeps():
    # check_every = F evaluates Algorithm 1 line 8 only after sweeps that are
    # multiples of F (R13): the first step stops at the first such sweep whose
    # norm is below tol, read off the paper-semantics run's stopping record
    g = gridgen.config_grid(0, dims=(2, 14, 16), steps=4)
    nl = netlist.from_grid(g)
    o = nodal.NodalOracle(nl)
    It = pwl.node_currents_table(nl, g.h, 4)
    order = nodal.red_black_order(g.layers, g.ny, g.nx)
    r1 = o.transient(g.h, 4, tol=1e-10, omega=1.8, order=order, Itab=It, trace=True)
    for F in (1, 2, 3):
        rF = o.transient(g.h, 4, tol=1e-10, omega=1.8, order=order, Itab=It, trace=True, check_every=F)
        k = int(r1.sweeps[1])
        norms = {k - 1: r1.dtrace[1, 0], k: r1.dtrace[1, 1]}
        norms.update({k + 1 + e: r1.dtrace[1, 2 + e] for e in range(4)})
        j = -(-k // F) * F
        while not norms[j] < 1e-10:
            j += F
        assert rF.sweeps[1] == j and np.all(rF.sweeps[1:] % F == 0)
        if F == 1:
            np.testing.assert_array_equal(rF.V, r1.V)


@pytest.mark.parametrize("rlc", [False, True])
def test_netlist_from_mesh_brute_force(rlc):
    # the oracle's branch list of a mesh (gridgen.mesh_to_edges + netlist.from_mesh)
    # against the PAPER.md §II-A element list written out node by node: an R
    # branch for every in-layer segment (l,y,x)-(l,y,x+1) / (l,y,x)-(l,y+1,x)
    # and every via (l,y,x)-(l+1,y,x) (R6, R16), a G0 branch from every pad
    # node to the Vdd source node, a capacitor to ground at every node and a
    # current source per load; RLC (R7, "node" model): a via or pad with
    # inductance is R to a new internal node, then L onward
    g = gridgen.mesh_grid(3, 4, 5, seed=4, pad_pitch=2, src_frac=0.5, h=2e-12, rlc=rlc)
    L, NY, NX = g.layers, g.ny, g.nx
    nid = lambda l, y, x: (l * NY + y) * NX + x                   # noqa: E731
    R, Lb = [], []
    nxt = g.n
    for l in range(L):
        for y in range(NY):
            for x in range(NX):
                if x + 1 < NX:
                    R.append((nid(l, y, x), nid(l, y, x + 1), float(g.gx[l, y, x])))
                if y + 1 < NY:
                    R.append((nid(l, y, x), nid(l, y + 1, x), float(g.gy[l, y, x])))
    for l in range(L - 1):
        for y in range(NY):
            for x in range(NX):
                a, b, gz = nid(l, y, x), nid(l + 1, y, x), float(g.gz[l, y, x])
                lz = 0.0 if g.lz is None else float(g.lz[l, y, x])
                if lz > 0:
                    R.append((a, nxt, gz))
                    Lb.append((nxt, b, lz))
                    nxt += 1
                else:
                    R.append((a, b, gz))
    for k in range(len(g.pad_node)):
        p, gp = int(g.pad_node[k]), float(g.pad_g[k])
        if g.pad_l is not None:
            R.append((p, nxt, gp))
            Lb.append((nxt, src(0), float(g.pad_l[k])))
            nxt += 1
        else:
            R.append((p, src(0), gp))
    nl = netlist.from_mesh(g)
    assert nl.n == nxt and nl.n_mesh == g.n
    got_r = sorted(zip(nl.ra.tolist(), nl.rb.tolist(), nl.rg.tolist()))
    assert got_r == sorted(R)
    got_l = sorted(zip(nl.la.tolist(), nl.lb.tolist(), nl.lv.tolist()))
    assert got_l == sorted(Lb)
    assert len(Lb) > 0 if rlc else len(Lb) == 0
    np.testing.assert_array_equal(nl.ca, np.arange(g.n))
    assert np.all(nl.cb == GROUND)
    np.testing.assert_array_equal(nl.cv, g.cap.reshape(-1))
    assert float(nl.vd[0]) == g.vdd
    np.testing.assert_array_equal(nl.ia, g.sources.node)
    assert np.all(nl.ib == GROUND)
