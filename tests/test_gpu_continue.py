"""pg_transient_continue / pg_group_transient_continue (-m gpu): a transient
cut into consecutive calls equals one call over all its steps bit for bit
(Algorithm 1: the time loop carries only V and the inductor
currents), on every sweep path (cluster-resident, two-sweep pipeline,
generic fused, CSR, RLC, slab groups); plus the fused RHS kernel's NaN / Inf
check (PG_ENONFINITE) and the continuation's argument checks."""
import numpy as np
import pytest

import gridgen

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
    return gridgen.mesh_grid(L, NY, NX, seed=seed, pad_pitch=3, src_frac=0.5, h=10e-12 if not rlc else 2e-12,
                             src_start=20e-12, src_width=40e-12, rlc=rlc)


def grid_of(P, g, options):
    G = P.Grid.from_mesh_grid(g, device=True) if hasattr(g, "gx") else P.Grid.from_edge_grid(g, device=True)
    for k, v in options.items():
        G.set_option(k, v)
    return G


CASES = [
    ("resident", lambda: mk(2, 20, 30, 1), {"resident": 1}),
    ("pipe", lambda: mk(4, 40, 150, 2), {"resident": 0}),
    ("fused_F3", lambda: mk(3, 33, 31, 3), {"resident": 0, "fuse": 3}),
    ("rlc", lambda: mk(4, 24, 70, 4, rlc=True), {"resident": 0}),
    ("csr", lambda: gridgen.edge_grid(2, 20, 18, seed=5, h=10e-12, src_start=20e-12, src_width=40e-12,
                                      src_frac=0.5, pad_pitch=4), {}),
    ("jacobi", lambda: mk(2, 10, 12, 6), {"resident": 0}),
]


@pytest.mark.parametrize("name,make,options", CASES, ids=[c[0] for c in CASES])
def test_continue_equals_one_call(pgb, name, make, options):
    g = make()
    method = "jacobi" if name == "jacobi" else "rbsor"
    tol, omega = (1e-9, 0.9) if method == "jacobi" else (1e-11, 1.6)
    pr = np.arange(g.n, dtype=np.int64)
    A = grid_of(pgb, g, options)
    ra = A.transient(g.h, 9, tol=tol, omega=omega, method=method, probes=pr)
    VA = A.voltages()
    B = grid_of(pgb, g, options)
    parts, sweeps = [], [0]
    for k, n in enumerate((2, 3, 4)):
        r = B.transient(g.h, n, tol=tol, omega=omega, method=method, probes=pr, cont=k > 0)
        parts.append(r.probes[1:])
        sweeps += list(r.sweeps[1:])
    np.testing.assert_array_equal(np.concatenate(parts), ra.probes[1:])
    np.testing.assert_array_equal(np.array(sweeps), ra.sweeps)
    np.testing.assert_array_equal(B.voltages(), VA)
    # a fresh pg_transient restarts from x(0)
    rb = B.transient(g.h, 9, tol=tol, omega=omega, method=method, probes=pr)
    np.testing.assert_array_equal(rb.probes, ra.probes)
    A.close()
    B.close()


def test_continue_from_set_voltages_and_dc(pgb):
    g = mk(3, 21, 40, 7)
    pr = np.arange(g.n, dtype=np.int64)
    A = grid_of(pgb, g, {"resident": 0})
    B = grid_of(pgb, g, {"resident": 0})
    v0 = 1.0 - 1e-3 * np.random.default_rng(0).random(g.n)
    A.set_voltages(v0)
    B.set_voltages(v0)
    ra = A.transient(g.h, 4, tol=1e-11, omega=1.6, probes=pr)
    rb = B.transient(g.h, 4, tol=1e-11, omega=1.6, probes=pr, cont=True)   # s0 = 0: same as from x(0)
    np.testing.assert_array_equal(ra.probes, rb.probes)
    # after pg_dc the state is the DC operating point at t = 0
    B.dc(t=0.0, tol=1e-12, omega=1.9)
    vdc = B.voltages()
    rc = B.transient(g.h, 2, tol=1e-11, omega=1.6, probes=pr, cont=True)
    np.testing.assert_array_equal(rc.probes[0], vdc)
    A.close()
    B.close()


def test_continue_rejects_other_h(pgb):
    g = mk(2, 10, 12, 8)
    G = grid_of(pgb, g, {})
    G.transient(g.h, 2, tol=1e-11, omega=1.5)
    with pytest.raises(pgb.PgError):
        G.transient(2 * g.h, 2, tol=1e-11, omega=1.5, cont=True)
    G.transient(g.h, 2, tol=1e-11, omega=1.5, cont=True)
    G.close()


@pytest.mark.parametrize("transport", ["copy", "p2p"])
def test_group_continue_equals_one_call(pgb, transport):
    g = mk(4, 48, 70, 9)
    grpA = pgb.SlabGroup.local(g, 3, fuse=2, transport=transport)
    ra = grpA.transient(g.h, 7, tol=1e-11, omega=1.6)
    VA = grpA.owned_voltages(g)
    grpB = pgb.SlabGroup.local(g, 3, fuse=2, transport=transport)
    sw = [0]
    for k, n in enumerate((3, 4)):
        r = grpB.transient(g.h, n, tol=1e-11, omega=1.6, cont=k > 0)
        sw += list(r.sweeps[1:])
    VB = grpB.owned_voltages(g)
    np.testing.assert_array_equal(np.array(sw), ra.sweeps)
    for (sa, va), (sb, vb) in zip(VA, VB):
        np.testing.assert_array_equal(va, vb)
    grpA.close()
    grpB.close()


def test_rhs_kernel_flags_nonfinite_iterates(pgb):
    # two finite loads of 1.7e308 A on one node overflow the right-hand side
    # to -inf: the fused RHS kernel's check of V(t) reports PG_ENONFINITE
    g = mk(2, 16, 20, 10)
    G = grid_of(pgb, g, {"resident": 0})
    G.set_sources(np.array([37, 37]), np.array([0, 1, 2]), np.array([0.0, 0.0]), np.array([1.7e308, 1.7e308]))
    with pytest.raises(pgb.PgError) as e:
        G.transient(g.h, 3, tol=1e-10, omega=1.5, max_sweeps=50)
    assert e.value.code == -6
    G.close()


@pytest.mark.parametrize("device", [False, True])
def test_set_voltages_must_be_finite(pgb, device):
    # host and device inputs are value-checked on the device before the grid's
    # state changes: a rejected call leaves V where it was
    import torch
    g = mk(2, 16, 20, 12)
    G = grid_of(pgb, g, {"resident": 0})
    v0 = np.linspace(0.9, 1.0, g.n)
    G.set_voltages(v0)
    bad = v0.copy()
    bad[37] = np.nan if device else np.inf
    with pytest.raises(pgb.PgError) as e:
        G.set_voltages(torch.from_numpy(bad).cuda() if device else bad)
    assert e.value.code == -1 and "finite" in str(e.value)
    np.testing.assert_array_equal(G.voltages(), v0)
    G.close()


def test_host_sources_must_be_finite(pgb):
    g = mk(2, 6, 5, 11)
    G = grid_of(pgb, g, {})
    with pytest.raises(pgb.PgError):
        G.set_sources(np.array([3]), np.array([0, 2]), np.array([0.0, np.nan]), np.array([0.0, 1e-3]))
    with pytest.raises(pgb.PgError):
        G.set_sources(np.array([3]), np.array([0, 1]), np.array([0.0]), np.array([np.inf]))
    G.close()
