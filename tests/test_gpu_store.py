"""Store-construction and kernel edge cases (-m gpu):

* the staged CSR sweep (bulk-copied 256-row tiles) on irregular graphs whose
  colour classes start at unaligned rows, with several colours (greedy
  colouring of non-bipartite graphs), tiles of varying entry counts and a
  star node too large for the stage (whole-grid fallback): bit-identical to the
  one-thread-per-row kernel, and converged to the oracle's solution (natural
  order, tol 1e-13 on both sides: the same exact solution, R14);
* the fused RHS kernel on meshes with several loads and several pads on one
  node, loads with different breakpoint counts, loads and pads on nodes at the
  2048-element tile boundaries of the storage layout: fixed-sweep iterates
  equal to the oracle's (1e-12 V);
* the device-side load store: sources given in any order (unsorted, repeated
  nodes) give the same store as sorted input (bit-identical iterates);
* the device CSR builder (bipartite graphs, one or several components)
  against the host builder (PGB200_CSR_HOST=1), which also serves
  non-bipartite graphs:
  bit-identical iterates, host and device inputs.
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


def random_graph(n, extra, seed, star=0):
    """Connected random graph: a random spanning tree plus `extra` random
    branches (triangles make it non-bipartite), optionally a star node joined
    to `star` others; pads on every 50th node, loads on a third of the nodes."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    u = [perm[k] for k in range(1, n)]
    v = [perm[rng.integers(0, k)] for k in range(1, n)]
    a = rng.integers(0, n, extra)
    b = rng.integers(0, n, extra)
    u = np.concatenate([np.array(u, np.int64), a])
    v = np.concatenate([np.array(v, np.int64), b])
    if star:
        c = int(rng.integers(0, n))
        others = rng.choice(n, size=min(star, n - 1), replace=False)
        others = others[others != c]
        u = np.concatenate([u, np.full(others.size, c)])
        v = np.concatenate([v, others])
    keep = u != v
    u, v = u[keep], v[keep]
    g = rng.lognormal(0.0, 0.5, u.size)
    cap = rng.uniform(1e-15, 1e-14, n)
    pads = np.arange(0, n, 50, dtype=np.int64)
    nodes = np.sort(rng.choice(n, size=max(1, n // 3), replace=False)).astype(np.int64)
    src = gridgen._triangle_sources(rng, nodes, 1e-3, 40e-12, 60e-12)
    return gridgen.EdgeGrid(n=n, eu=u, ev=v, eg=g, cap=cap, pad_node=pads, pad_g=np.full(pads.size, 10.0),
                            vdd=1.0, sources=src, h=5e-12, steps=8)


def run(P, g, steps, tol, omega, k, options=None, probes=True):
    G = P.Grid.from_edge_grid(g, device=True) if not hasattr(g, "gx") else P.Grid.from_mesh_grid(g, device=True)
    for key, val in (options or {}).items():
        G.set_option(key, val)
    r = G.transient(g.h, steps, tol=tol, omega=omega, max_sweeps=k, probes=np.arange(g.n) if probes else None,
                    raise_on_noconv=False)
    n_col = G.info()["n_colors"]
    G.close()
    return r, n_col


@pytest.mark.parametrize("n,extra,star", [(37, 20, 0), (1001, 700, 0), (3001, 2500, 0), (20011, 15000, 0),
                                          (5003, 3000, 4000)])
def test_staged_csr_equals_row_kernel_and_oracle(pgb, n, extra, star):
    g = random_graph(n, extra, seed=n + star, star=star)
    ra, nc = run(pgb, g, 6, 0.0, 1.5, 7, {"csr_stage": 1})
    rb, _ = run(pgb, g, 6, 0.0, 1.5, 7, {"csr_stage": 0})
    print(f"n = {n}: {nc} colours")
    np.testing.assert_array_equal(ra.probes, rb.probes)
    assert np.abs(ra.probes[-1] - 1.0).max() > 1e-9
    # converged: the exact solution of both iterations (oracle in natural order)
    nl = netlist.from_edges(g)
    o = nodal.NodalOracle(nl)
    ro = o.transient(g.h, 6, tol=1e-13, omega=1.5, Itab=pwl.node_currents_table(nl, g.h, 6))
    rc, _ = run(pgb, g, 6, 1e-13, 1.5, 200000)
    assert ro.status == 0 and rc.status == 0
    np.testing.assert_allclose(rc.probes, ro.V, rtol=0, atol=1e-9)


@pytest.mark.parametrize("n,extra,star,graph", [(1001, 700, 0, 1), (20011, 15000, 0, 1), (20011, 15000, 0, 0),
                                                (5003, 3000, 4000, 1)])
def test_staged_csr_pdl_is_bit_identical(pgb, n, extra, star, graph):
    """Option pdl on the CSR path (programmatic dependent launch of the staged
    colour launches: the first tiles' row data requested before
    griddepcontrol.wait): same iterates, same converged results and sweep
    counts (a converged step's queued launches drain their copies and exit)."""
    g = random_graph(n, extra, seed=n + star, star=star)
    ra, _ = run(pgb, g, 6, 0.0, 1.5, 7, {"pdl": 1, "graph": graph})
    rb, _ = run(pgb, g, 6, 0.0, 1.5, 7, {"pdl": 0, "graph": graph})
    np.testing.assert_array_equal(ra.probes, rb.probes)
    ca, _ = run(pgb, g, 6, 1e-11, 1.5, 200000, {"pdl": 1, "graph": graph})
    cb, _ = run(pgb, g, 6, 1e-11, 1.5, 200000, {"pdl": 0, "graph": graph})
    assert ca.status == 0 and cb.status == 0
    np.testing.assert_array_equal(ca.probes, cb.probes)
    np.testing.assert_array_equal(np.asarray(ca.sweeps), np.asarray(cb.sweeps))


def _two_components(n, seed):
    """Two disjoint random bipartite pieces (a path plus odd-offset chords):
    the device builder seeds each piece at its smallest node (minimum-label
    propagation), as the host's BFS per component does."""
    rng = np.random.default_rng(seed)
    h = n // 2
    us, vs = [], []
    for off, m in ((0, h), (h, n - h)):
        us.append(np.arange(off, off + m - 1)); vs.append(np.arange(off + 1, off + m))
        a = rng.integers(off, off + m - 3, m // 2)
        us.append(a); vs.append(a + 3)                     # odd distance: keeps the piece bipartite
    u, v = np.concatenate(us).astype(np.int64), np.concatenate(vs).astype(np.int64)
    g = rng.lognormal(0.0, 0.5, u.size)
    pads = np.array([0, h], np.int64)
    nodes = np.arange(1, n, 7, dtype=np.int64)
    src = gridgen._triangle_sources(rng, nodes, 1e-3, 40e-12, 60e-12)
    return gridgen.EdgeGrid(n=n, eu=u, ev=v, eg=g, cap=rng.uniform(1e-15, 1e-14, n), pad_node=pads,
                            pad_g=np.full(2, 10.0), vdd=1.0, sources=src, h=5e-12, steps=8)


@pytest.mark.parametrize("case", ["config2_small", "config2_ragged", "non_bipartite", "two_components"])
def test_device_csr_builder_equals_host_builder(pgb, case, monkeypatch):
    # pg_create_csr builds the colour-permuted store on the device for
    # bipartite graphs (pg_csr_device.cu) and on the host otherwise or with
    # PGB200_CSR_HOST set: same colours, permutation, rows, so bit-identical
    # iterates; both memories of the inputs
    if case == "config2_small":
        g = gridgen.config_grid(2, dims=(2, 64, 96), steps=4)
    elif case == "config2_ragged":
        g = gridgen.config_grid(2, dims=(3, 37, 53), steps=4)
    elif case == "non_bipartite":
        g = random_graph(3001, 2500, seed=7)
    else:
        g = _two_components(4001, seed=5)
    runs = {}
    for host in (False, True):
        if host:
            monkeypatch.setenv("PGB200_CSR_HOST", "1")
        else:
            monkeypatch.delenv("PGB200_CSR_HOST", raising=False)
        for device in (False, True):
            G = pgb.Grid.from_edge_grid(g, device=device)
            nc = G.info()["n_colors"]
            r = G.transient(g.h, 4, tol=0.0, omega=1.7, max_sweeps=9, probes=np.arange(g.n),
                            raise_on_noconv=False)
            G.close()
            runs[(host, device)] = (nc, r.probes)
    ref_nc, ref = runs[(True, False)]
    for key, (nc, pr) in runs.items():
        assert nc == ref_nc, key
        np.testing.assert_array_equal(pr, ref, err_msg=str(key))
    assert np.abs(ref[-1] - 1.0).max() > 1e-9


def test_rhs_tiles_multi_pads_and_loads(pgb):
    # 3 x 40 x 70 mesh: np = 3 * 40 * 128 = 15360 storage elements = 7.5 RHS tiles
    L, NY, NX = 3, 40, 70
    g = gridgen.mesh_grid(L, NY, NX, seed=21, pad_pitch=7, src_frac=0.3, h=10e-12, src_start=5e-12,
                          src_width=40e-12)
    # extra pads (some on nodes that already have one), on the top layer
    rng = np.random.default_rng(3)
    top = (L - 1) * NY * NX
    extra_pads = np.concatenate([g.pad_node[:5], top + rng.choice(NY * NX, 12, replace=False)])
    g.pad_node = np.concatenate([g.pad_node, extra_pads]).astype(np.int64)
    g.pad_g = np.concatenate([g.pad_g, rng.uniform(2.0, 20.0, extra_pads.size)])
    # storage index s = l*NY*128 + y*128 + (x&1)*64 + x//2: nodes whose storage
    # index is at / next to a multiple of 2048 (tile boundaries)
    def node_of_storage(s):
        l, r = divmod(s, NY * 128)
        y, o = divmod(r, 128)
        x = 2 * (o - 64) + 1 if o >= 64 else 2 * o
        return (l * NY + y) * NX + x if x < NX else None
    edge_nodes = [node_of_storage(t * 2048 + d) for t in range(1, 8) for d in (-1, 0, 1)]
    edge_nodes = [e for e in edge_nodes if e is not None and e < L * NY * NX]
    assert len(edge_nodes) >= 10
    # loads: the generator's (3 breakpoints) + extra ones with 2 and 5
    # breakpoints, several on the same node, in shuffled order
    s = g.sources
    node, ts, vs = [], [], []
    for k in range(s.count):
        node.append(int(s.node[k])); ts.append(s.t[s.ptr[k]:s.ptr[k + 1]]); vs.append(s.i[s.ptr[k]:s.ptr[k + 1]])
    for e in edge_nodes + edge_nodes[:4]:
        nb = int(rng.integers(1, 6))
        t0 = rng.uniform(0, 30e-12)
        node.append(int(e)); ts.append(t0 + np.cumsum(rng.uniform(5e-12, 20e-12, nb)))
        vs.append(rng.uniform(0, 2e-3, nb))
    order = rng.permutation(len(node))
    ptr = np.zeros(len(node) + 1, np.int64)
    ptr[1:] = np.cumsum([ts[k].size for k in order])
    g.sources = gridgen.Sources(node=np.array([node[k] for k in order], np.int64), ptr=ptr,
                                t=np.concatenate([ts[k] for k in order]), i=np.concatenate([vs[k] for k in order]))
    steps, k = 6, 5
    nl = netlist.from_mesh(g)
    ro = nodal.NodalOracle(nl).transient(g.h, steps, tol=0.0, omega=1.6,
                                         order=nodal.red_black_order(L, NY, NX),
                                         Itab=pwl.node_currents_table(nl, g.h, steps), max_sweeps=k)
    for opts in ({"resident": 0}, {"resident": 0, "fuse": 1}):
        rg, _ = run(pgb, g, steps, 0.0, 1.6, k, opts)
        np.testing.assert_allclose(rg.probes, ro.V, rtol=0, atol=1e-12)
    assert np.abs(ro.V[-1] - 1.0).max() > 1e-6


def test_source_order_does_not_matter(pgb):
    # the device-side store sorts loads by storage index (ties in input
    # order): the same loads given sorted or shuffled give identical iterates
    # when no node carries two loads (sums in the same order)
    g = gridgen.mesh_grid(2, 33, 45, seed=9, pad_pitch=5, src_frac=0.5, h=10e-12, src_start=5e-12,
                          src_width=30e-12)
    ra, _ = run(pgb, g, 5, 0.0, 1.7, 6, {"resident": 0})
    s = g.sources
    perm = np.random.default_rng(1).permutation(s.count)
    lens = np.diff(s.ptr)[perm]
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    t = np.concatenate([s.t[s.ptr[k]:s.ptr[k + 1]] for k in perm])
    i = np.concatenate([s.i[s.ptr[k]:s.ptr[k + 1]] for k in perm])
    g.sources = gridgen.Sources(node=s.node[perm], ptr=ptr, t=t, i=i)
    rb, _ = run(pgb, g, 5, 0.0, 1.7, 6, {"resident": 0})
    np.testing.assert_array_equal(ra.probes, rb.probes)


def test_bad_sources_rejected_and_store_kept(pgb):
    g = gridgen.mesh_grid(2, 10, 12, seed=2, pad_pitch=4, src_frac=0.5, h=10e-12, src_start=5e-12,
                          src_width=30e-12)
    G = pgb.Grid.from_mesh_grid(g)
    G.set_option("resident", 0)
    r0 = G.transient(g.h, 3, tol=0.0, omega=1.5, max_sweeps=4, probes=np.arange(g.n))
    bad = [
        (np.array([3]), np.array([1, 2]), np.array([0.0, 1.0]), np.array([1e-3, 0.0])),  # ptr[0] != 0
        (np.array([3, 4]), np.array([0, 1, 1]), np.array([0.0]), np.array([1e-3])),     # empty source
        (np.array([g.n]), np.array([0, 1]), np.array([0.0]), np.array([1e-3])),         # node out of range
        (np.array([3]), np.array([0, 2]), np.array([1.0, 1.0]), np.array([0.0, 1.0])),  # not increasing
        (np.array([3, 4]), np.array([0, 10**6, 3]), np.zeros(3), np.zeros(3)),         # offset past the end
    ]
    for args in bad:
        with pytest.raises(pgb.PgError):
            G.set_sources(*args)
    r1 = G.transient(g.h, 3, tol=0.0, omega=1.5, max_sweeps=4, probes=np.arange(g.n))
    np.testing.assert_array_equal(r0.probes, r1.probes)      # the previous store is intact
    G.close()


def test_release_memory_returns_the_pool_cache(pgb):
    # a destroyed grid's blocks stay cached in the library's pools (for the
    # next grid) until pg_release_memory hands them back to the driver
    import torch
    g = gridgen.config_grid(1, dims=(4, 1024, 1024), steps=1)
    G = pgb.Grid.from_mesh_grid(g)
    G.close()
    torch.cuda.synchronize()
    free_cached, _ = torch.cuda.mem_get_info()
    pgb.release_memory(-1)
    free_released, _ = torch.cuda.mem_get_info()
    # ~12 per-node arrays of 4.2M doubles (33.6 MB each) were cached
    assert free_released - free_cached >= 10 * 33_554_432
    pgb.release_memory(torch.cuda.current_device())   # idempotent, single device
    G = pgb.Grid.from_mesh_grid(g)                     # the pools serve new grids afterwards
    r = G.transient(g.h, 1, tol=1e-10, omega=1.96, max_sweeps=100000)
    G.close()
    assert r.status == 0


@pytest.mark.parametrize("host_builder", [False, True])
@pytest.mark.parametrize("device", [False, True])
def test_csr_input_errors(pgb, host_builder, device, monkeypatch):
    # bad branch lists and capacitances are rejected (PG_EINVAL) by the device
    # builder and the host builder alike, host and device inputs
    import torch
    if host_builder:
        monkeypatch.setenv("PGB200_CSR_HOST", "1")
    else:
        monkeypatch.delenv("PGB200_CSR_HOST", raising=False)
    put = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()) if device else (lambda a: a)
    n = 6
    u, v = np.array([0, 1, 2, 3, 4], np.int64), np.array([1, 2, 3, 4, 5], np.int64)
    g, cap = np.ones(5), np.full(n, 1e-15)
    pads, pg = np.array([0], np.int64), np.array([10.0])
    G = pgb.Grid.csr(n, put(u), put(v), put(g), put(cap), put(pads), put(pg))   # valid
    G.close()
    for bu, bv, bg, c, what in [(np.array([0, 1, 2, 3, 9]), v, g, cap, "branch 4"),
                                (u, np.array([1, -2, 3, 4, 5]), g, cap, "branch 1"),
                                (u, v, np.array([1.0, 1.0, -1.0, 1.0, 1.0]), cap, "branch 2"),
                                (u, v, np.array([1.0, np.nan, 1.0, 1.0, 1.0]), cap, "branch 1"),
                                (u, v, g, np.array([1e-15, 1e-15, np.inf, 1e-15, 1e-15, 1e-15]), "cap")]:
        with pytest.raises(pgb.PgError) as e:
            pgb.Grid.csr(n, put(bu.astype(np.int64)), put(bv.astype(np.int64)), put(bg), put(c), put(pads), put(pg))
        assert e.value.code == -1 and what in str(e.value), str(e.value)
