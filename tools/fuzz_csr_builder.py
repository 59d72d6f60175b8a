"""Randomised cross-check of the device CSR builder (pg_csr_device.cu) against
the host builder (PGB200_CSR_HOST=1) on the GPU (not part of the suite):
config-2-recipe grids of random shape (connected, bipartite: the device path)
and random graphs (trees plus chords -- half of them between the tree's two
colours, so bipartite: the device path; the others mostly not: the host
fallback -- some split into pieces, with open branches or self loops).  Both stores must give bit-identical iterates.
usage: python tools/fuzz_csr_builder.py N_CASES SEED"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import gridgen  # noqa: E402
import paper_1409_7166_b200 as P  # noqa: E402


def random_graph(rng, n):
    perm = rng.permutation(n)
    u = [perm[k] for k in range(1, n)]
    v = [perm[rng.integers(0, k)] for k in range(1, n)]
    extra = int(rng.integers(0, n))
    a, b = rng.integers(0, n, extra), rng.integers(0, n, extra)
    if rng.random() < 0.5:           # bipartite: chords between the two colours of the tree
        depth = np.zeros(n, np.int64)
        for k in range(1, n):        # the tree's parent of perm[k] is perm[j], j < k
            depth[perm[k]] = depth[v[k - 1]] + 1
        b = np.where((depth[a] ^ depth[b]) & 1, b, -1)
        a, b = a[b >= 0], b[b >= 0]
    u = np.concatenate([np.array(u, np.int64), a])
    v = np.concatenate([np.array(v, np.int64), b])
    if rng.random() < 0.3:           # cut into two pieces
        keep = (u < n // 2) == (v < n // 2)
        u, v = u[keep], v[keep]
    g = rng.lognormal(0.0, 0.5, u.size)
    if rng.random() < 0.2:           # some open branches and self loops
        g[rng.random(u.size) < 0.05] = 0.0
        v = np.where(rng.random(u.size) < 0.02, u, v)
    pads = np.arange(0, n, int(rng.integers(5, 60)), dtype=np.int64)
    nodes = np.sort(rng.choice(n, size=max(1, n // 3), replace=False)).astype(np.int64)
    src = gridgen._triangle_sources(rng, nodes, 1e-3, 40e-12, 60e-12)
    return gridgen.EdgeGrid(n=n, eu=u, ev=v, eg=g, cap=rng.uniform(1e-15, 1e-14, n), pad_node=pads,
                            pad_g=np.full(pads.size, 10.0), vdd=1.0, sources=src, h=5e-12, steps=4)


def run(g, host, pdl=0):
    if host:
        os.environ["PGB200_CSR_HOST"] = "1"
    else:
        os.environ.pop("PGB200_CSR_HOST", None)
    G = P.Grid.from_edge_grid(g, device=bool(host is False))
    nc = G.info()["n_colors"]
    if pdl:
        G.set_option("pdl", 1)
    r = G.transient(g.h, 3, tol=0.0, omega=1.6, max_sweeps=7, probes=np.arange(g.n), raise_on_noconv=False)
    G.close()
    return nc, r.probes


n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
fails = 0
for case in range(n_cases):
    if rng.random() < 0.6:
        dims = (int(rng.integers(1, 5)), int(rng.integers(2, 90)), int(rng.integers(2, 130)))
        g = gridgen.config_grid(2, dims=dims, steps=4, seed=int(rng.integers(1 << 30)))
        kind = f"config2 {dims}"
    else:
        n = int(rng.integers(3, 6000))
        g = random_graph(rng, n)
        kind = f"random n={n} m={g.eu.size}"
    nd, pd = run(g, False)
    nh, ph = run(g, True)
    _, pp = run(g, False, pdl=1)     # programmatic dependent launch of the staged colour launches
    ok = nd == nh and np.array_equal(pd, ph) and np.array_equal(pd, pp)
    fails += not ok
    print(f"case {case}: {kind} colours {nd}/{nh} {'OK' if ok else 'MISMATCH'}", flush=True)
print(f"{n_cases - fails}/{n_cases} passed")
sys.exit(1 if fails else 0)
