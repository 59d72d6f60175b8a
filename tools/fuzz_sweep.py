"""Randomised cross-check on the GPU (not part of the suite): random mesh
shapes, layer counts, rows-per-CTA, omega, RC/RLC; the pipeline kernel
(pipe=1) must equal the generic kernel (pipe=0) bit for bit and the oracle to
1e-12 V; peer-memory slab groups (random slab counts) must equal the single
grid bit for bit; the per-colour sweep (option colour) must equal the pipeline
bit for bit, and on meshes of 9-24 layers (a quarter of the cases, only the
per-colour sweep exists there) the oracle to 1e-12 V.
usage: python tools/fuzz_sweep.py N_CASES SEED"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gridgen
import paper_1409_7166_b200 as P
from oracle import netlist, nodal, pwl

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
fails = 0
for case in range(n_cases):
    tall = bool(rng.random() < 0.25)
    L = int(rng.integers(9, 25)) if tall else int(rng.integers(1, 9))
    NY = int(rng.integers(1, 80))
    NX = int(rng.integers(1, 200))
    rlc = bool(rng.random() < 0.3)
    rows = int(rng.choice([0, 1, 3, 7, 13, 29, 61]))
    omega = float(rng.uniform(0.8, 1.95))
    k = int(rng.choice([2, 4, 6, 8]))
    steps = int(rng.integers(1, 4))
    g = gridgen.mesh_grid(L, NY, NX, seed=int(rng.integers(1 << 30)), pad_pitch=int(rng.integers(2, 9)),
                          src_frac=0.4, h=10e-12 if not rlc else 2e-12, src_start=5e-12, src_width=30e-12,
                          rlc=rlc)
    res = {}
    variants = ("colour",) if tall else (1, 0, "colour")
    for var in variants:
        G = P.Grid.from_mesh_grid(g, device=True)
        opts = [("resident", 0), ("fuse", 2), ("rows", rows)]
        opts += [("colour", 1)] if var == "colour" else [("pipe", var)]
        for key, v in opts:
            G.set_option(key, v)
        r = G.transient(g.h, steps, tol=0.0, omega=omega, max_sweeps=k, probes=np.arange(g.n, dtype=np.int64),
                        raise_on_noconv=False)
        res[var] = r.probes
        G.close()
    if tall:
        res[1] = res["colour"]
        ok = True
    else:
        ok = np.array_equal(res[1], res[0]) and np.array_equal(res[1], res["colour"])
    nl = netlist.from_grid(g, "element" if rlc else "node")
    ro = nodal.NodalOracle(nl).transient(g.h, steps, tol=0.0, omega=omega, max_sweeps=k,
                                         order=nodal.red_black_order(L, NY, NX),
                                         Itab=pwl.node_currents_table(nl, g.h, steps))
    err = float(np.abs(res[1] - ro.V[:, :g.n]).max())
    ok = ok and err <= 1e-12
    # peer group
    perr = None
    nsl = int(rng.integers(2, 6))
    if NY >= nsl * 5 + 8 and not tall:
        try:
            grp = P.SlabGroup.local(g, nsl, fuse=2, transport="p2p", options={"rows": rows} if rows else None)
            grp.transient(g.h, steps, tol=0.0, omega=omega, max_sweeps=k, raise_on_noconv=False)
            V = np.zeros((L, NY, NX))
            for sp, Vo in grp.owned_voltages(g):
                V[:, sp.y0:sp.y1, :] = Vo
            grp.close()
            perr = float(np.abs(V.reshape(-1) - res[1][-1]).max())
            ok = ok and perr == 0.0
        except ValueError:
            pass
    if not ok:
        fails += 1
    print(f"case {case}: L={L} NY={NY} NX={NX} rlc={rlc} rows={rows} k={k} steps={steps} "
          f"{'tall (colour only)' if tall else 'pipe==generic==colour %s' % ok} oracle {err:.1e} p2p({nsl}) {perr} {'OK' if ok else 'FAIL'}",
          flush=True)
print(f"{n_cases - fails}/{n_cases} passed")
sys.exit(1 if fails else 0)
