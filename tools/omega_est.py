"""pg_estimate_omega (Rayleigh-quotient estimate) for several sweep counts, per config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen
import paper_1409_7166_b200 as P

for cfg in [int(c) for c in sys.argv[1].split(",")]:
    g = gridgen.config_grid(cfg)
    mk = P.Grid.from_mesh_grid if hasattr(g, "gx") else P.Grid.from_edge_grid
    G = mk(g, device=True)
    for sw in [int(x) for x in sys.argv[2].split(",")]:
        t0 = time.time()
        rho, om = G.estimate_omega(g.h, sw)
        print(f"config{cfg}: {sw} sweeps: rho {rho!r} omega {om!r} ({time.time() - t0:.1f} s)", flush=True)
    G.close()
