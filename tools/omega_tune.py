"""pg_tune_omega per config (the run-time counterpart of bench.py's recorded OMEGA)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen
import paper_1409_7166_b200 as P

for cfg in [int(c) for c in sys.argv[1].split(",")]:
    g = gridgen.config_grid(cfg)
    mk = P.Grid.from_mesh_grid if hasattr(g, "gx") else P.Grid.from_edge_grid
    G = mk(g, device=True)
    t0 = time.time()
    om, sw = G.tune_omega(g.h, steps=8, tol=1e-10, n=8, d_omega=4e-4)
    print(f"config{cfg}: tuned omega {om:.6f} ({time.time() - t0:.1f} s); sweeps over 8 steps per candidate "
          f"{sw.tolist()}", flush=True)
    G.close()
