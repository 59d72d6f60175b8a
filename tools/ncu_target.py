"""Small fixed workload for ncu captures: BASELINE config 1 grid, `steps` time
steps with a fixed number of sweeps each (tol = 0) -> deterministic launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen
import paper_1409_7166_b200 as P
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
method = sys.argv[4] if len(sys.argv) > 4 else "rbsor"
g = gridgen.config_grid(cfg)
G = P.Grid.from_mesh_grid(g, device=True) if hasattr(g, "gx") else P.Grid.from_edge_grid(g, device=True)
r = G.transient(g.h, steps, tol=0.0, omega=1.98, method=method, max_sweeps=sweeps, raise_on_noconv=False)
print("ok", r.stats.sweeps_total, r.stats.device_ms)
