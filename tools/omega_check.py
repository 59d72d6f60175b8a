"""Young's omega (pg_estimate_omega) for a BASELINE config vs the hand-picked one."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen  # noqa: E402
import paper_1409_7166_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
tsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
g = gridgen.config_grid(cfg)
mk = P.Grid.from_mesh_grid if hasattr(g, "gx") else P.Grid.from_edge_grid
G = mk(g, device=True)
for sweeps in (500, 2000, 8000):
    t0 = time.time()
    rho, om = G.estimate_omega(g.h, sweeps)
    print(f"config{cfg}: {sweeps} Jacobi sweeps -> rho_J = {rho:.8f}, omega_Young = {om:.5f} ({time.time() - t0:.2f} s)")
for om in sorted({1.9, 1.95, 1.98, 1.99, round(om, 4)}):
    r = G.transient(g.h, tsteps, tol=1e-10, omega=om, max_sweeps=200000)
    print(f"   omega {om:.4f}: {r.stats.sweeps_total} sweeps over {tsteps} steps, {r.stats.device_ms:.1f} ms")
