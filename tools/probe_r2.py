"""Round-2 probe: Young's omega (pg_estimate_omega) per BASELINE config, the
converged sweep counts and time per step at that omega, and the box's host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import gridgen  # noqa: E402
import paper_1409_7166_b200 as P  # noqa: E402

print("host cores", os.cpu_count(), flush=True)
with open("/proc/meminfo") as f:
    print(f.readline().strip(), flush=True)
cfgs = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 3, 4]
tsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for cfg in cfgs:
    t0 = time.time()
    g = gridgen.config_grid(cfg)
    mk = P.Grid.from_mesh_grid if hasattr(g, "gx") else P.Grid.from_edge_grid
    G = mk(g, device=True)
    print(f"config{cfg}: n = {g.n}, create {time.time() - t0:.1f} s", flush=True)
    for sweeps in (8000, 20000):
        t0 = time.time()
        rho, om = G.estimate_omega(g.h, sweeps)
        print(f"  {sweeps} Jacobi sweeps: rho_J = {rho!r}, omega_Young = {om!r} ({time.time() - t0:.2f} s)",
              flush=True)
        if sweeps == 8000:
            om8 = om
    for o in (om8, 1.99):
        r = G.transient(g.h, tsteps, tol=1e-10, omega=o, max_sweeps=200000)
        print(f"  omega {o:.6f}: sweeps/step {r.sweeps[1:].tolist()}, {r.stats.device_ms / tsteps:.1f} ms/step",
              flush=True)
    G.close()
