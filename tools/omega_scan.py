"""Sweeps per time step against omega: the first T time steps from x(0) and a
later window of T steps (continued after S steps), per omega.
usage: python tools/omega_scan.py CFG T S om1,om2,..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen
import paper_1409_7166_b200 as P

cfg, T, S = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
oms = [float(x) for x in sys.argv[4].split(",")]
g = gridgen.config_grid(cfg)
mk = P.Grid.from_mesh_grid if hasattr(g, "gx") else P.Grid.from_edge_grid
G = mk(g, device=True)
for om in oms:
    r1 = G.transient(g.h, T, tol=1e-10, omega=om, max_sweeps=200000)
    line = f"config{cfg} omega {om:.5f}: steps 1-{T} mean {r1.sweeps[1:].mean():.1f}"
    if S > T:
        G.transient(g.h, S - T, tol=1e-10, omega=om, max_sweeps=200000, cont=True)
        r2 = G.transient(g.h, T, tol=1e-10, omega=om, max_sweeps=200000, cont=True)
        line += f", steps {S + 1}-{S + T} mean {r2.sweeps[1:].mean():.1f}"
    print(line, flush=True)
