"""Scratch: sweep-kernel time vs (kernel, rows per CTA, ring stages) on config 1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen, paper_1409_7166_b200 as P
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = gridgen.config_grid(cfg)
G = P.Grid.from_mesh_grid(g, device=True)
G.set_option("timing", 1)
def run(kernel, rows, stages):
    G.set_option("kernel", kernel); G.set_option("rows", rows); G.set_option("stages", stages)
    G.transient(g.h, 1, tol=0.0, omega=1.98, max_sweeps=10, raise_on_noconv=False)
    r = G.transient(g.h, 2, tol=0.0, omega=1.98, max_sweeps=60, raise_on_noconv=False)
    us = r.stats.sweep_ms / r.stats.sweep_launches * 1e3
    print(f"kernel={kernel} rows={rows:4d} stages={stages:2d}: {us:6.1f} us/sweep  {56*g.n/us/1e3:6.0f} GB/s", flush=True)
for kernel, stages in [(3, 6), (3, 8)]:
    for rows in [0, 24, 32, 43, 48, 64]:
        run(kernel, rows, stages)
