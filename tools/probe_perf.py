"""Scratch perf probe: per-sweep time and effective bandwidth on BASELINE configs."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gridgen
import paper_1409_7166_b200 as P

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
t0 = time.time()
g = gridgen.config_grid(cfg)
print(f"gen {time.time()-t0:.1f}s n={g.n}", flush=True)
G = P.Grid.from_mesh_grid(g, device=False) if hasattr(g, "gx") else P.Grid.from_edge_grid(g)
print(f"create {time.time()-t0:.1f}s", flush=True)
for method, kern in [("rbsor", 1), ("rbsor", 0), ("jacobi", 1)]:
    for fuse in [1]:
        G.set_option("batch", 16)
        G.set_option("kernel", kern)
        r = G.transient(g.h, 2, tol=0.0, omega=1.9, method=method, max_sweeps=20, raise_on_noconv=False)
        r = G.transient(g.h, 4, tol=0.0, omega=1.9, method=method, max_sweeps=100, raise_on_noconv=False)
        st = r.stats
        ms_per_sweep = st.device_ms / st.sweeps_total
        gbs = 56.0 * g.n / (ms_per_sweep * 1e-3) / 1e9
        print(f"{method} k{kern}: {st.sweeps_total} sweeps {st.device_ms:.1f} ms -> {ms_per_sweep*1e3:.1f} us/sweep, "
              f"{g.n/ms_per_sweep/1e6:.1f} GNode-sweeps/s, ~{gbs:.0f} GB/s at 56 B/node", flush=True)
G.set_option("kernel", 1)
for om in [1.98, 1.99]:
    r = G.transient(g.h, 60, tol=1e-10, omega=om, max_sweeps=200000)
    print(f"omega {om}: 60 steps sweeps/step mean {r.sweeps[1:].mean():.1f} max {r.sweeps.max()} "
          f"time {r.stats.device_ms:.0f} ms, launches {r.stats.kernel_launches}", flush=True)
