import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch, gridgen, paper_1409_7166_b200 as P
g = gridgen.config_grid(1)
pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(g, k))).pin_memory().numpy() for k in ("gx", "gy", "gz", "cap")}
s = g.sources
print("sources", s.node.shape, s.t.shape, s.node.dtype, s.t.dtype, "sorted nodes:", bool(np.all(np.diff(s.node) >= 0)))
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    H = P.Grid.mesh(g.layers, g.ny, g.nx, pin["gx"], pin["gy"], pin["gz"], pin["cap"], g.pad_node, g.pad_g, g.vdd, None, None)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    H.set_sources(s.node, s.ptr, s.t, s.i)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    H.close()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  set_sources {1e3*(t2-t1):.1f} ms  close {1e3*(t3-t2):.1f} ms")
