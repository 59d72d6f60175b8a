"""Where the end-to-end (host-buffer) call spends its time on a config: grid
creation from host arrays, set_sources, transient, voltage read-back."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gridgen
import paper_1409_7166_b200 as P

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = gridgen.config_grid(cfg)
pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(g, k))).pin_memory().numpy() for k in ("gx", "gy", "gz", "cap")}
out = torch.empty(g.n, dtype=torch.float64).pin_memory().numpy()
s = g.sources
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    H = P.Grid.mesh(g.layers, g.ny, g.nx, pin["gx"], pin["gy"], pin["gz"], pin["cap"], g.pad_node, g.pad_g, g.vdd,
                    None, None)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    H.set_sources(s.node, s.ptr, s.t, s.i)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    r = H.transient(g.h, T, tol=1e-10, omega=1.9639)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    H.voltages(out)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    H.close()
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, set_sources {1e3*(t2-t1):.1f} ms, transient({T}) {1e3*(t3-t2):.1f} ms "
          f"(device {r.stats.device_ms:.1f}), voltages {1e3*(t4-t3):.1f} ms, close {1e3*(t5-t4):.1f} ms")
