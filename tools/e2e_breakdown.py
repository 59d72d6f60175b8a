"""Where the end-to-end (host-buffer) call spends its time on a config: grid
creation from pinned host arrays, set_sources, transient window, voltage
read-back, destroy.  usage: python tools/e2e_breakdown.py CFG T REPS"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gridgen
import paper_1409_7166_b200 as P
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = gridgen.config_grid(cfg)
omega = bench.OMEGA.get(cfg, 1.9)
pinned = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
pin = {k: pinned(getattr(g, k, None)) for k in ("gx", "gy", "gz", "cap", "lz", "pad_node", "pad_g", "pad_l",
                                                "eu", "ev", "eg")}
s = g.sources
src = [pinned(a) for a in (s.node, s.ptr, s.t, s.i)]
out = torch.empty(g.n, dtype=torch.float64).pin_memory().numpy()
# as in bench.py: the device-resident grid of the timed region stays alive
keep = ((P.Grid.from_mesh_grid if hasattr(g, "gx") else P.Grid.from_edge_grid)(g, device=True)
        if os.environ.get("E2E_KEEP") else None)
for rep in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if hasattr(g, "gx"):
        H = P.Grid.mesh(g.layers, g.ny, g.nx, pin["gx"], pin["gy"], pin["gz"], pin["cap"], pin["pad_node"],
                        pin["pad_g"], g.vdd, pin["lz"], pin["pad_l"])
    else:
        H = P.Grid.csr(g.n, pin["eu"], pin["ev"], pin["eg"], pin["cap"], pin["pad_node"], pin["pad_g"], g.vdd)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    H.set_sources(*src)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    r = H.transient(g.h, T, tol=1e-10, omega=omega, max_sweeps=200000)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    H.voltages(out)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    H.close()
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"config{cfg} rep {rep}: create {1e3*(t1-t0):.1f} ms, set_sources {1e3*(t2-t1):.1f} ms, "
          f"transient({T}) {1e3*(t3-t2):.1f} ms (device {r.stats.device_ms:.1f}), voltages {1e3*(t4-t3):.1f} ms, "
          f"close {1e3*(t5-t4):.1f} ms", flush=True)
# raw PCIe rates for comparison: torch copies of one pinned 1 GiB array
hb = torch.empty(1 << 27, dtype=torch.float64).pin_memory()
db = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    db.copy_(hb, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    hb.copy_(db, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"raw 1 GiB pinned: H2D {1e3*(t1-t0):.1f} ms ({(1<<30)/(t1-t0)/1e9:.1f} GB/s), "
          f"D2H {1e3*(t2-t1):.1f} ms ({(1<<30)/(t2-t1)/1e9:.1f} GB/s)", flush=True)
