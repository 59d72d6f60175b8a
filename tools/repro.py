"""Small transient through the C ABI (debug helper): python tools/repro.py L NY NX [F]"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gridgen
import paper_1409_7166_b200 as P

L, NY, NX = (int(a) for a in sys.argv[1:4])
F = int(sys.argv[4]) if len(sys.argv) > 4 else 2
g = gridgen.mesh_grid(L, NY, NX, seed=1, pad_pitch=3, src_frac=0.5, h=10e-12, src_start=20e-12,
                      src_width=40e-12)
G = P.Grid.from_mesh_grid(g)
G.set_option("fuse", F)
for method in ("jacobi", "rbsor"):
    try:
        r = G.transient(g.h, 3, tol=0.0, omega=1.5, method=method, max_sweeps=3,
                        probes=np.arange(g.n))
        print(method, "ok", r.probes[-1, :4])
    except Exception as e:
        print(method, "FAILED", e)
        break
