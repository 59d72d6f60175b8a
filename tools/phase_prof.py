"""Per-phase cycle breakdown of the fused sweep (instrumented build).

    python -m paper_1409_7166_b200.build --prof
    PGB200_LIB=paper_1409_7166_b200/lib/libpgb200_prof.so python tools/phase_prof.py [opts...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen  # noqa: E402
import paper_1409_7166_b200 as P  # noqa: E402
from paper_1409_7166_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.pg_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
g = gridgen.config_grid(1)
names = ["wait TMA", "phase A", "bar 1", "phase B", "fence+write", "bar 2+issue"]
for opt in sys.argv[1:] or ["fuse=2"]:
    G = P.Grid.from_mesh_grid(g, device=True)
    for kv in opt.split(","):
        k, v = kv.split("=")
        G.set_option(k, int(v))
    G.transient(g.h, 5, tol=1e-10, omega=1.98, max_sweeps=200000)
    buf = (ctypes.c_ulonglong * 8)()
    lib.pg_debug_prof(buf, 1)
    r = G.transient(g.h, 20, tol=1e-10, omega=1.98, max_sweeps=200000)
    lib.pg_debug_prof(buf, 1)
    tot = sum(buf[k] for k in range(6))
    warps = buf[6]
    print(f"{opt}: launches ~{r.stats.sweeps_total // r.stats.sweeps_per_launch}, warp-launches {warps}, "
          f"device {r.stats.device_ms:.1f} ms")
    for k in range(6):
        print(f"   {names[k]:12s} {buf[k] / tot * 100:5.1f}%  {buf[k] / max(warps, 1):10.0f} cycles/warp-launch")
    G.close()
