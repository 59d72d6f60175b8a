"""Per-launch cost of the fused peer-memory exchange on one GPU: config 1 as a
single grid vs a one-slab p2p group (same kernel, plus the exchange epilogue:
system fences, remote atomics to itself, the arrival wait of the next launch)
and a 2-slab p2p group vs a 2-slab copy group."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gridgen
import paper_1409_7166_b200 as P

g = gridgen.config_grid(1)
T, omega = int(sys.argv[1]) if len(sys.argv) > 1 else 40, 1.9639


def timed(run):
    run()  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    r = run()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1), r


G = P.Grid.from_mesh_grid(g, device=True)
ms, r = timed(lambda: G.transient(g.h, T, tol=1e-10, omega=omega))
launches = int(r.stats.sweeps_total) // 2
print(f"single grid: {ms:.1f} ms, {launches} launches, {1e3 * ms / launches:.2f} us per launch")
G.close()
for n, tr in [(1, "p2p"), (2, "p2p"), (2, "copy")]:
    grp = P.SlabGroup.local(g, n, fuse=2, transport=tr)
    ms, r = timed(lambda: grp.transient(g.h, T, tol=1e-10, omega=omega))
    launches = int(r.stats.sweeps_total) // 2
    print(f"{n} slab(s), {tr}: {ms:.1f} ms, {launches} launches, {1e3 * ms / launches:.2f} us per launch (all slabs)")
    grp.close()
