"""Per-launch cost of the NCCL slab exchange inside the sweep-batch CUDA graph,
measured with a 1-rank NCCL group (the 8-byte norm allreduce per launch runs;
a 1-rank group has no send/recv) against the single grid, and with graphs off.
usage: python tools/nccl_overhead.py CFG T"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import gridgen
import paper_1409_7166_b200 as P
import bench

cfg, T = int(sys.argv[1]), int(sys.argv[2])
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("gloo", rank=0, world_size=1)
g = gridgen.config_grid(cfg)
om = bench.OMEGA[cfg]


def per_launch(run, grids):
    for q in grids:
        q.set_option("timing", 1)
    run(1)                                  # warm-up (graph capture)
    r = run(T)
    return r.stats.sweep_ms / max(r.stats.sweep_launches, 1) * 1e3, int(r.stats.sweeps_total)


G = P.Grid.from_mesh_grid(g, device=True)
single = per_launch(lambda n: G.transient(g.h, n, tol=1e-10, omega=om, max_sweeps=200000), [G])
G.close()
print(f"config{cfg} single grid: {single[0]:.1f} us per launch ({single[1]} sweeps)", flush=True)
for graph in (1, 0):
    grp = P.SlabGroup.nccl(g, 0, 1, fuse=2)
    grp.grids[0].set_option("graph", graph)
    res = per_launch(lambda n: grp.transient(g.h, n, tol=1e-10, omega=om, max_sweeps=200000), grp.grids)
    grp.close()
    print(f"config{cfg} 1-rank NCCL group, graph={graph}: {res[0]:.1f} us per launch ({res[1]} sweeps)", flush=True)
dist.destroy_process_group()
