"""Full-size converged-waveform parity (-m gpu) against oracle goldens.

tests/golden/fullsize_<job>.npz were written by tools/make_golden_fullsize.py,
which calls only gridgen + oracle/ (the plain-C nodal SOR of PAPER.md §IV,
Algorithm 1): BASELINE.json configs 1-4 at FULL size, converged to tol at
every step from x(0) = Vdd, at the omega bench.py uses (Young's estimate,
DESIGN.md R15).  Each golden holds V at >= 64k sampled nodes (seeded random
nodes plus the all-layer 3 x 3 columns around the 32 earliest-starting loads)
for every step, the oracle's sweep counts and its stopping record.

Here the GPU runs the same transient in the launch configuration bench.py
times (default options) and records the same nodes with pg_transient's probes:

* V: |V_gpu - V_oracle| <= 1e-8 V at every sampled node and step
  (BASELINE.json north_star);
* sweep counts: the GPU tests its stopping criterion (Algorithm 1 line 8)
  every F sweeps (R13), so its count at step s is the first multiple
  of F at or after the oracle's k with ||V^(j) - V^(j-1)|| < tol, read from the
  oracle's stopping record (norms of sweeps k-1 .. k+4).  Steps where a norm
  that decides it lies within 1e-6 * tol of tol (fp64 summation order may flip
  the decision) are listed and allowed +-F; all others must be equal.
* c3_node_tight: the paper's internal-node model of the series R-L branches
  (R7) in natural order at tol = 1e-13 against the GPU's eliminated-node
  red-black iteration at tol = 1e-13 -- two different iterations of the same
  exact solution, so only V is compared (1e-8 V; DESIGN.md §5 for the bound).
"""
import glob
import os

import numpy as np
import pytest

import gridgen
from sweepcount import check_counts

pytestmark = [pytest.mark.gpu]

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDENS = sorted(glob.glob(os.path.join(HERE, "golden", "fullsize_*.npz")))
ATOL_CONV = 1e-8


@pytest.fixture(scope="module")
def pgb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1409_7166_b200 as P
    from paper_1409_7166_b200 import build
    build.build()
    return P


def _jobs():
    return [os.path.basename(p)[len("fullsize_"):-len(".npz")] for p in GOLDENS]


@pytest.mark.parametrize("job", _jobs())
def test_fullsize_converged_vs_oracle_golden(pgb, job):
    z = np.load(os.path.join(HERE, "golden", f"fullsize_{job}.npz"))
    cfg, steps = int(z["config"]), int(z["steps"])
    tol, omega = float(z["tol"]), float(z["omega"])
    nodes, Vo = z["nodes"], z["V"]
    g = gridgen.config_grid(cfg)
    assert abs(g.h - float(z["h"])) == 0.0
    mk = pgb.Grid.from_mesh_grid if hasattr(g, "gx") else pgb.Grid.from_edge_grid
    G = mk(g, device=True)
    r = G.transient(g.h, steps, tol=tol, omega=omega, max_sweeps=200000, probes=nodes)
    F = int(r.stats.sweeps_per_launch)
    G.close()
    assert r.status == 0
    err = np.abs(r.probes - Vo).max(axis=1)
    print(f"{job}: max |V_gpu - V_oracle| per step {np.array2string(err, precision=2)}; "
          f"max IR drop {1e3 * (1.0 - Vo.min()):.3f} mV")
    assert np.abs(Vo[-1] - 1.0).max() > 1e-6                   # the loads act
    assert err.max() <= ATOL_CONV
    if str(z["order"]) != "redblack":
        return                                                   # different iteration (model check only)
    flagged = check_counts(r.sweeps, z["sweeps"], z["dtrace"], tol, F)
    print(f"{job}: F = {F}, sweep counts equal at {steps - len(flagged)} of {steps} steps; "
          f"rounding-band steps {flagged}")
