"""Integrity of the full-size oracle goldens (-m "not gpu"): each file under
tests/golden/fullsize_*.npz was written by tools/make_golden_fullsize.py from
gridgen + oracle/ only; here its metadata is checked against the bench's
workload (omega = bench.OMEGA, h and steps of the BASELINE config), the
sampled nodes against the generator's seeded recipe, and the stored record
against Algorithm 1's stopping rule (line 8: the last sweep of every step is
the first one below tol, with the paper's check after every sweep)."""
import glob
import os
import sys

import numpy as np
import pytest

import gridgen

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tools"))
GOLDENS = sorted(glob.glob(os.path.join(HERE, "golden", "fullsize_*.npz")))


@pytest.mark.parametrize("path", GOLDENS, ids=[os.path.basename(p) for p in GOLDENS])
def test_golden_metadata_and_stopping_record(path):
    import bench
    import make_golden_fullsize as mg
    z = np.load(path)
    job = str(z["job"])
    cfg, steps, tol, srl, order, omega = mg.JOBS[job]
    assert int(z["config"]) == cfg and int(z["steps"]) == steps and float(z["tol"]) == tol
    assert str(z["series_rl"]) == srl and str(z["order"]) == order
    assert float(z["omega"]) == omega
    if job == f"c{cfg}" or job == f"c{cfg}_element":
        assert omega == bench.OMEGA[cfg] == mg.OMEGA[cfg]          # the bench's omega
    c = gridgen.CONFIGS[cfg]
    assert float(z["h"]) == c["h"]
    V, sw, dt = z["V"], z["sweeps"], z["dtrace"]
    assert V.shape == (steps + 1, z["nodes"].size) and z["nodes"].size >= 65536
    np.testing.assert_array_equal(V[0], 1.0)                     # x(0) = Vdd (R11)
    assert sw[0] == 0 and np.all(sw[1:] >= 1)
    assert np.all(dt[1:, 1] < tol)                                 # line 8 met at the last sweep
    assert np.all((sw[1:] == 1) | (dt[1:, 0] >= tol))              # ... and not one sweep earlier
    assert np.all(np.abs(V[1:] - 1.0) < 0.1)                      # IR drops of mV, no runaway
    assert np.abs(V[-1] - 1.0).max() > 1e-6


@pytest.mark.parametrize("path", [p for p in GOLDENS if "c2" not in os.path.basename(p)],
                         ids=[os.path.basename(p) for p in GOLDENS if "c2" not in os.path.basename(p)])
def test_golden_nodes_are_the_seeded_sample(path):
    import make_golden_fullsize as mg
    z = np.load(path)
    cfg = int(z["config"])
    g = gridgen.config_grid(cfg)
    np.testing.assert_array_equal(z["nodes"], mg.sample_nodes(g, cfg))
