"""Slab partition on one GPU (-m gpu): pg_group_local runs the n-rank protocol
(global max of the convergence norm + ghost-row exchange after every sweep
launch) with device copies in place of NCCL.  The owned rows of
every slab must equal the single-grid run bit for bit (same arithmetic, same
red-black numbering) and the oracle to rounding; the stopping decisions
(sweep counts) must be the same on every slab and equal to the single grid's."""
import numpy as np
import pytest

import gridgen
from oracle import netlist, nodal, pwl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pgb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1409_7166_b200 as P
    from paper_1409_7166_b200 import build
    build.build()
    return P


def single(P, g, steps, tol, omega, k, F):
    G = P.Grid.from_mesh_grid(g, device=True)
    G.set_option("fuse", F)
    G.set_option("resident", 0)   # the slabs run the streaming sweep
    r = G.transient(g.h, steps, tol=tol, omega=omega, max_sweeps=k, raise_on_noconv=False)
    V = G.voltages().reshape(g.layers, g.ny, g.nx)
    G.close()
    return r, V


def grouped(P, g, n, steps, tol, omega, k, F):
    grp = P.SlabGroup.local(g, n, fuse=F)
    r = grp.transient(g.h, steps, tol=tol, omega=omega, max_sweeps=k, raise_on_noconv=False)
    V = np.zeros((g.layers, g.ny, g.nx))
    for sp, Vo in grp.owned_voltages(g):
        V[:, sp.y0:sp.y1, :] = Vo
    grp.close()
    return r, V


CASES = [((4, 70, 100), 2, 2), ((4, 70, 100), 3, 1), ((2, 64, 33), 4, 2), ((3, 90, 64), 5, 3),
         ((8, 40, 20), 2, 2), ((1, 33, 70), 3, 4)]


@pytest.mark.parametrize("shape,n,F", CASES)
def test_slabs_equal_single_grid_fixed_sweeps(pgb, shape, n, F):
    g = gridgen.mesh_grid(*shape, seed=sum(shape) + n, pad_pitch=5, src_frac=0.4, h=10e-12,
                          src_start=20e-12, src_width=40e-12)
    steps, k, omega = 5, 7, 1.7
    r1, V1 = single(pgb, g, steps, 0.0, omega, k, F)
    rn, Vn = grouped(pgb, g, n, steps, 0.0, omega, k, F)
    np.testing.assert_array_equal(Vn, V1)
    # and the oracle (red-black numbering, same sweeps)
    nl = netlist.from_mesh(g)
    ro = nodal.NodalOracle(nl).transient(g.h, steps, tol=0.0, omega=omega, max_sweeps=k,
                                         order=nodal.red_black_order(*shape),
                                         Itab=pwl.node_currents_table(nl, g.h, steps))
    np.testing.assert_allclose(Vn.reshape(-1), ro.V[-1], rtol=0, atol=1e-12)


@pytest.mark.parametrize("n,F", [(2, 2), (4, 2), (3, 1)])
def test_slabs_converged_global_stopping(pgb, n, F):
    g = gridgen.config_grid(0, dims=(2, 96, 64), steps=12)
    steps, omega = 12, 1.9
    r1, V1 = single(pgb, g, steps, 1e-10, omega, 200000, F)
    rn, Vn = grouped(pgb, g, n, steps, 1e-10, omega, 200000, F)
    assert r1.status == 0 and rn.status == 0
    np.testing.assert_array_equal(rn.sweeps, r1.sweeps)
    np.testing.assert_array_equal(Vn, V1)


def test_rlc_slabs(pgb):
    g = gridgen.mesh_grid(4, 60, 40, seed=9, pad_pitch=4, src_frac=0.5, rlc=True, h=2e-12,
                          src_start=10e-12, src_width=20e-12)
    r1, V1 = single(pgb, g, 10, 0.0, 1.6, 6, 2)
    rn, Vn = grouped(pgb, g, 3, 10, 0.0, 1.6, 6, 2)
    assert np.abs(V1 - 1.0).max() > 1e-6
    np.testing.assert_array_equal(Vn, V1)


def test_slab_errors(pgb):
    P = pgb
    g = gridgen.mesh_grid(2, 40, 30, seed=1, pad_pitch=5)
    grp = P.SlabGroup.local(g, 2, fuse=1)        # ghost rows G = 2
    grp.grids[0].set_option("fuse", 2)           # 2F = 4 > G
    with pytest.raises(P.PgError):
        grp.transient(g.h, 2, tol=0.0, omega=1.5, max_sweeps=3)
    with pytest.raises(P.PgError):               # slab grids are driven by their group
        grp.grids[0].transient(g.h, 2, tol=0.0, omega=1.5, max_sweeps=3)
    grp.close()


def test_nccl_group_single_rank(pgb):
    # the NCCL transport end to end on one GPU: dlopen of libnccl, unique id,
    # communicator, the per-launch norm allreduce (a 1-rank group has no
    # neighbours, so no send/recv) -- same results as the plain grid
    import os
    import torch
    import torch.distributed as dist
    P = pgb
    g = gridgen.mesh_grid(4, 40, 70, seed=4, pad_pitch=5, src_frac=0.4, h=10e-12,
                          src_start=20e-12, src_width=40e-12)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("gloo", rank=0, world_size=1)
    res = {}
    try:
        # graph = 1: full batches of sweep launches replayed from a CUDA graph
        # with the NCCL allreduce (and send/recv) captured after every launch;
        # graph = 0: host-enqueued; and the transient cut into two calls
        for graph in (1, 0):
            grp = P.SlabGroup.nccl(g, 0, 1, fuse=2)
            grp.grids[0].set_option("graph", graph)
            rn = grp.transient(g.h, 6, tol=1e-10, omega=1.8, max_sweeps=200000)
            (sp, Vn), = grp.owned_voltages(g)
            r2 = grp.transient(g.h, 2, tol=1e-10, omega=1.8, max_sweeps=200000)
            r3 = grp.transient(g.h, 4, tol=1e-10, omega=1.8, max_sweeps=200000, cont=True)
            (sp, Vc), = grp.owned_voltages(g)
            grp.close()
            res[graph] = (rn, Vn, np.concatenate([r2.sweeps, r3.sweeps[1:]]), Vc)
    finally:
        dist.destroy_process_group()
    r1, V1 = single(P, g, 6, 1e-10, 1.8, 200000, 2)
    assert r1.sweeps.max() > 8 * 2      # several sweep batches per step: the graph path runs
    for graph in (1, 0):
        rn, Vn, sc, Vc = res[graph]
        np.testing.assert_array_equal(rn.sweeps, r1.sweeps)
        np.testing.assert_array_equal(Vn, V1)
        np.testing.assert_array_equal(sc, r1.sweeps)
        np.testing.assert_array_equal(Vc, V1)
