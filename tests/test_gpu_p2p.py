"""Peer-memory slab exchange on one GPU (-m gpu): pg_group_local_p2p runs the
n-slab protocol with the exchange fused into the sweep kernel:
each launch stores its boundary rows straight into the neighbours' receive
buffers (double-buffered by launch epoch), max-reduces its norm into every
slab's norm ring and bumps every slab's arrival counter; the next launch waits
on its counter.  On one device the "peers" are the other slabs' buffers and
the launches are ordered on one stream, so the same kernels and pointers are
exercised without ranks waiting on one another.  Bars as for the copy
transport (test_gpu_slab.py): owned rows bit-identical to the single-grid run
(the same pipeline kernel), oracle to 1e-12 V, identical stopping decisions."""
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


def single(P, g, steps, tol, omega, k, options=None):
    G = P.Grid.from_mesh_grid(g, device=True)
    G.set_option("fuse", 2)
    G.set_option("resident", 0)
    for key, v in (options or {}).items():
        G.set_option(key, v)
    r = G.transient(g.h, steps, tol=tol, omega=omega, max_sweeps=k, raise_on_noconv=False)
    V = G.voltages().reshape(g.layers, g.ny, g.nx)
    G.close()
    return r, V


def grouped(P, g, n, steps, tol, omega, k, transport="p2p", options=None, repeat=1):
    grp = P.SlabGroup.local(g, n, fuse=2, transport=transport, options=options)
    for _ in range(repeat):  # epochs continue across transients of one group
        r = grp.transient(g.h, steps, tol=tol, omega=omega, max_sweeps=k, raise_on_noconv=False)
    V = np.zeros((g.layers, g.ny, g.nx))
    for sp, Vo in grp.owned_voltages(g):
        V[:, sp.y0:sp.y1, :] = Vo
    grp.close()
    return r, V


CASES = [((4, 70, 100), 2, None), ((2, 64, 33), 4, None), ((3, 90, 64), 5, {"rows": 7}),
         ((8, 40, 20), 2, None), ((1, 33, 70), 3, {"rows": 5}), ((4, 48, 130), 8, None)]


@pytest.mark.parametrize("shape,n,opts", CASES)
def test_p2p_slabs_equal_single_grid_fixed_sweeps(pgb, shape, n, opts):
    g = gridgen.mesh_grid(*shape, seed=sum(shape) + n, pad_pitch=5, src_frac=0.4, h=10e-12,
                          src_start=20e-12, src_width=40e-12)
    steps, k, omega = 5, 8, 1.7
    r1, V1 = single(pgb, g, steps, 0.0, omega, k)
    rn, Vn = grouped(pgb, g, n, steps, 0.0, omega, k, options=opts)
    assert rn.status == 0
    np.testing.assert_array_equal(Vn, V1)
    nl = netlist.from_mesh(g)
    ro = nodal.NodalOracle(nl).transient(g.h, steps, tol=0.0, omega=omega, max_sweeps=k,
                                         order=nodal.red_black_order(*shape),
                                         Itab=pwl.node_currents_table(nl, g.h, steps))
    np.testing.assert_allclose(Vn.reshape(-1), ro.V[-1], rtol=0, atol=1e-12)


@pytest.mark.parametrize("n", [2, 3, 6])
def test_p2p_converged_global_stopping(pgb, n):
    g = gridgen.config_grid(0, dims=(2, 96, 64), steps=12)
    steps, omega = 12, 1.9
    r1, V1 = single(pgb, g, steps, 1e-10, omega, 200000)
    rn, Vn = grouped(pgb, g, n, steps, 1e-10, omega, 200000)
    rc, Vc = grouped(pgb, g, n, steps, 1e-10, omega, 200000, transport="copy")
    assert r1.status == 0 and rn.status == 0
    np.testing.assert_array_equal(rn.sweeps, r1.sweeps)
    np.testing.assert_array_equal(rn.sweeps, rc.sweeps)
    np.testing.assert_array_equal(Vn, V1)


def test_p2p_repeated_transients_and_rlc(pgb):
    # a second transient on the same group continues the launch epochs (the
    # arrival counters are never reset); RLC meshes carry inductor currents
    g = gridgen.mesh_grid(4, 60, 40, seed=9, pad_pitch=4, src_frac=0.5, rlc=True, h=2e-12,
                          src_start=10e-12, src_width=20e-12)
    steps, omega = 6, 1.8
    r1, V1 = single(pgb, g, steps, 1e-11, omega, 200000)
    rn, Vn = grouped(pgb, g, 3, steps, 1e-11, omega, 200000, repeat=2)
    np.testing.assert_array_equal(rn.sweeps, r1.sweeps)
    np.testing.assert_array_equal(Vn, V1)


def test_p2p_rejects_unsupported(pgb):
    g = gridgen.mesh_grid(2, 40, 30, seed=1, pad_pitch=5, h=10e-12)
    P = pgb
    with pytest.raises(P.PgError):   # F = 1 launches are not the pipeline kernel
        P.SlabGroup.local(g, 2, fuse=1, ghost=4, transport="p2p")
    grp = P.SlabGroup.local(g, 2, fuse=2, transport="p2p")
    with pytest.raises(P.PgError):   # odd max_sweeps would need a partial launch
        grp.transient(g.h, 2, tol=0.0, omega=1.5, max_sweeps=5, raise_on_noconv=False)
    grp.close()


@pytest.mark.parametrize("pdl", [0, 1])
def test_p2p_single_slab_uses_graphs_and_pdl(pgb, pdl):
    # one slab per process (the multi-GPU shape): the exchange lives in the
    # sweep kernels, so the driver replays graph batches (with PDL between
    # launches when the option is on); the result equals the single grid bit
    # for bit
    g = gridgen.config_grid(0, dims=(4, 80, 96), steps=10)
    steps, omega = 10, 1.9
    r1, V1 = single(pgb, g, steps, 1e-10, omega, 200000)
    rn, Vn = grouped(pgb, g, 1, steps, 1e-10, omega, 200000, options={"pdl": pdl}, repeat=2)
    np.testing.assert_array_equal(rn.sweeps, r1.sweeps)
    np.testing.assert_array_equal(Vn, V1)


def test_p2p_ipc_group_one_rank(pgb):
    # the CUDA-IPC setup path (create, export, all-gather over torch.distributed,
    # connect) with one rank: nothing to map, the records still round-trip
    import os
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        g = gridgen.config_grid(0, dims=(4, 64, 80), steps=6)
        grp = pgb.SlabGroup.p2p(g, 0, 1, fuse=2)
        rn = grp.transient(g.h, 6, tol=1e-10, omega=1.9, max_sweeps=200000)
        V = np.zeros((g.layers, g.ny, g.nx))
        for sp, Vo in grp.owned_voltages(g):
            V[:, sp.y0:sp.y1, :] = Vo
        grp.close()
    finally:
        dist.destroy_process_group()
    r1, V1 = single(pgb, g, 6, 1e-10, 1.9, 200000)
    np.testing.assert_array_equal(rn.sweeps, r1.sweeps)
    np.testing.assert_array_equal(V, V1)


def test_p2p_slab_grid_alone_is_refused(pgb):
    # a slab grid of a peer group cannot be swept on its own (its launches
    # would wait for slabs that are not running, and advance its epoch alone);
    # the library refuses, and the group keeps working
    g = gridgen.mesh_grid(2, 40, 30, seed=4, pad_pitch=5, h=10e-12, src_start=5e-12, src_width=30e-12)
    grp = pgb.SlabGroup.local(g, 2, fuse=2, transport="p2p")
    r1 = grp.transient(g.h, 2, tol=1e-10, omega=1.8, max_sweeps=200000)
    G = grp.grids[0]
    with pytest.raises(pgb.PgError):
        G.dc(t=20e-12, tol=1e-9, omega=1.9, max_sweeps=20000)
    with pytest.raises(pgb.PgError):
        G.transient(g.h, 1, tol=1e-10, omega=1.8)
    r2 = grp.transient(g.h, 2, tol=1e-10, omega=1.8, max_sweeps=200000)
    assert np.array_equal(r1.sweeps, r2.sweeps)
    grp.close()


def _ipc_rank(rank, world, port, q):
    # one process per rank, all on cuda:0: the CUDA-IPC export / all-gather /
    # cudaIpcOpenMemHandle connect path across processes, then the self-test
    # (plain stores and loads through the mappings, no kernel waits on another
    # rank -- B200_PROFILING.md forbids waiting ranks on one GPU)
    import os
    import torch
    import torch.distributed as dist
    import paper_1409_7166_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = gridgen.mesh_grid(2, 48, 40, seed=3, pad_pitch=5, h=10e-12, src_start=5e-12, src_width=30e-12)
        grp = P.SlabGroup.p2p(g, rank, world, fuse=2)
        grp.p2p_selftest(0)
        torch.cuda.synchronize()
        dist.barrier()
        out = grp.p2p_selftest(1)
        dist.barrier()
        grp.close()
        q.put((rank, out.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_ipc_mapping_across_processes(pgb, world):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        out = res[r]
        assert out[:world] == [0x5EED0000 + k for k in range(world)]          # every control block
        assert out[world] == (0x5EED0000 + r - 1 if r > 0 else -1)            # lower neighbour's store
        assert out[world + 1] == (0x5EED0000 + r + 1 if r < world - 1 else -1)  # upper neighbour's store
