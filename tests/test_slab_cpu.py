"""Multi-rank slab partition on CPU (-m "not gpu"): the product's partition
helpers (paper_1409_7166_b200.slab) and the exchange protocol of
pg_group_transient run across world_size 2 and 3 processes with
the torch.distributed gloo backend, the sweeps done by the numpy model of
tests/slab_model.py.  Bar: every rank's owned rows equal the monolithic model
bit for bit (same arithmetic, same global red-black numbering), the stopping
decisions are the same on every rank, and the monolithic model equals the
oracle's red-black iteration to rounding."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import gridgen  # noqa: E402
from paper_1409_7166_b200 import slab  # noqa: E402
import slab_model  # noqa: E402


def mesh(seed=3, dims=(3, 30, 14)):
    return gridgen.mesh_grid(*dims, seed=seed, pad_pitch=4, src_frac=0.5, h=10e-12,
                             src_start=10e-12, src_width=40e-12)


# ------------------------------------------------------------ partition helpers
def test_partition_rows():
    for ny, n in [(10, 1), (10, 3), (1024, 8), (7, 7)]:
        parts = slab.partition_rows(ny, n)
        assert parts[0][0] == 0 and parts[-1][1] == ny
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab.partition_rows(3, 4)


@pytest.mark.parametrize("L,n,G", [(3, 2, 4), (3, 3, 2), (3, 4, 6), (1, 3, 2)])
def test_slab_mesh_rows_pads_sources(L, n, G):
    m = mesh(dims=(L, 30, 14))
    gy_before = m.gy.copy()
    gx, gy, gz, cap = slab_model.arrays(m)
    owned_pads, owned_src = 0, 0
    for r in range(n):
        sp = slab.slab_spec(m.ny, r, n, G)
        sm = slab.slab_mesh(m, sp)
        assert sm.ny == sp.hi - sp.lo
        assert sp.y_begin == (G if r > 0 else 0)
        assert sp.y_end == sm.ny - (G if r < n - 1 else 0)
        lgx, lgy, lgz, lcap = slab_model.arrays(sm)
        np.testing.assert_array_equal(lgx, gx[:, sp.lo:sp.hi])
        np.testing.assert_array_equal(lgz, gz[:, sp.lo:sp.hi])
        np.testing.assert_array_equal(lcap, cap[:, sp.lo:sp.hi])
        np.testing.assert_array_equal(lgy[:, :-1], gy[:, sp.lo:sp.hi - 1])
        assert np.all(lgy[:, -1] == 0)
        # pads / loads: exactly those of rows [lo, hi), same values
        np.testing.assert_array_equal(slab_model.pad_sum(sm), slab_model.pad_sum(m)[:, sp.lo:sp.hi])
        for t in (15e-12, 30e-12):
            np.testing.assert_array_equal(slab_model.loads(sm, t), slab_model.loads(m, t)[:, sp.lo:sp.hi])
        own = np.zeros(sm.layers * sm.ny * sm.nx, bool).reshape(sm.layers, sm.ny, sm.nx)
        own[:, sp.y_begin:sp.y_end] = True
        owned_pads += int(own.reshape(-1)[sm.pad_node].sum())
        owned_src += int(own.reshape(-1)[sm.sources.node].sum())
    assert owned_pads == m.pad_node.size and owned_src == m.sources.node.size
    np.testing.assert_array_equal(m.gy, gy_before)   # the global arrays are not modified
    with pytest.raises(ValueError):
        slab.slab_spec(8, 1, 4, 3)       # slabs of 2 rows cannot hold 3 ghost rows


# ----------------------------------------------------------- gloo protocol run
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, F, steps, k_max, tol, omega, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    m = mesh()
    G = 2 * F
    sp = slab.slab_spec(m.ny, rank, world, G)
    sm = slab.slab_mesh(m, sp)
    rows = (1 if rank > 0 else 0, sm.ny - 1 if rank < world - 1 else sm.ny)
    md = slab_model.Model(sm, row0=sp.lo, rows=rows, owned=(sp.y_begin, sp.y_end))

    def exchange():
        ops = []
        V = md.V
        recv_lo = torch.zeros((sm.layers, G, sm.nx), dtype=torch.float64)
        recv_hi = torch.zeros((sm.layers, G, sm.nx), dtype=torch.float64)
        if rank > 0:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(
                np.ascontiguousarray(V[:, sp.y_begin:sp.y_begin + G])), rank - 1))
            ops.append(dist.P2POp(dist.irecv, recv_lo, rank - 1))
        if rank < world - 1:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(
                np.ascontiguousarray(V[:, sp.y_end - G:sp.y_end])), rank + 1))
            ops.append(dist.P2POp(dist.irecv, recv_hi, rank + 1))
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        if rank > 0:
            V[:, sp.y_begin - G:sp.y_begin] = recv_lo.numpy()
        if rank < world - 1:
            V[:, sp.y_end:sp.y_end + G] = recv_hi.numpy()

    def allmax(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sweeps = slab_model.run([md], exchange, allmax, steps, F, k_max, tol, omega)
    out[rank] = (sp.y0, sp.y1, md.V[:, sp.y_begin:sp.y_end].copy(), sweeps)
    dist.destroy_process_group()


def _run_world(world, F, steps, k_max, tol, omega):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, F, steps, k_max, tol, omega, out), nprocs=world, join=True)
        return dict(out)


@pytest.mark.parametrize("world,F,tol", [(2, 2, 0.0), (3, 1, 0.0), (2, 2, 1e-11), (3, 3, 1e-11)])
def test_gloo_slabs_equal_monolithic(world, F, tol):
    steps, k_max, omega = 3, 6 if tol == 0 else 100000, 1.7
    res = _run_world(world, F, steps, k_max, tol, omega)
    m = mesh()
    mono = slab_model.Model(m)
    sweeps = slab_model.run([mono], lambda: None, lambda x: x, steps, F, k_max, tol, omega)
    V = np.zeros_like(mono.V)
    for r in range(world):
        y0, y1, Vo, sw = res[r]
        V[:, y0:y1] = Vo
        assert sw == sweeps, (r, sw, sweeps)
    np.testing.assert_array_equal(V, mono.V)


def test_monolithic_model_is_the_oracle_iteration():
    # the model used above is the red-black SOR of Eq. (13)/(15)
    from oracle import netlist, nodal, pwl
    m = mesh()
    steps, k, omega = 3, 4, 1.7
    mono = slab_model.Model(m)
    slab_model.run([mono], lambda: None, lambda x: x, steps, 1, k, 0.0, omega)
    nl = netlist.from_mesh(m)
    ro = nodal.NodalOracle(nl).transient(m.h, steps, tol=0.0, omega=omega, max_sweeps=k,
                                         order=nodal.red_black_order(m.layers, m.ny, m.nx),
                                         Itab=pwl.node_currents_table(nl, m.h, steps))
    np.testing.assert_allclose(mono.V.reshape(-1), ro.V[-1], rtol=0, atol=1e-12)


# ------------------------------------------ peer-memory protocol (gloo model)
def _worker_p2p(rank, world, port, F, steps, k_max, tol, omega, repeat, out):
    """The peer-memory exchange of DESIGN.md §10 with real processes: receive
    buffers double-buffered by launch epoch e (launch e reads parity e & 1,
    its boundary rows land in the neighbours' parity (e + 1) & 1 buffers),
    the epoch counts working launches and continues across transients, the
    receive buffers are seeded from x(0) at a transient's start and unpacked
    into V after a step's last launch.  Remote stores are modelled by
    send/recv into the parity buffer, the arrival wait by their completion and
    the remote norm maxima by an allreduce."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    m = mesh()
    G = 2 * F
    sp = slab.slab_spec(m.ny, rank, world, G)
    sm = slab.slab_mesh(m, sp)
    rows = (1 if rank > 0 else 0, sm.ny - 1 if rank < world - 1 else sm.ny)
    md = slab_model.Model(sm, row0=sp.lo, rows=rows, owned=(sp.y_begin, sp.y_end))
    shape = (sm.layers, G, sm.nx)
    recv = {(side, p): np.zeros(shape) for side in ("lo", "hi") for p in (0, 1)}
    lo, hi = rank > 0, rank < world - 1
    epoch = 0

    def ghosts_from(p):
        if lo:
            md.V[:, sp.y_begin - G:sp.y_begin] = recv[("lo", p)]
        if hi:
            md.V[:, sp.y_end:sp.y_end + G] = recv[("hi", p)]

    def store_to_neighbours(p):
        ops, bufs = [], {}
        if lo:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(
                md.V[:, sp.y_begin:sp.y_begin + G])), rank - 1))
            bufs["lo"] = torch.zeros(shape, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, bufs["lo"], rank - 1))
        if hi:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(
                md.V[:, sp.y_end - G:sp.y_end])), rank + 1))
            bufs["hi"] = torch.zeros(shape, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, bufs["hi"], rank + 1))
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        for side, t in bufs.items():
            recv[(side, p)] = t.numpy().copy()

    def allmax(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    runs = []
    for _ in range(repeat):
        md.V[:] = m.vdd                           # x(0)
        if lo:                                    # seed parity epoch & 1 from x(0)
            recv[("lo", epoch & 1)] = md.V[:, sp.y_begin - G:sp.y_begin].copy()
        if hi:
            recv[("hi", epoch & 1)] = md.V[:, sp.y_end:sp.y_end + G].copy()
        sweeps = []
        for s in range(1, steps + 1):
            b = md.rhs(s)
            k = 0
            while True:
                ghosts_from(epoch & 1)
                d = md.launch(b, F, omega)
                store_to_neighbours((epoch + 1) & 1)
                d = allmax(d)                     # pnorm[e & 3] after the arrival wait
                epoch += 1
                k += F
                if (tol > 0 and d < tol) or k >= k_max:
                    break
            ghosts_from(epoch & 1)                # end-of-step unpack into V
            sweeps.append(k)
        runs.append((md.V[:, sp.y_begin:sp.y_end].copy(), sweeps))
    out[rank] = (sp.y0, sp.y1, runs, epoch)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,tol", [(2, 0.0), (3, 1e-11)])
def test_gloo_p2p_protocol_equals_monolithic(world, tol):
    F, steps, omega, repeat = 2, 3, 1.7, 2
    k_max = 6 if tol == 0 else 100000
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker_p2p, args=(world, port, F, steps, k_max, tol, omega, repeat, out), nprocs=world,
                 join=True)
        res = dict(out)
    m = mesh()
    mono = slab_model.Model(m)
    sweeps = slab_model.run([mono], lambda: None, lambda x: x, steps, F, k_max, tol, omega)
    epochs = {res[r][3] for r in range(world)}
    assert epochs == {repeat * sum(sweeps) // F}      # every rank counted the same launches
    for rep in range(repeat):                         # a second transient continues the epochs
        V = np.zeros_like(mono.V)
        for r in range(world):
            y0, y1, runs, _ = res[r]
            Vo, sw = runs[rep]
            V[:, y0:y1] = Vo
            assert sw == sweeps, (r, rep, sw, sweeps)
        np.testing.assert_array_equal(V, mono.V)
