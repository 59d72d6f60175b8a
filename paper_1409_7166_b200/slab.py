"""Multi-GPU slab partition of a layered mesh (binding of include/pgrid.h's
pg_set_slab / pg_group_*).

The global mesh is cut into contiguous blocks of rows, one per rank; each
rank's slab grid holds its owned rows plus ``ghost`` rows of each neighbour.
The exchange after every sweep launch (convergence max-reduction + ghost-row
halo exchange) runs inside the library: over NCCL between processes
(``SlabGroup.nccl``) or by device copies between slabs of one process
(``SlabGroup.local``, the same protocol on one GPU).  torch.distributed is used
only to broadcast the 128-byte NCCL id.  This module only slices arrays and
marshals arguments.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from .api import Grid


def partition_rows(ny: int, nranks: int) -> List[Tuple[int, int]]:
    """Owned rows [Y0, Y1) of each rank: contiguous blocks whose sizes differ
    by at most one row, in rank order."""
    if nranks < 1 or ny < nranks:
        raise ValueError(f"cannot split {ny} rows over {nranks} ranks")
    base, extra = divmod(ny, nranks)
    out, y = [], 0
    for r in range(nranks):
        h = base + (1 if r < extra else 0)
        out.append((y, y + h))
        y += h
    return out


@dataclass
class SlabSpec:
    rank: int
    nranks: int
    y0: int          # first owned global row
    y1: int          # one past the last owned global row
    lo: int          # first global row held (owned or ghost)
    hi: int          # one past the last global row held
    ghost: int

    @property
    def y_begin(self) -> int:   # owned rows in local row numbering
        return self.y0 - self.lo

    @property
    def y_end(self) -> int:
        return self.y1 - self.lo

    @property
    def parity(self) -> int:    # parity of the global index of local row 0
        return self.lo & 1


def slab_spec(ny: int, rank: int, nranks: int, ghost: int) -> SlabSpec:
    y0, y1 = partition_rows(ny, nranks)[rank]
    if nranks > 1 and (y1 - y0) < ghost:
        raise ValueError(f"slab of {y1 - y0} rows is thinner than the {ghost} ghost rows")
    lo = max(0, y0 - ghost) if rank > 0 else 0
    hi = min(ny, y1 + ghost) if rank < nranks - 1 else ny
    return SlabSpec(rank, nranks, y0, y1, lo, hi, ghost)


def _local_index(m, idx, sp: SlabSpec):
    """Global natural node index -> (inside mask, local natural index)."""
    idx = np.asarray(idx, dtype=np.int64)
    l, r = np.divmod(idx, m.ny * m.nx)
    y, x = np.divmod(r, m.nx)
    inside = (y >= sp.lo) & (y < sp.hi)
    nyl = sp.hi - sp.lo
    return inside, (l * nyl + (y - sp.lo)) * m.nx + x


def slab_mesh(m, sp: SlabSpec):
    """The slab's mesh (rows [lo, hi) of every array, gy of the last local
    row zeroed, pads and loads of those rows): a gridgen.MeshGrid-like object."""
    rows = slice(sp.lo, sp.hi)

    def cut(a):
        if a is None:
            return None
        # always a copy: the caller's arrays must not see the zeroed gy row
        return np.array(np.asarray(a).reshape(m.layers, m.ny, m.nx)[:, rows, :], order="C", copy=True)

    gy = cut(m.gy)
    gy[:, -1, :] = 0.0
    pin, pidx = _local_index(m, m.pad_node, sp)
    s = m.sources
    sin, sidx = _local_index(m, s.node, sp)
    keep = np.flatnonzero(sin)
    cnt = (s.ptr[keep + 1] - s.ptr[keep]).astype(np.int64)
    ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    take = np.concatenate([np.arange(s.ptr[q], s.ptr[q + 1]) for q in keep]) if keep.size else \
        np.zeros(0, np.int64)
    src = type(s)(node=sidx[keep].astype(np.int64), ptr=ptr, t=np.asarray(s.t)[take],
                  i=np.asarray(s.i)[take])
    return replace(m, ny=sp.hi - sp.lo, gx=cut(m.gx), gy=gy, gz=cut(m.gz), cap=cut(m.cap),
                   lz=cut(m.lz), pad_node=pidx[pin].astype(np.int64),
                   pad_g=np.asarray(m.pad_g)[pin],
                   pad_l=None if m.pad_l is None else np.asarray(m.pad_l)[pin], sources=src)


def make_slab_grid(m, sp: SlabSpec, device: bool = True, fuse: Optional[int] = None) -> Grid:
    g = Grid.from_mesh_grid(slab_mesh(m, sp), device=device)
    if fuse is not None:
        g.set_option("fuse", int(fuse))
    L.check(g._lib.pg_set_slab(g._h, sp.y_begin, sp.y_end, sp.parity))
    return g


@dataclass
class GroupResult:
    sweeps: np.ndarray
    stats: L.PgStats
    status: int


class SlabGroup:
    """Slab grids advanced together by pg_group_transient."""

    def __init__(self, handle, grids: Sequence[Grid], specs: Sequence[SlabSpec]):
        self._h = ctypes.c_void_p(handle)
        self._lib = L.load()
        self.grids = list(grids)
        self.specs = list(specs)

    # ----------------------------------------------------------------- create
    @classmethod
    def local(cls, m, nslabs: int, fuse: int = 2, ghost: Optional[int] = None,
              device: bool = True, stream=None, transport: str = "copy",
              options: Optional[dict] = None) -> "SlabGroup":
        """nslabs slabs of mesh m on the current device (the n-rank protocol
        emulated in one process).  transport "copy": per-launch norm max and
        ghost-row copies (the NCCL protocol); "p2p": the peer-memory exchange
        inside the sweep kernel (pg_group_local_p2p).  `options` are set on
        every slab grid before the group is formed."""
        G = ghost if ghost is not None else 2 * fuse
        specs = [slab_spec(m.ny, r, nslabs, G) for r in range(nslabs)]
        grids = [make_slab_grid(m, sp, device, fuse) for sp in specs]
        for g in grids:
            if stream is not None:
                g.set_stream(stream)
            for k, v in (options or {}).items():
                g.set_option(k, int(v))
        arr = (ctypes.c_void_p * nslabs)(*[g._h.value for g in grids])
        out = ctypes.c_void_p()
        fn = L.load().pg_group_local_p2p if transport == "p2p" else L.load().pg_group_local
        if transport not in ("copy", "p2p"):
            raise ValueError("transport must be 'copy' or 'p2p'")
        L.check(fn(nslabs, arr, G, ctypes.byref(out)))
        return cls(out.value, grids, specs)

    @classmethod
    def p2p(cls, m, rank: int, nranks: int, fuse: int = 2, ghost: Optional[int] = None,
            stream=None, group=None, device: bool = True, options: Optional[dict] = None) -> "SlabGroup":
        """This process's slab (one GPU per rank) with the peer-memory exchange:
        CUDA IPC records of all ranks are gathered over torch.distributed (the
        default process group or `group`), then every rank maps its
        neighbours' receive buffers and all control blocks."""
        import torch.distributed as dist
        G = ghost if ghost is not None else 2 * fuse
        sp = slab_spec(m.ny, rank, nranks, G)
        g = make_slab_grid(m, sp, device, fuse)
        if stream is not None:
            g.set_stream(stream)
        for k, v in (options or {}).items():
            g.set_option(k, int(v))
        lib = L.load()
        out = ctypes.c_void_p()
        L.check(lib.pg_group_p2p_create(g._h, nranks, rank, G, ctypes.byref(out)))
        n = ctypes.c_int64()
        L.check(lib.pg_group_p2p_export(out, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_uint8 * n.value)()
        L.check(lib.pg_group_p2p_export(out, buf, n.value, ctypes.byref(n)))
        recs = [None] * nranks
        dist.all_gather_object(recs, bytes(buf), group=group)
        blob = b"".join(recs)
        L.check(lib.pg_group_p2p_connect(out, blob, n.value))
        dist.barrier(group=group)
        return cls(out.value, [g], [sp])

    @classmethod
    def nccl(cls, m, rank: int, nranks: int, fuse: int = 2, ghost: Optional[int] = None,
             stream=None, group=None, device: bool = True) -> "SlabGroup":
        """This process's slab (one GPU per rank) in an NCCL group; collective
        over the default torch.distributed process group (or `group`)."""
        import torch
        import torch.distributed as dist
        G = ghost if ghost is not None else 2 * fuse
        sp = slab_spec(m.ny, rank, nranks, G)
        g = make_slab_grid(m, sp, device, fuse)
        if stream is not None:
            g.set_stream(stream)
        lib = L.load()
        idbuf = (ctypes.c_uint8 * 128)()
        if rank == 0:
            L.check(lib.pg_nccl_unique_id(idbuf))
        t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0, group=group)
        idbuf = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        out = ctypes.c_void_p()
        L.check(lib.pg_group_nccl(g._h, idbuf, nranks, rank, G, ctypes.byref(out)))
        return cls(out.value, [g], [sp])

    # -------------------------------------------------------------- transient
    def transient(self, h, steps, tol=1e-10, omega=1.0, max_sweeps=100000,
                  raise_on_noconv=True, cont=False) -> GroupResult:
        """pg_group_transient (from x(0)) or, with cont=True,
        pg_group_transient_continue (from the slabs' current state)."""
        sweeps = np.zeros(steps + 1, dtype=np.int64)
        st = L.PgStats()
        fn = self._lib.pg_group_transient_continue if cont else self._lib.pg_group_transient
        code = fn(self._h, float(h), int(steps), float(tol), float(omega),
                  int(max_sweeps), sweeps.ctypes.data, ctypes.byref(st))
        if code not in (L.PG_OK, L.PG_ENOCONV) or (code == L.PG_ENOCONV and raise_on_noconv):
            L.check(code)
        return GroupResult(sweeps=sweeps, stats=st, status=code)

    def p2p_selftest(self, phase: int):
        """pg_group_p2p_selftest (CUDA-IPC groups): phase 0 marks, phase 1
        returns the marks read through the mappings (nranks + 2 int64)."""
        out = np.zeros(self.specs[0].nranks + 2, dtype=np.int64)
        L.check(self._lib.pg_group_p2p_selftest(self._h, int(phase), out.ctypes.data))
        return out

    def owned_voltages(self, m) -> List[Tuple[SlabSpec, np.ndarray]]:
        """[(spec, V)] per slab of this process: V[l, y - y0, x] for owned rows."""
        out = []
        for g, sp in zip(self.grids, self.specs):
            V = g.voltages().reshape(m.layers, sp.hi - sp.lo, m.nx)
            out.append((sp, V[:, sp.y_begin:sp.y_end, :].copy()))
        return out

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.pg_group_destroy(self._h)
            self._h = ctypes.c_void_p()
        for g in self.grids:
            g.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
