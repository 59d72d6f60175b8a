"""Python binding of the C ABI (argument marshalling only; every step of the
hot path runs in libpgb200.so's sm_100a kernels).

Arrays may be numpy arrays (host, ``PG_MEM_HOST``) or CUDA torch tensors
(device, ``PG_MEM_DEVICE``); torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib as L


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _mem_of(*arrs) -> int:
    kinds = set()
    for a in arrs:
        if a is None:
            continue
        if _is_torch(a):
            kinds.add(L.PG_MEM_DEVICE if a.is_cuda else L.PG_MEM_HOST)
        else:
            kinds.add(L.PG_MEM_HOST)
    if len(kinds) > 1:
        raise ValueError("all arrays of one call must live in the same memory (host or device)")
    return kinds.pop() if kinds else L.PG_MEM_HOST


class _Arr:
    """Holds a contiguous buffer of the required dtype and exposes its address."""

    def __init__(self, x, dtype):
        if x is None:
            self.obj, self.ptr = None, None
            return
        if _is_torch(x):
            import torch
            tdt = {np.float64: torch.float64, np.int64: torch.int64}[dtype]
            t = x.to(tdt).contiguous()
            self.obj, self.ptr = t, t.data_ptr()
        else:
            a = np.ascontiguousarray(x, dtype=dtype)
            self.obj, self.ptr = a, a.ctypes.data
        if self.ptr == 0:
            self.ptr = None


def _d(x):
    return _Arr(x, np.float64)


def _len(x) -> int:
    return 0 if x is None else int(x.numel() if _is_torch(x) else np.size(x))


def _need(name, x, n):
    """The C side reads / writes exactly n elements: refuse other sizes."""
    if x is not None and _len(x) != n:
        raise ValueError(f"{name} has {_len(x)} elements, expected {n}")


def _i(x):
    return _Arr(x, np.int64)


@dataclass
class TransientResult:
    probes: Optional[np.ndarray]   # [(steps+1), n_probe] (host) or the device tensor passed in
    sweeps: np.ndarray             # per-step sweep counts, [steps+1]
    stats: L.PgStats
    status: int


class Grid:
    """A power grid resident on the current CUDA device."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)
        self._lib = L.load()

    # ----------------------------------------------------------------- create
    @classmethod
    def mesh(cls, layers, ny, nx, gx, gy, gz, cap, pad_node, pad_g, vdd=1.0, lz=None,
             pad_l=None) -> "Grid":
        lib = L.load()
        n = int(layers) * int(ny) * int(nx)
        for name, a in (("gx", gx), ("gy", gy), ("gz", gz), ("cap", cap), ("lz", lz)):
            _need(name, a, n)
        npad = _len(pad_node)
        _need("pad_g", pad_g, npad)
        _need("pad_l", pad_l, npad)
        mem = _mem_of(gx, gy, gz, cap, lz)
        pmem = _mem_of(pad_node, pad_g, pad_l)
        if pmem != mem:
            raise ValueError("pads must live in the same memory as the grid arrays")
        A = [_d(gx), _d(gy), _d(gz), _d(lz), _d(cap)]
        pn, pg, pl = _i(pad_node), _d(pad_g), _d(pad_l)
        out = ctypes.c_void_p()
        L.check(lib.pg_create_mesh(int(layers), int(ny), int(nx), A[0].ptr, A[1].ptr, A[2].ptr,
                                   A[3].ptr, A[4].ptr, npad, pn.ptr, pg.ptr, pl.ptr, float(vdd),
                                   mem, ctypes.byref(out)))
        return cls(out.value)

    @classmethod
    def from_mesh_grid(cls, m, device: bool = False) -> "Grid":
        """From a gridgen.MeshGrid-like object (attributes layers, ny, nx, gx,
        gy, gz, cap, pad_node, pad_g, vdd, lz, pad_l, sources)."""
        conv = _to_device if device else (lambda a: a)
        g = cls.mesh(m.layers, m.ny, m.nx, conv(m.gx), conv(m.gy), conv(m.gz), conv(m.cap),
                     conv(m.pad_node), conv(m.pad_g), m.vdd, conv(m.lz), conv(m.pad_l))
        s = m.sources
        g.set_sources(conv(s.node), conv(s.ptr), conv(s.t), conv(s.i))
        return g

    @classmethod
    def csr(cls, n, bu, bv, bg, cap, pad_node, pad_g, vdd=1.0) -> "Grid":
        lib = L.load()
        m = _len(bu)
        _need("bv", bv, m)
        _need("bg", bg, m)
        _need("cap", cap, int(n))
        _need("pad_g", pad_g, _len(pad_node))
        mem = _mem_of(bu, bv, bg, cap, pad_node, pad_g)
        u, v, w, c = _i(bu), _i(bv), _d(bg), _d(cap)
        pn, pg = _i(pad_node), _d(pad_g)
        out = ctypes.c_void_p()
        L.check(lib.pg_create_csr(int(n), int(len(bu)), u.ptr, v.ptr, w.ptr, c.ptr,
                                  int(len(pad_node)), pn.ptr, pg.ptr, float(vdd), mem,
                                  ctypes.byref(out)))
        return cls(out.value)

    @classmethod
    def from_edge_grid(cls, e, device: bool = False) -> "Grid":
        conv = _to_device if device else (lambda a: a)
        g = cls.csr(e.n, conv(e.eu), conv(e.ev), conv(e.eg), conv(e.cap), conv(e.pad_node),
                    conv(e.pad_g), e.vdd)
        s = e.sources
        g.set_sources(conv(s.node), conv(s.ptr), conv(s.t), conv(s.i))
        return g

    # ------------------------------------------------------------------ state
    def set_sources(self, node, ptr, t, i):
        ns = _len(node)
        _need("ptr", ptr, ns + 1)
        npts = int(ptr[-1]) if ns > 0 else _len(t)
        _need("t", t, npts)
        _need("i", i, npts)
        mem = _mem_of(node, ptr, t, i)
        a, b, c, d = _i(node), _i(ptr), _d(t), _d(i)
        L.check(self._lib.pg_set_sources(self._h, int(len(node)), a.ptr, b.ptr, c.ptr, d.ptr, mem))

    def set_voltages(self, v):
        _need("v", v, self.n)
        a = _d(v)
        L.check(self._lib.pg_set_voltages(self._h, a.ptr, _mem_of(v)))

    def voltages(self, out=None):
        if out is None:
            out = np.empty(self.n)
        _need("out", out, self.n)
        mem = _mem_of(out)
        L.check(self._lib.pg_get_voltages(self._h, _ptr_of(out), mem))
        return out

    def set_stream(self, stream):
        """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None."""
        h = getattr(stream, "cuda_stream", stream)
        L.check(self._lib.pg_set_stream(self._h, ctypes.c_void_p(h or 0)))

    def set_option(self, key: str, value: int):
        L.check(self._lib.pg_set_option(self._h, key.encode(), int(value)))

    def info(self):
        n, l, y, x, c = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        L.check(self._lib.pg_info(self._h, ctypes.byref(n), ctypes.byref(l), ctypes.byref(y),
                                  ctypes.byref(x), ctypes.byref(c)))
        return dict(n=n.value, layers=l.value, ny=y.value, nx=x.value, n_colors=c.value)

    @property
    def n(self) -> int:
        return self.info()["n"]

    # -------------------------------------------------------------- Algorithm 1
    def transient(self, h, steps, tol=1e-10, omega=1.0, method="rbsor", max_sweeps=100000,
                  probes=None, probe_out=None, raise_on_noconv=True, cont=False) -> TransientResult:
        """pg_transient (from x(0)) or, with cont=True, pg_transient_continue
        (from the state the previous call left)."""
        m = {"rbsor": L.PG_METHOD_RBSOR, "jacobi": L.PG_METHOD_JACOBI}[method]
        npr = 0 if probes is None else int(len(probes))
        if npr and probe_out is None:
            if _is_torch(probes) and probes.is_cuda:
                import torch
                probe_out = torch.empty((steps + 1, npr), dtype=torch.float64, device=probes.device)
            else:
                probe_out = np.empty((steps + 1, npr))
        if npr:
            _need("probe_out", probe_out, (int(steps) + 1) * npr)
        mem = _mem_of(probes, probe_out) if npr else L.PG_MEM_HOST
        pa = _i(probes)
        sweeps = np.zeros(steps + 1, dtype=np.int64)
        st = L.PgStats()
        fn = self._lib.pg_transient_continue if cont else self._lib.pg_transient
        code = fn(self._h, float(h), int(steps), float(tol), float(omega), m, int(max_sweeps), npr,
                  pa.ptr, _ptr_of(probe_out) if npr else None, mem, sweeps.ctypes.data,
                  ctypes.byref(st))
        if code not in (L.PG_OK, L.PG_ENOCONV) or (code == L.PG_ENOCONV and raise_on_noconv):
            L.check(code)
        return TransientResult(probes=probe_out if npr else None, sweeps=sweeps, stats=st,
                               status=code)

    def estimate_omega(self, h, sweeps=2000):
        """(rho_Jacobi, omega_opt) by Young's formula (pg_estimate_omega)."""
        rho, om = ctypes.c_double(), ctypes.c_double()
        L.check(self._lib.pg_estimate_omega(self._h, float(h), int(sweeps), ctypes.byref(rho),
                                            ctypes.byref(om)))
        return rho.value, om.value

    def tune_omega(self, h, steps=8, tol=1e-10, n=6, d_omega=4e-4):
        """(omega, sweeps per candidate) from pg_tune_omega: Young's omega_b and
        n - 1 candidates above it, each run for the first `steps` time steps."""
        om = ctypes.c_double()
        sw = np.zeros(int(n), dtype=np.int64)
        L.check(self._lib.pg_tune_omega(self._h, float(h), int(steps), float(tol), int(n), float(d_omega),
                                        ctypes.byref(om), sw.ctypes.data))
        return om.value, sw

    def dc(self, t=0.0, tol=1e-10, omega=1.9, method="rbsor", max_sweeps=1000000,
           raise_on_noconv=True):
        """DC operating point G v = G0 Vdd - i(t) (pg_dc); returns the stats.
        Voltages: ``voltages()``."""
        m = {"rbsor": L.PG_METHOD_RBSOR, "jacobi": L.PG_METHOD_JACOBI}[method]
        st = L.PgStats()
        code = self._lib.pg_dc(self._h, float(t), float(tol), float(omega), m, int(max_sweeps),
                               ctypes.byref(st))
        if code not in (L.PG_OK, L.PG_ENOCONV) or (code == L.PG_ENOCONV and raise_on_noconv):
            L.check(code)
        return st

    # ------------------------------------------------------------------ cleanup
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.pg_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def release_memory(device: int = -1) -> None:
    """pg_release_memory: return the freed blocks the library's device memory
    pools keep cached (for the next grid) to the CUDA driver; -1 = all devices."""
    L.check(L.load().pg_release_memory(int(device)))


def _ptr_of(x):
    if _is_torch(x):
        if not x.is_contiguous() or x.dtype.__str__() != "torch.float64":
            raise ValueError("output tensors must be contiguous float64")
        return x.data_ptr()
    if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous):
        raise ValueError("output arrays must be contiguous float64")
    return x.ctypes.data


def _to_device(a):
    if a is None:
        return None
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()
