"""CPU model of the slab protocol (test helper, numpy): a vectorised
red-black SOR on a layered mesh's raw arrays, the fused launch of F sweeps
over a slab's local rows (outermost ghost rows held fixed, as the kernel's
halo recompute does), and the exchange after every launch.  Used by
tests/test_slab_cpu.py to check, with real inter-process communication
(torch.distributed gloo), that the product's partition (paper_1409_7166_b200.slab)
plus G = 2F ghost rows exchanged after every launch reproduces the monolithic
iteration bit for bit.  Not product code; the GPU protocol is checked against
the single-grid GPU run in tests/test_gpu_slab.py."""
import numpy as np


def arrays(m):
    L, NY, NX = m.layers, m.ny, m.nx
    r = lambda a: np.asarray(a, dtype=np.float64).reshape(L, NY, NX)
    return r(m.gx), r(m.gy), r(m.gz), r(m.cap)


def pad_sum(m):
    out = np.zeros(m.layers * m.ny * m.nx)
    np.add.at(out, np.asarray(m.pad_node), np.asarray(m.pad_g))
    return out.reshape(m.layers, m.ny, m.nx)


def loads(m, t):
    s = m.sources
    out = np.zeros(m.layers * m.ny * m.nx)
    for k in range(s.node.shape[0]):
        tt, ii = s.t[s.ptr[k]:s.ptr[k + 1]], s.i[s.ptr[k]:s.ptr[k + 1]]
        out[s.node[k]] += np.interp(t, tt, ii)
    return out.reshape(m.layers, m.ny, m.nx)


def colour(m, row0):
    l, y, x = np.meshgrid(np.arange(m.layers), np.arange(m.ny) + row0, np.arange(m.nx), indexing="ij")
    return ((l + y + x) & 1) == 0


def neighbour_sum(V, gx, gy, gz, b):
    S = b.copy()
    S[:, :, 1:] += gx[:, :, :-1] * V[:, :, :-1]
    S[:, :, :-1] += gx[:, :, :-1] * V[:, :, 1:]
    S[:, 1:, :] += gy[:, :-1, :] * V[:, :-1, :]
    S[:, :-1, :] += gy[:, :-1, :] * V[:, 1:, :]
    S[1:] += gz[:-1] * V[:-1]
    S[:-1] += gz[:-1] * V[1:]
    return S


class Model:
    """One (slab or whole) mesh with the iteration state."""

    def __init__(self, m, row0=0, rows=None, owned=None):
        self.m = m
        self.gx, self.gy, self.gz, self.cap = arrays(m)
        self.pads = pad_sum(m)
        d = self.cap / m.h + self.pads + self.gx + self.gy + self.gz
        d[:, :, 1:] += self.gx[:, :, :-1]
        d[:, 1:, :] += self.gy[:, :-1, :]
        d[1:] += self.gz[:-1]
        self.invd = 1.0 / d
        self.red = colour(m, row0)
        self.rows = rows or (0, m.ny)        # rows the sweep updates
        self.owned = owned or (0, m.ny)      # rows counted / compared
        self.V = np.full((m.layers, m.ny, m.nx), m.vdd)

    def rhs(self, s):
        m = self.m
        return self.cap / m.h * self.V + self.pads * m.vdd - loads(m, s * m.h)

    def launch(self, b, F, omega):
        """F red-black sweeps; returns max |dV| of the last sweep on owned rows."""
        r0, r1 = self.rows
        o0, o1 = self.owned
        upd = np.zeros(self.V.shape, dtype=bool)
        upd[:, r0:r1, :] = True
        dmax = 0.0
        for f in range(F):
            last = np.zeros(self.V.shape)
            for c in (self.red, ~self.red):
                S = neighbour_sum(self.V, self.gx, self.gy, self.gz, b)
                Vn = self.V + omega * (S * self.invd - self.V)
                mask = c & upd
                last[mask] = np.abs(Vn - self.V)[mask]
                self.V[mask] = Vn[mask]
            dmax = float(last[:, o0:o1, :].max())
        return dmax


def run(models, exchange, allmax, steps, F, k_max, tol, omega):
    """Algorithm 1 over the given models (one per local slab) with `exchange()`
    after every launch and `allmax(x)` the global max of the norm."""
    sweeps = []
    for s in range(1, steps + 1):
        bs = [md.rhs(s) for md in models]
        k = 0
        while True:
            d = max(md.launch(b, F, omega) for md, b in zip(models, bs))
            d = allmax(d)
            exchange()
            k += F
            if (tol > 0 and d < tol) or k >= k_max:
                break
        sweeps.append(k)
    return sweeps
