import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import gridgen
import paper_1409_7166_b200 as P
from test_gpu_slab import single
def case(shape, n, F, G, label, rows=0, k=1):
    g = gridgen.mesh_grid(*shape, seed=1+34+70+2, pad_pitch=5, src_frac=0.4, h=10e-12, src_start=20e-12, src_width=40e-12)
    r1, V1 = single(P, g, 1, 0.0, 1.7, k, F)
    grp = P.SlabGroup.local(g, n, fuse=F, ghost=G)
    if rows:
        for q in grp.grids: q.set_option("rows", rows)
    grp.transient(g.h, 1, tol=0.0, omega=1.7, max_sweeps=k)
    Vn = np.zeros((g.layers, g.ny, g.nx))
    for sp, Vo in grp.owned_voltages(g):
        Vn[:, sp.y0:sp.y1, :] = Vo
    specs = grp.specs
    grp.close()
    D = np.abs(Vn - V1)
    bad = np.argwhere(D > 1e-13)
    print(label, [(s.y0, s.lo, s.hi) for s in specs], "max", D.max(), "bad (l,y)", sorted(set((int(a), int(b)) for a, b, c in bad))[:10])
case((1,34,70), 2, 1, 2, "base")
case((1,34,70), 2, 1, 4, "G=4")
case((1,34,64), 2, 1, 2, "NX=64")
case((1,68,70), 2, 1, 2, "NY=68")
case((1,34,70), 2, 1, 2, "rows=17", rows=17)
case((1,34,70), 3, 1, 2, "n=3")
case((1,34,200), 2, 1, 2, "NX=200")
