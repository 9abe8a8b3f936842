"""Exploration: accuracy test with the advection direction (1,1,1) aligned with the
Kuhn diagonal (default) vs not aligned ((-1,1,1): mirrored split)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2407_00656_b200 import hgks, workloads as W

def ic(mi, t, sx):
    f = lambda x, y, z: 1 + 0.2 * np.sin(np.pi * (sx * x + y + z - 3 * t))
    rho = W.tet_cell_means(mi, f, order=7)
    Q = np.empty((mi.n_cells, 5)); Q[:, 0] = rho; Q[:, 1] = sx * rho; Q[:, 2] = rho; Q[:, 3] = rho
    Q[:, 4] = 1 / 0.4 + 1.5 * rho
    return Q

for sx in (1.0, -1.0):
    prev = None
    for N in (10, 20, 40):
        mi = W.kuhn_box(N)
        s = hgks.Solver(hgks.Mesh(mi), ic(mi, 0.0, sx), hgks.SolverConfig(cfl=0.3))
        while s.step(500, t_stop=2.0)["t"] < 2.0:
            pass
        Q, _, t = s.get_state()
        e = Q[:, 0] - ic(mi, 2.0, sx)[:, 0]
        L1 = float(np.abs(e).mean())
        print(json.dumps(dict(sx=sx, N=N, L1=L1, order=(np.log2(prev / L1) if prev else None))), flush=True)
        prev = L1
