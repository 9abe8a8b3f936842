"""Exploration: convergence of the accuracy test for other wave directions k (velocity = k)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2407_00656_b200 import hgks, workloads as W

def ic(mi, t, k):
    k = np.asarray(k, float)
    sp = k @ k
    f = lambda x, y, z: 1 + 0.2 * np.sin(np.pi * (k[0] * x + k[1] * y + k[2] * z - sp * t))
    rho = W.tet_cell_means(mi, f, order=7)
    Q = np.empty((mi.n_cells, 5)); Q[:, 0] = rho
    for a in range(3): Q[:, 1 + a] = k[a] * rho
    Q[:, 4] = 1 / 0.4 + 0.5 * sp * rho
    return Q

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-10
for k in ([-1, 1, 1], [1, 0, 0], [1, 1, 0]):
    prev = None
    for N in (10, 20, 40):
        mi = W.kuhn_box(N)
        s = hgks.Solver(hgks.Mesh(mi), ic(mi, 0.0, k), hgks.SolverConfig(cfl=0.3, eps=eps))
        T = 0.5
        while s.step(500, t_stop=T)["t"] < T:
            pass
        Q, _, t = s.get_state()
        e = Q[:, 0] - ic(mi, T, k)[:, 0]
        L1 = float(np.abs(e).mean())
        print(json.dumps(dict(eps=eps, k=k, N=N, L1=L1, order=(np.log2(prev / L1) if prev else None))), flush=True)
        prev = L1
