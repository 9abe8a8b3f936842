"""Accuracy test (Table 3) on the GPU path: L1/L2 at t=2 and orders.

python scripts/convergence_gpu.py [--N 10 20 40] [--omega-pow 1] [--cfl 0.3]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2407_00656_b200 import hgks, workloads as W

T3 = {10: 6.6070e-2, 20: 8.7117e-3, 40: 1.0994e-3, 80: 1.3768e-4, 160: 1.7252e-5}
ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, nargs="+", default=[10, 20, 40])
ap.add_argument("--omega-pow", type=int, default=1)
ap.add_argument("--cfl", type=float, default=0.3)
ap.add_argument("--eps", type=float, default=None)
ap.add_argument("--precision", type=int, default=64, choices=[64, 32])
ap.add_argument("--dq0-mode", type=int, default=0, help="SURVEY Q9 reading: 0 R9, 1 R9k, 2 R9s")
ap.add_argument("--jitter", type=float, default=0.0, help="interior node jitter (fraction of h), seed 656")
args = ap.parse_args()
prev = None
for N in args.N:
    mi = W.kuhn_box(N, jitter=args.jitter)
    Q0 = W.advection_ic(mi)
    s = hgks.Solver(hgks.Mesh(mi), Q0, hgks.SolverConfig(cfl=args.cfl, omega_pow=args.omega_pow, eps=args.eps,
                                                            precision=args.precision, dq0_mode=args.dq0_mode))
    t0 = time.time()
    steps = 0
    while True:
        info = s.step(200, t_stop=2.0)
        steps += info["steps_done"]
        if info["t"] >= 2.0:
            break
    Q, gid, t = s.get_state()
    v = mi.xyz[mi.cell_nodes[:, :4]]  # tet volumes |det| / 6 (uniform for the plain Kuhn box)
    V = np.abs(np.einsum("ij,ij->i", v[:, 1] - v[:, 0], np.cross(v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]))) / 6.0
    e = Q[:, 0] - W.advection_ic(mi, t=t)[:, 0]
    VD = float(V.sum())
    L1 = float(np.sum(np.abs(e) * V) / VD)
    L2 = float(np.sqrt(np.sum(e * e * V)) / VD)
    order = np.log2(prev / L1) if prev else None
    print(json.dumps(dict(N=N, steps=steps, t=t, L1=L1, L2=L2, order=order, paper_L1=T3.get(N),
                          ratio=L1 / T3[N] if N in T3 else None, fallbacks=info["fallbacks"],
                          omega_pow=args.omega_pow, cfl=args.cfl, dq0_mode=args.dq0_mode, precision=args.precision, jitter=args.jitter, secs=time.time() - t0)), flush=True)
    prev = L1
    s.close()
