"""Time the CPU oracle (mesh build + steps) and its peak RSS on a bench-size workload.
python scripts/oracle_probe.py c5|c4|c3|c2 [steps]   (probe for sizing the full-size parity tests)"""
import os, resource, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_2407_00656_b200 import workloads as W

wl = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
t0 = time.time()
if wl in ("c2", "c5"):
    N = 48 if wl == "c2" else 110
    mi = W.kuhn_box(N)
    Q0 = W.advection_ic(mi)
    cfg = O.OracleConfig(cfl=0.3)
else:
    N, ma, re = (35, 0.2535, 118.0) if wl == "c3" else (70, 1.5, 300.0)
    mi = W.sphere_shell(N)
    Q0 = W.random_smooth_ic(mi) if hasattr(W, "random_smooth_ic") else W.uniform_state(mi.n_cells, 1.0, (ma, 0, 0), 1 / 1.4)
    cfg = O.OracleConfig(cfl=0.5, tau_mode=1, mu_inf=ma / re, c1=1.0, t_inf=1 / 1.4, freestream=(1.0, ma, 0, 0, 1 / 1.4))
t1 = time.time()
m = O.OracleMesh(mi)
t2 = time.time()
s = O.OracleSolver(m, Q0, cfg)
t3 = time.time()
s.step(steps)
t4 = time.time()
rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
print(f"{wl}: cells {m.n_cells} gen {t1-t0:.1f}s mesh {t2-t1:.1f}s solver {t3-t2:.1f}s {steps} steps {t4-t3:.1f}s "
      f"({m.n_cells*steps/(t4-t3):.3g} cell-updates/s, {s.threads} threads) peak RSS {rss:.1f} GB", flush=True)
