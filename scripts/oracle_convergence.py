"""Run the CPU oracle on the accuracy test to t=2 and write
tests/golden/oracle_convergence.json.  Calls only oracle/ and the input
generators (no CUDA path).  Usage: python scripts/oracle_convergence.py 10 20"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2407_00656_b200 import workloads as W

out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                        "oracle_convergence.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
# CFL 0.7: the reading under which the GPU path reproduces T3 at N = 20, 40, 80 within 2 %
# (R6a, profiles/r02/t3_readings.md); override with CFL=...
cfl = float(os.environ.get("CFL", "0.7"))
dq0_mode = int(os.environ.get("DQ0_MODE", "0"))
for N in map(int, sys.argv[1:]):
    mi = W.kuhn_box(N)
    m = O.OracleMesh(mi)
    V = m.geometry()[0][: m.n_cells]
    s = O.OracleSolver(m, W.advection_ic(mi), O.OracleConfig(cfl=cfl, dq0_mode=dq0_mode))
    t0 = time.time()
    steps = s.step(100000, 2.0)
    Q, t, dt, fb = s.state()
    rho_e = W.advection_ic(mi, t=t)[:, 0]
    L1, L2 = O.error_norms(Q[:, 0], rho_e, V, 8.0)
    res[str(N)] = dict(N=N, cells=m.n_cells, steps=steps, t=t, L1=L1, L2=L2, cfl=cfl, dq0_mode=dq0_mode, fallbacks=fb,
                       seconds=time.time() - t0, threads=s.threads)
    print(res[str(N)], flush=True)
    json.dump(res, open(out_path, "w"), indent=1)
