"""Diagnose per-step time vs kernel time on the bench workload (host enqueue vs device)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2407_00656_b200 import hgks, workloads as W
N = int(sys.argv[1]) if len(sys.argv) > 1 else 48
mi = W.kuhn_box(N)
s = hgks.Solver(hgks.Mesh(mi), W.advection_ic(mi), hgks.SolverConfig(cfl=0.3))
s.step(10, info=False); torch.cuda.synchronize()
st = s.stream
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st); t0 = time.perf_counter()
    s.step(50, info=False)
    t1 = time.perf_counter(); e1.record(st); e1.synchronize(); t2 = time.perf_counter()
    print(f"enqueue {1e3*(t1-t0)/50:.3f} ms/step, host total {1e3*(t2-t0)/50:.3f}, gpu {e0.elapsed_time(e1)/50:.3f} ms/step", flush=True)
s.set_profiling(True)
s.step(50, info=False)
kt = s.kernel_times()
tot = sum(v["ms"] for v in kt.values())
print("kernel sum per step", tot / 50, {k: round(v["ms"] / v["launches"], 4) for k, v in kt.items()})
