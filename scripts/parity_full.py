"""10-step parity at full size for the two largest configs (north_star: "every config matches
the CPU oracle within 1e-10 relative after 10 steps"), outside the pytest suite (the oracle
needs ~15 min per config on 16 host cores): C5 (110^3 Kuhn box, 7,986,000 tets, bench default)
and C4 (sphere shell N = 70, 4,116,000 hexes, Ma 1.5, Re 300).  Prints one JSON line per config.

    python scripts/parity_full.py [c5] [c4] [--steps 10]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402
from paper_2407_00656_b200 import hgks, workloads as W  # noqa: E402
from test_gpu_parity import TOL, gpu_and_oracle, rel_err, sphere_case  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c5", "c4"])
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    for c in args.configs:
        t0 = time.time()
        if c == "c5":
            mi = W.kuhn_box(110)
            Q0 = W.advection_ic(mi)
            gc, oc = hgks.SolverConfig(cfl=0.3), O.OracleConfig(cfl=0.3)
        else:
            mi, Q0, oc, gc = sphere_case(70, 1.5, 300.0)
        Qg, tg, (Qo, to, _, fbo) = gpu_and_oracle(mi, Q0, gc, oc, args.steps)
        e = rel_err(Qg, Qo)
        print(json.dumps({"config": c, "cells": int(mi.n_cells), "steps": args.steps, "t_gpu": tg, "t_oracle": to,
                          "max_rel_err_per_variable": [float(x) for x in e], "bar": TOL, "pass": bool(e.max() <= TOL
                          and abs(tg - to) <= 1e-13 * max(1.0, to)), "fallbacks_oracle": int(fbo),
                          "wall_s": round(time.time() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
