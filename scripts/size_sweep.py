"""Per-unit kernel times vs box size (C2 Kuhn boxes): does the flux run faster per face
when the reconstruction records fit the 126 MB L2?  (50 B x 8 per cell: 48^3 -> 265 MB.)
python scripts/size_sweep.py [N ...]"""
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2407_00656_b200 import hgks, workloads as W  # noqa: E402

for N in [int(a) for a in sys.argv[1:]] or [16, 24, 32, 40, 48, 64]:
    mi = W.kuhn_box(N)
    s = hgks.Solver(hgks.Mesh(mi), W.advection_ic(mi), hgks.SolverConfig(cfl=0.3))
    s.step(5)
    s.set_profiling(True)
    s.step(40)
    kt = s.kernel_times()
    nc, nf = mi.n_cells, 2 * mi.n_cells
    row = {"N": N, "cells": nc, "records_MB": nc * 400 / 1e6}
    for k, v in kt.items():
        if v["launches"] and k.startswith(("k_recon", "k_flux")):
            per = nc if k.startswith("k_recon") else nf
            row[k + "_ns_per_unit"] = round(v["ms"] / v["launches"] * 1e6 / per, 4)
    print(json.dumps(row), flush=True)
    s.close()
