"""Edge cut of the k-way partition (hgks_mesh_stats.edge_cut_rcb / edge_cut): plain RCB vs RCB +
Fiduccia-Mattheyses refinement (csrc/setup.cpp refine_partition), with the part sizes.

    python scripts/edge_cut.py [c4|c3|c5] [ranks]      (host only; no GPU needed)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00656_b200 import hgks, workloads as W

wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mi = {"c3": lambda: W.sphere_shell(35), "c4": lambda: W.sphere_shell(70), "c5": lambda: W.kuhn_box(110),
      "c4j": lambda: W.sphere_shell(69)}[wl]()
t0 = time.time()
m = hgks.Mesh(mi, n_ranks=nr)
st = [m.info(r) for r in range(nr)]
sizes = [s["n_owned"] for s in st]
print(json.dumps({"workload": wl, "cells": mi.n_cells, "ranks": nr, "edge_cut_rcb": st[0]["edge_cut_rcb"],
                  "edge_cut_refined": st[0]["edge_cut"],
                  "reduction": 1 - st[0]["edge_cut"] / max(1, st[0]["edge_cut_rcb"]),
                  "owned_min": min(sizes), "owned_max": max(sizes),
                  "ghosts_per_rank": [s["n_ghost"] for s in st], "peers": [s["n_peers"] for s in st],
                  "seconds": round(time.time() - t0, 1)}), flush=True)
