"""Host setup cost of one rank for the C5 weak-scaling layout.

    python scripts/setup_memory.py [--gpus 8] [--block 110] [--whole]

Generates the bench.py weak-scaling box for --gpus ranks (one --block^3 Kuhn block per
rank; 8 x 110^3 = 220^3 cubes = 63,888,000 tets) and builds rank 0's mesh the way a
multi-process run does (hgks_mesh_desc.rank_only: only its region), reporting wall time and
peak RSS of the build (resource.getrusage in this process, after the input arrays exist).
--whole builds the whole-mesh path instead (every rank's connectivity; not feasible at 8 x
110^3 on small hosts -- about 1.7 KB per global cell)."""
import argparse, json, os, resource, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00656_b200 import hgks, workloads as W
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=8)
ap.add_argument("--block", type=int, default=110)
ap.add_argument("--whole", action="store_true")
args = ap.parse_args()
t0 = time.time()
nx, ny, nz = bench.box_dims(args.gpus, args.block)
mi = W.kuhn_box(nx, ny, nz, h=2.0 / args.block)
t_gen = time.time() - t0
rss0 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
t1 = time.time()
m = hgks.Mesh(mi, n_ranks=args.gpus, rank=None if args.whole else 0)
info = m.info(0)
t_build = time.time() - t1
rss1 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
print(json.dumps({"layout": f"{args.gpus} x {args.block}^3 Kuhn blocks ({mi.n_cells} tets)", "build": "whole" if args.whole else "region (rank_only)",
                  "input_generation_s": round(t_gen, 1), "rank0_setup_s": round(t_build, 1),
                  "peak_rss_before_build_GB": round(rss0 / 1e6, 2), "peak_rss_after_build_GB": round(rss1 / 1e6, 2),
                  "build_increment_GB": round((rss1 - rss0) / 1e6, 2), "n_owned": info["n_owned"], "n_ghost": info["n_ghost"],
                  "rank_cut_faces": info["rank_cut_faces"], "n_peers": info["n_peers"]}), flush=True)
