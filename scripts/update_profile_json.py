"""Regenerate profiles/flops_per_unit.json, profiles/traffic.json and
profiles/fp64_peak.json from a scripts/gpu/profile.sh capture.

python scripts/update_profile_json.py [gpurun_out/prof] [profiles/r01]

Inputs (all written on the B200 by scripts/gpu/profile.sh):
  flops_{c2,c3}_{64,32}.csv  ncu SASS op counts (dfma/dadd/dmul, ffma/fadd/fmul)
  full_c2.ncu-rep             ncu --set full (DRAM bytes per launch)
  peaks.json                  tools/microbench/fp64_peak (DFMA / FFMA chains, copy)
The per-unit counts are per INTERIOR face (flux) or per reconstructed cell (recon);
the face counts follow from the mesh generators (tet box: 2 faces per cell;
sphere shell N: (6 * cells - 2 * 6 N^2) / 2).
"""
import csv, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof")
DST = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r01")

N_BOX = 48
CELLS = {"c2": 6 * N_BOX ** 3, "c3": 12 * 35 ** 3, "c4": 12 * 70 ** 3, "c5": 6 * 110 ** 3}
IFACES = {"c2": 2 * CELLS["c2"], "c3": (6 * CELLS["c3"] - 2 * 6 * 35 ** 2) // 2,
          "c4": (6 * CELLS["c4"] - 2 * 6 * 70 ** 2) // 2}
NAMES = {"k_flux<3, 1, 1, 0, 0, 0>": "k_flux_tau0_s1", "k_flux<3, 2, 1, 0, 0, 0>": "k_flux_tau0_s2",
         "k_flux<4, 1, 0, 0, 0, 0>": "k_flux_s1", "k_flux<4, 2, 0, 0, 0, 0>": "k_flux_s2"}
SCALE = {"": 1.0, "inst": 1.0, "K": 1e3, "M": 1e6, "G": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6}


def op_counts(path):
    out = {}
    for r in csv.reader(open(path)):
        if len(r) < 15 or r[0] == "ID":
            continue
        name = r[4].split("(")[0].replace("void ", "").strip()
        out.setdefault((r[0], name), {})[r[12]] = float(r[14].replace(",", "")) * SCALE.get(r[13], 1.0)
    return out


def main():
    flops = {"_doc": "flops per interior face (flux) or per cell (recon) per launch = (2*fma + add + mul) "
                     "SASS thread-instruction counts from ncu on the B200 (profiles/r01/flops_*.csv); "
                     "tet faces have 3 Gauss points, quad faces 4; fp64 for --precision 64, fp32 for 32"}
    for w in ("c2", "c3"):
        for p in ("64", "32"):
            f = os.path.join(SRC, f"flops_{w}_{p}.csv")
            if not os.path.exists(f):
                continue
            shutil.copy(f, os.path.join(DST, f"flops_{w}_{p}.csv"))
            for (_, name), m in op_counts(f).items():
                pre = "d" if p == "64" else "f"
                n = (2 * m.get(f"smsp__sass_thread_inst_executed_op_{pre}fma_pred_on.sum", 0)
                     + m.get(f"smsp__sass_thread_inst_executed_op_{pre}add_pred_on.sum", 0)
                     + m.get(f"smsp__sass_thread_inst_executed_op_{pre}mul_pred_on.sum", 0))
                if name.startswith("k_recon"):
                    key, unit, per = "k_recon", "cell", n / CELLS[w]
                elif name in NAMES:
                    key, unit, per = NAMES[name], "face", n / IFACES[w]
                else:
                    continue
                ent = flops.setdefault(w, {}).setdefault(key, {})
                ent[f"fp{p}_flops_per_{unit}"] = round(per)
    flops["c4"] = flops.get("c3", {})  # same kernels and per-face work (sphere shell, tau > 0)
    old_path = os.path.join(ROOT, "profiles", "flops_per_unit.json")
    if os.path.exists(old_path):  # keep entries this capture does not regenerate (c3h)
        for k, v in json.load(open(old_path)).items():
            flops.setdefault(k, v)
    json.dump(flops, open(old_path, "w"), indent=1)

    for wl in ("c2", "c5"):
        rep = os.path.join(SRC, f"full_{wl}.ncu-rep")
        gz = os.path.join(SRC, f"ncu_full_{wl}.csv.gz")  # exported on the box (gpurun copies <= 64 MiB)
        if os.path.exists(rep):
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        elif os.path.exists(gz):
            import gzip
            raw = gzip.open(gz, "rt").read()
        else:
            continue
        rows = list(csv.reader(raw.splitlines()))
        h, units = rows[0], rows[1]
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
        seen = set()
        for row in rows[2:]:
            d = {k: (v, u) for k, v, u in zip(h, row, units)}
            val = lambda k: float(d[k][0].replace(",", "")) * SCALE.get(d[k][1], 1.0)
            name = d["Kernel Name"][0].split("(")[0].replace("void ", "").strip()
            key = "k_recon" if name.startswith("k_recon") else NAMES.get(name, name)
            if key in seen:
                continue
            seen.add(key)
            traffic[key] = {"dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                            "time_ns": val("gpu__time_duration.sum"), "cells": CELLS[wl],
                            "source": f"ncu --set full --clock-control none, {wl} Kuhn box, one launch "
                                      f"({os.path.relpath(DST, ROOT)}/ncu_full_{wl}.csv)"}
        json.dump(traffic, open(tpath, "w"), indent=1)
        open(os.path.join(DST, f"ncu_full_{wl}.csv"), "w").write(raw)
    pk = os.path.join(SRC, "peaks.json")
    if os.path.exists(pk):
        shutil.copy(pk, os.path.join(ROOT, "profiles", "fp64_peak.json"))
    for f in ("launches_c2.csv", "launches_c5.csv", "launches_c5.csv.gz"):
        if os.path.exists(os.path.join(SRC, f)):
            shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))
    print(json.dumps(flops, indent=1))


if __name__ == "__main__":
    main()
