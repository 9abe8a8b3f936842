"""Per-source-line SASS instruction counts and stall samples of one kernel from an
ncu report (captured with -lineinfo builds): maps ncu's SASS addresses to source
lines with nvdisasm -g of a cubin compiled from the same sources.

python scripts/sass_lines.py REPORT.ncu-rep MANGLED_KERNEL_NAME [top] [units_per_warp]
"""
import collections, csv, os, re, subprocess, sys, tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
warps = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
cub = os.path.join(tempfile.gettempdir(), "hgks_lines.cubin")
subprocess.run(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-cubin",
                "-o", cub, os.path.join(ROOT, "paper_2407_00656_b200", "csrc", "solver.cu"),
                "-I", os.path.join(ROOT, "include")], check=True, capture_output=True)
sass = subprocess.run(["nvdisasm", "-g", "-fun", fn, cub], capture_output=True, text=True).stdout
if not sass:
    full = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout.splitlines()
    i = full.index(fn + ":")
    out = []
    for l in full[i + 2:]:
        if l.startswith(".text."):
            break
        out.append(l)
    sass = "\n".join(out)
cur, a2l = None, {}
for l in sass.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", l)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[1]
data = rows[2:]
ends = [k for k, r in enumerate(data) if r and r[0] == "Kernel Name"]
data = data[:ends[0]] if ends else data
iA, iE, iS, iW = (h.index(k) for k in ("Address", "Instructions Executed", "Source",
                                       "Warp Stall Sampling (All Samples)"))
base = int(data[0][iA], 16)
per, perw, fp = collections.Counter(), collections.Counter(), collections.Counter()
for r in data:
    if len(r) <= iE or not r[iE].isdigit():
        continue
    key = a2l.get(int(r[iA], 16) - base, ("?", 0))
    n = int(r[iE])
    per[key] += n
    perw[key] += int(r[iW] or 0)
    t = r[iS].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "")
    if op.startswith("D") or op.startswith("F"):
        fp[key] += n
tw = sum(perw.values())
print(f"{'line':>24} {'instr/unit':>10} {'fp/unit':>9} {'stall %':>8}")
for k, n in sorted(per.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{k[0] + ':' + str(k[1]):>24} {n / warps:10.1f} {fp[k] / warps:9.1f} {100 * perw[k] / max(tw, 1):8.1f}")
