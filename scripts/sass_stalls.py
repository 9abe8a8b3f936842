"""Stall samples of an ncu source page (--page source --csv --print-source sass), by windows of
SASS instructions: python scripts/sass_stalls.py profiles/r02/sass/k_flux_tau0_s1_c2_sass.csv.gz [W]"""
import collections
import csv
import gzip
import io
import re
import sys

path = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
rows = list(csv.reader(io.StringIO(txt)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ix["# Samples"]]) for r in data)
agg = collections.Counter()
for r in data:
    for h in st:
        agg[h[6:]] += int(r[ix[h]])
print(f"{len(data)} SASS instructions, {tot} samples:", ", ".join(f"{k} {v / tot:.1%}" for k, v in agg.most_common(8)))
for k in range(0, len(data), W):
    seg = data[k:k + W]
    s = sum(int(r[ix["# Samples"]]) for r in seg)
    if s < tot / 200:
        continue
    c = collections.Counter()
    for r in seg:
        for h in st:
            c[h[6:]] += int(r[ix[h]])
    ops = collections.Counter(m.group(2) for r in seg
                              for m in [re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[ix["Source"]])] if m)
    print(f"{k:5d} {s / tot:6.1%}  " + " ".join(f"{a}:{b}" for a, b in c.most_common(3)) + " | " +
          " ".join(f"{a}{b}" for a, b in ops.most_common(4)))
