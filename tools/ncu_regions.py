"""Stall samples of an ncu source page (--print-source sass) grouped into
regions that start at every BAR / TLD-block / STG-block (filter-loop phases).

    ncu -i rep --page source --csv --print-source sass > src.csv
    python tools/ncu_regions.py src.csv
"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
keys = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return 0.0


regions = []
cur = None
prev_op = ""
for d in data:
    src = d["Source"].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    opb = op.split(".")[0]
    if cur is None or opb == "BAR" or (opb in ("TLD", "STG") and prev_op != opb):
        cur = {"start": src[:40], "n": 0, "samples": Counter(), "ops": Counter()}
        regions.append(cur)
    cur["n"] += 1
    cur["ops"][opb] += num(d["Instructions Executed"])
    for k in keys:
        cur["samples"][k] += num(d[k])
    prev_op = opb
tot = sum(sum(r["samples"].values()) for r in regions)
for r in regions:
    s = sum(r["samples"].values())
    if s < 0.005 * tot:
        continue
    top = ", ".join(f"{k[6:]}={v:.0f}" for k, v in r["samples"].most_common(5))
    print(f"{s / tot * 100:5.1f}% n={r['n']:4d} [{r['start']}] {top}")
