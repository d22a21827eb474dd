"""Stall samples of an ncu source page (--print-source sass csv) grouped by
reason and opcode: where the warps of a kernel wait."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return 0.0


tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
allk = "Warp Stall Sampling (All Samples)"
total = sum(num(d[allk]) for d in data)
for d in data:
    parts = d["Source"].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    op = op.split(".")[0]
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h:
            v = num(d[h])
            tot[h] += v
            byop[h][op] += v
print(f"total samples {total:.0f}")
for h, v in tot.most_common(10):
    print(f"{h:20s} {v:8.0f} ({100 * v / total:4.1f}%)  {byop[h].most_common(5)}")
