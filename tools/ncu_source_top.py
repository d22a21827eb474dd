"""Top SASS lines of an ncu source page by a metric (default: stall samples)."""
import csv
import sys

path = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return 0.0


tot = sum(num(d[key]) for d in data)
print(f"total {key}: {tot:.0f}")
cols = ["stall_short_sb", "stall_long_sb", "stall_barrier", "stall_mio",
        "stall_wait", "stall_dispatch", "L1 Conflicts Shared N-Way",
        "L1 Wavefronts Shared Excessive"]
for d in sorted(data, key=lambda d: -num(d[key]))[:n]:
    extra = " ".join(f"{c.split('_')[-1][:6]}={d.get(c, '')}" for c in cols
                     if num(d.get(c, "0")))
    print(f"{d['Address']:>6} {num(d[key]):8.0f}  {d['Source'][:60]:60s} {extra}")
