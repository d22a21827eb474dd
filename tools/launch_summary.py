"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py launches.csv "<command it profiled>"
"""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
agg = collections.OrderedDict()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    short = name.split("(")[0][:100] if "olsb" in name else name[:60]
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
out = [f"# ncu launch list: {sys.argv[2] if len(sys.argv) > 2 else ''}",
       "# --metrics gpu__time_duration.sum --clock-control none (cold-cache, "
       "serialised: compare shares, not absolutes)",
       f"# total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches",
       "count  total_ms  share  kernel"]
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{n:5d} {t / 1e6:9.3f} {t / tot * 100:5.1f}%  {k}")
print("\n".join(out))
