"""Aggregate an ncu --csv launch list with gpu__time_duration.sum and
launch__grid_size by (kernel name, grid size) -- separates the multigrid levels."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[ii]] = r[ki].split("(")[0][:90]
agg = collections.defaultdict(lambda: [0, 0.0])
for i, m in per.items():
    key = (names[i], int(m.get("launch__grid_size", 0)))
    agg[key][0] += 1
    agg[key][1] += m.get("gpu__time_duration.sum", 0.0)
tot = sum(v[1] for v in agg.values())
for (name, g), (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 60]:
    print(f"{v / tot * 100:6.2f}%  {n:6d}  {v / 1e6:9.3f} ms  {v / n / 1e3:8.2f} us  grid {g:7d}  {name}")
print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
