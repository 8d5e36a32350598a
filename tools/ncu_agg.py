"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
unit = "ns"
for name, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v / tot * 100:6.2f}%  {n:6d}  {v / 1e6:10.3f} ms  {v / n / 1e3:9.2f} us/launch  {name}")
print(f"total {tot / 1e6:.3f} ms")
