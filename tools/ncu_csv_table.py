"""Print an ncu --csv --metrics log (header preceded by program output) as one
row per launch: python tools/ncu_csv_table.py FILE [max_rows]"""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    if len(r) == len(h):
        d.setdefault(r[ii], [r[ki].split("(")[0][:48], {}])[1][r[mi]] = r[vi]
for i, (name, m) in list(d.items())[: int(sys.argv[2]) if len(sys.argv) > 2 else 50]:
    print(f"{i:>4} {name:48s} " + " ".join(f"{k.split('__')[1].split('.')[0][:14]}={v}" for k, v in sorted(m.items())))
