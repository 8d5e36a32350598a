"""Top SASS instructions per stall reason from an ncu report's source page."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reasons = sys.argv[2].split(",") if len(sys.argv) > 2 else ["stall_long_sb", "stall_barrier", "stall_wait", "stall_short_sb", "stall_math", "stall_mio", "stall_lg"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
seen = {}
for r in data:
    if len(r) == len(hdr) and r[0] not in seen:
        seen[r[0]] = r
uniq = list(seen.values())
idx = {h: i for i, h in enumerate(hdr)}


def iv(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(iv(r[idx["Warp Stall Sampling (All Samples)"]]) for r in uniq)
print("samples", tot)
for reason in reasons:
    k = idx[reason]
    s = sum(iv(r[k]) for r in uniq)
    print(f"== {reason}: {s} ({100.0 * s / max(tot, 1):.1f}%)")
    for r in sorted(uniq, key=lambda r: -iv(r[k]))[:6]:
        if iv(r[k]) == 0:
            break
        print(f"   {iv(r[k]):6d} {r[0][-5:]} {r[idx['Source']][:90]}")
