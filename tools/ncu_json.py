"""Extract per-kernel numbers from an ncu --set full report into the JSON that
bench.py reads for roofline.traffic:  python tools/ncu_json.py REP OUT.json SOURCE"""
import csv, io, json, re, subprocess, sys

rep, out, src = sys.argv[1], sys.argv[2], sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
col = {k: hdr.index(k) for k in hdr}
res = {"_source": src}
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    m = re.match(r"void (\w+)<([^>]*)>", name) or re.match(r"(\w+)", name)
    args = m.group(2).replace(" ", "") if m.lastindex and m.lastindex > 1 else None
    if args is not None:   # k_mv_wht<8,3,0,2,float> -> k_mv_wht<8,3,0,2> (the element-operator type is not part of the key)
        args = re.sub(r"(,(double|float))+$", "", args)
    key = m.group(1) + ("<" + args + ">" if args is not None else "")
    if key in res:
        continue
    def g(k, scale=1.0):
        try:
            return float(r[col[k]].replace(",", "")) * scale
        except Exception:
            return None
    ur = rows[1]
    def gb(k):
        v = g(k)
        u = ur[col[k]]
        f = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "B": 1e-9, "KB": 1e-6, "MB": 1e-3, "GB": 1.0}.get(u, None)
        return v * f if (v is not None and f) else None
    tu = ur[col["gpu__time_duration.sum"]]
    res[key] = {"gpu_time_us": g("gpu__time_duration.sum") * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[tu],
                "dram_read_GB": gb("dram__bytes_read.sum"), "dram_write_GB": gb("dram__bytes_write.sum"),
                "dram_pct_peak": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "regs": g("launch__registers_per_thread"),
                "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active")}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
