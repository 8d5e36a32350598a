"""Summarise an ncu report (run here, no GPU needed):
   python tools/ncu_summary.py gpurun_out/mv_full.ncu-rep [more.ncu-rep]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_barrier",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(rep, "empty")
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            print("----", rep)
            for k in KEYS:
                if k in d:
                    u = units[hdr.index(k)]
                    print(f"  {k:70s} {d[k]} {u}")
            stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled") or
                      k.startswith("smsp__pcsamp_warps_issue_stalled")]
            vals = []
            for k, v in stalls:
                try:
                    vals.append((float(v.replace(",", "")), k))
                except ValueError:
                    pass
            for v, k in sorted(vals, reverse=True)[:10]:
                print(f"  stall {k:66s} {v}")


if __name__ == "__main__":
    main()
