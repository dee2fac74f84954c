"""Diagnostic: summarize an ncu report (per kernel: duration, DRAM, issue, occupancy, stalls)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
idx = {w: hdr.index(w) for w in want if w in hdr}
stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled") and h.endswith(".ratio")]
if not stall:
    stall = [i for i, h in enumerate(hdr) if "warp_issue_stalled" in h and h.endswith("_per_warp_active.pct")]
for r in rows[2:]:
    print("==", r[idx["Kernel Name"]][:100])
    for w, i in idx.items():
        if w != "Kernel Name":
            print(f"   {w:55s} {r[i]} {units[i]}")
    top = sorted(((float(r[i] or 0), hdr[i]) for i in stall), reverse=True)[:6]
    for v, h in top:
        print(f"   stall {h.replace('smsp__average_warp_latency_issue_stalled_','').replace('smsp__warp_issue_stalled_',''):50s} {v:.2f}")
