"""Diagnostic: turn ncu outputs into the committed summaries under profiles/.

  python tests/ncu_report.py launches <launches.csv> <out.md>
  python tests/ncu_report.py full <report.ncu-rep> <out.md> [traffic_json cfg]
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, mi, idi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[idi]] = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list — {path}\n\n")
        f.write("Cold-cache, serialised device times of every kernel in one partition "
                "(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                "--clock-control none`). Compare shares, not absolutes.\n\n")
        f.write(f"Total kernel time {tot / 1e6:.2f} ms over {sum(a[0] for a in agg.values())} launches.\n\n")
        f.write("| kernel | launches | total us | share | us/launch | DRAM GB/s |\n|---|---|---|---|---|---|\n")
        for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{k[-70:]}` | {a[0]} | {a[1] / 1e3:.1f} | {a[1] / tot * 100:.1f}% | "
                    f"{a[1] / a[0] / 1e3:.1f} | {a[2] / max(a[1], 1):.0f} |\n")


def full(rep, out, traffic_json=None, cfg=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "lts__t_sector_hit_rate.pct",
            "l1tex__t_sector_hit_rate.pct"]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary — {rep}\n\n")
        tr = {}
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            f.write(f"## `{name[:140]}`\n\n| metric | value |\n|---|---|\n")
            for k in keys:
                if k in hdr:
                    f.write(f"| {k} | {r[hdr.index(k)]} {units[hdr.index(k)]} |\n")
            st = [(float(r[i].replace(",", "") or 0), h) for i, h in enumerate(hdr)
                  if "pcsamp_warps_issue_stalled" in h and "not_issued" not in h and r[i]]
            tot = sum(v for v, _ in st) or 1.0
            f.write("\nTop stall reasons (PC sampling share):\n\n")
            for v, h in sorted(st, reverse=True)[:5]:
                f.write(f"- {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {v / tot * 100:.1f}%\n")
            f.write("\n")
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            mult = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
            tr = {"dram_bytes_per_launch": rd * mult.get(units[hdr.index("dram__bytes_read.sum")], 1.0)
                  + wr * mult.get(units[hdr.index("dram__bytes_write.sum")], 1.0), "kernel": name[:120]}
    if traffic_json and cfg:
        try:
            d = json.load(open(traffic_json))
        except Exception:
            d = {}
        d[cfg] = tr
        json.dump(d, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], *(sys.argv[4:6] if len(sys.argv) > 5 else []))
