"""One-time OMP_NUM_THREADS sweep of the reference CPU implementation.

Runs the compiled reference (oracle/_ref) partition_graph on a BASELINE workload
with OMP_WAIT_POLICY=active for OMP_NUM_THREADS in {1, 2, 4, ..., nproc}
(max_iters=3: setup + three LOBPCG iterations, the part that scales) and writes
profiles/cpu_thread_sweep.json; bench.py then times full reference runs at the
best count. Usage on the GPU box:  python scripts/cpu_thread_sweep.py [cfg2]
"""
import json
import os
import platform
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import SWEEP, cpu_sample  # noqa: E402


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    nproc = os.cpu_count() or 1
    counts, t = [], 1
    while t < nproc:
        counts.append(t)
        t *= 2
    counts.append(nproc)
    rows = []
    for thr in counts:
        s = cpu_sample(cfg, 1, thr, max_iters=3)
        r = s["runs"][0]
        rows.append({"threads": thr, "total_s": round(r["total_s"], 3), "times": r["times"]})
        print(json.dumps(rows[-1]), flush=True)
    best = min(rows, key=lambda r: r["total_s"])
    out = {"config": cfg, "nproc": nproc, "cpu": cpu_model(), "wait_policy": "active", "max_iters": 3,
           "sweep": rows, "best_threads": best["threads"]}
    SWEEP.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({"best_threads": best["threads"], "nproc": nproc}))


if __name__ == "__main__":
    main()
