#!/usr/bin/env python
"""bench.py — time-to-partition of the BASELINE workload on N B200s.

One step = one full partition_graph (Laplacian assembly -> LOBPCG with the
GMRES-polynomial preconditioner -> multi-jagged -> cut/imbalance) of the
workload graph. At N=1 the workload is BASELINE.json configs[1] (cfg2: 7-point
128^3 mesh, K=64); the same graph is used at every N (strong scaling, 1-D row
partition over NCCL).

  value : graph arrays already in HBM (sp_partition_resident), device-timed
  e2e   : host CSR in pinned memory -> host assignment (sp_partition), H2D and
          D2H inside the timed region
  roofline : SpMM (the dominant kernel) algorithmic bytes / CUDA-event time of
          every SpMM launch inside the timed resident steps
  cpu_baseline : the compiled reference (oracle/_ref) on this host: 3 full
          partition_graph runs (min / median), OMP_WAIT_POLICY=active, at the best
          thread count of the committed sweep (scripts/cpu_thread_sweep.py)

`--impl reference` times the reference's own CPU implementation instead (rank 0
only): every timed step is one full partition_graph of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "time-to-partition (s) + edge cut/imbalance at 1/2/4/8 B200; SpMM HBM GB/s"

CONFIGS = {
    "cfg1": dict(desc="2D 5-point grid 256x256, K=4, combinatorial, Jacobi", gen=("grid2d", 256, 256),
                 K=4, problem="combinatorial", precond="jacobi"),
    "cfg2": dict(desc="3D 7-point mesh 128^3, K=64, combinatorial, GMRES polynomial (degree 25)",
                 gen=("stencil3d", 128, 128, 128, 7), K=64, problem="combinatorial", precond="polynomial"),
    "cfg3": dict(desc="R-MAT scale 22 ef16 (LCC), K=64, normalized, Jacobi", gen=("rmat", 22, 16, 1),
                 K=64, problem="normalized", precond="jacobi"),
    "cfg4": dict(desc="3D 27-point Brick mesh 256^3, K=256, generalized, GMRES polynomial",
                 gen=("stencil3d", 256, 256, 256, 27), K=256, problem="generalized", precond="polynomial"),
    # diagnostics: the per-GPU row block of cfg2 at 4 and 8 GPUs, on one GPU
    "cfg2q": dict(desc="3D 7-point mesh 128x128x32 (cfg2 / 4), K=64, combinatorial, GMRES polynomial",
                  gen=("stencil3d", 128, 128, 32, 7), K=64, problem="combinatorial", precond="polynomial"),
    "cfg2h": dict(desc="3D 7-point mesh 128x128x64 (cfg2 / 2), K=64, combinatorial, GMRES polynomial",
                  gen=("stencil3d", 128, 128, 64, 7), K=64, problem="combinatorial", precond="polynomial"),
    "cfg2e": dict(desc="3D 7-point mesh 128x128x16 (cfg2 / 8), K=64, combinatorial, GMRES polynomial",
                  gen=("stencil3d", 128, 128, 16, 7), K=64, problem="combinatorial", precond="polynomial"),
    "cfg5": dict(desc="R-MAT scale 24 ef16 (LCC), K=256, normalized, Jacobi", gen=("rmat", 24, 16, 1),
                 K=256, problem="normalized", precond="jacobi"),
}


GRAPH_CACHE = Path(os.environ.get("SPB_GRAPH_CACHE", "/tmp/spb_graph_cache"))


def make_graph(spec):
    """The synthetic input of a config (the same bytes every time: the tests check their sha256).
    R-MAT graphs take minutes to generate in numpy, so generated CSRs are cached under
    SPB_GRAPH_CACHE (default /tmp/spb_graph_cache) for later processes on the same host."""
    from paper_2105_00578_b200.api import Graph
    key = "_".join(map(str, spec))
    f_o, f_c = GRAPH_CACHE / f"{key}.offs.npy", GRAPH_CACHE / f"{key}.cols.npy"
    if spec[0] == "rmat" and f_o.exists() and f_c.exists():
        import numpy as np
        try:
            return Graph(np.load(f_o), np.load(f_c))
        except (OSError, ValueError):
            pass
    g = _generate(spec)
    if spec[0] == "rmat":
        import numpy as np
        try:
            GRAPH_CACHE.mkdir(parents=True, exist_ok=True)
            tmp_o, tmp_c = f_o.with_suffix(".tmp.npy"), f_c.with_suffix(".tmp.npy")
            np.save(tmp_c, g.col_indices)
            np.save(tmp_o, g.row_offsets)
            os.replace(tmp_c, f_c)
            os.replace(tmp_o, f_o)
        except OSError:
            pass
    return g


def _generate(spec):
    from paper_2105_00578_b200 import generators as gen
    kind = spec[0]
    if kind == "grid2d":
        return gen.grid2d(spec[1], spec[2])
    if kind == "stencil3d":
        return gen.stencil3d(*spec[1:])
    if kind == "rmat":
        g, _ = gen.rmat(spec[1], spec[2], spec[3])
        return g
    raise ValueError(kind)


def run_config(c, seed=42, max_iters=1000):
    from paper_2105_00578_b200 import RunConfig
    return RunConfig(num_parts=c["K"], problem=c["problem"], precond=c["precond"], seed=seed, max_iters=max_iters)


# ---------------------------------------------------------------- clocks ------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout=20.0):
        # NVML start-up inside nvidia-smi can stall driver calls of other processes;
        # let it finish before any timed work
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.05)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [x for x in sm if mx and x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def flush_l2(torch, dev):
    # write a buffer larger than the 126 MB L2 between timed steps
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = flush_l2.buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB
    buf.fill_(1.0)


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_from_profiles(cfg_name):
    p = ROOT / "profiles" / "spmm_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(cfg_name)
    except Exception:
        return None


# ------------------------------------------------------------ CPU baseline ----
SWEEP = ROOT / "profiles" / "cpu_thread_sweep.json"


def cpu_sample_main(args):
    """Runs in a subprocess (OMP_NUM_THREADS fixed before libgomp loads): the
    reference's partition_graph, full runs (max_iters 1000) unless asked otherwise."""
    from oracle.ref import RefLib
    c = CONFIGS[args.config]
    g = make_graph(c["gen"])
    ref = RefLib()
    out = {"kind": ref.kind, "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), "runs": []}
    for k in range(args.cpu_warmup + args.cpu_runs):
        mi = 1 if k < args.cpu_warmup else args.cpu_max_iters
        t0 = time.perf_counter()
        r = ref.partition_graph(g, run_config(c, max_iters=mi))
        wall = time.perf_counter() - t0
        if k >= args.cpu_warmup:
            out["runs"].append({"wall": wall, "total_s": r.report.times["total_s"], "times": r.report.times,
                                "iterations": r.report.iterations, "cut": r.report.cutsize,
                                "imbalance": r.report.imbalance})
            print("CPU_RUN " + json.dumps(out["runs"][-1]), flush=True)
    print("CPU_SAMPLE " + json.dumps(out), flush=True)


def cpu_sample(config, runs, threads, max_iters=1000, warmup=0, timeout=3600):
    env = dict(os.environ)
    env["OMP_NUM_THREADS"] = str(threads)
    env.setdefault("OMP_WAIT_POLICY", "active")
    env["OMP_PROC_BIND"] = env.get("OMP_PROC_BIND", "false")
    cmd = [sys.executable, str(Path(__file__).resolve()), "--cpu-sample", "--config", config,
           "--cpu-runs", str(runs), "--cpu-max-iters", str(max_iters), "--cpu-warmup", str(warmup)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    for ln in r.stdout.splitlines():
        if ln.startswith("CPU_SAMPLE "):
            return json.loads(ln[len("CPU_SAMPLE "):])
    raise RuntimeError(f"cpu sample failed: {r.stderr[-2000:]}")


def best_threads():
    """Thread count for the reference: the best of the committed OMP_NUM_THREADS sweep
    (scripts/cpu_thread_sweep.py) when it was taken on a host with this core count,
    else every core."""
    nproc = os.cpu_count() or 1
    try:
        sw = json.loads(SWEEP.read_text())
        if int(sw.get("nproc", -1)) == nproc and sw.get("best_threads"):
            return int(sw["best_threads"]), sw
    except (OSError, ValueError):
        pass
    return nproc, None


def summarize_runs(s):
    t = [r["total_s"] for r in s["runs"]]
    return {"min": round(min(t), 3), "median": round(statistics.median(t), 3), "mean": round(statistics.mean(t), 3),
            "runs_s": [round(x, 3) for x in t]}


# ------------------------------------------------------------------ main ------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", action="store_true")
    ap.add_argument("--cpu-runs", type=int, default=3)
    ap.add_argument("--cpu-max-iters", type=int, default=1000)
    ap.add_argument("--cpu-warmup", type=int, default=0)
    args = ap.parse_args()
    if args.cpu_sample:
        return cpu_sample_main(args)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    c = CONFIGS[args.config]

    if args.impl == "reference":
        return reference_arm(args, c, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2105_00578_b200 import Context

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        obj = [Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = Context(local, rank, world, nccl_id)

    g = make_graph(c["gen"])
    # pinned host copies of the caller's CSR (e2e inputs)
    offs_p = torch.from_numpy(g.row_offsets).pin_memory()
    cols_p = torch.from_numpy(g.col_indices).pin_memory()
    from paper_2105_00578_b200.api import Graph
    gp = Graph(offs_p.numpy(), cols_p.numpy())
    cfg = run_config(c)
    asg_p = torch.empty(g.n, dtype=torch.int32).pin_memory()  # pinned D2H target of the result
    asg_np = asg_p.numpy()
    h2d_bytes = gp.row_offsets.nbytes + gp.col_indices.nbytes
    d2h_bytes = 4 * g.n

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # clock sampler started before the warm-up: nvidia-smi's NVML start-up stalls
    # driver calls for a while, which must not land inside a timed step
    clk = ClockSampler(local)
    clk.start()
    clk.wait_first()
    ctx.set_timing(True)
    if os.environ.get("SPB_RECURRENCE") == "1":  # A/B of the AX/AH/AP recurrence
        ctx.set_recurrence(True)
    if os.environ.get("SPB_RELABEL") == "0":  # A/B of the irregular-graph relabel
        ctx.set_relabel(False)
    dg = ctx.upload(gp)
    for _ in range(args.warmup):
        ctx.partition_resident(dg, cfg, copy_assignment=False)
    ctx.partition_graph(gp, cfg, out=asg_np)  # e2e warm-up

    def timed(fn):
        ts, reps = [], []
        for _ in range(args.steps):
            flush_l2(torch, dev)
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn()
            e1.record()
            e1.synchronize()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
            reps.append(r)
        barrier()
        return ts, reps

    t_res, r_res = timed(lambda: ctx.partition_resident(dg, cfg, copy_assignment=False))
    t_e2e, r_e2e = timed(lambda: ctx.partition_graph(gp, cfg, out=asg_np))
    clocks = clk.stop()

    value = max_over_ranks(statistics.mean(t_res))
    e2e = max_over_ranks(statistics.mean(t_e2e))
    rep = r_res[-1].report
    spmm_bytes = sum(r.report.device["spmm_bytes"] for r in r_res)
    spmm_ms = sum(r.report.device["spmm_ms"] for r in r_res)
    launches = sum(r.report.device["kernel_launches"] for r in r_res)
    spmm_launches = sum(r.report.device["spmm_launches"] for r in r_res)
    poly_launches = sum(r.report.device["poly_launches"] for r in r_res)
    # dominant kernel: the fused GMRES-polynomial step SpMM when the polynomial
    # preconditioner runs, else every SpMM launch
    if poly_launches:
        keff = sum(r.report.device["poly_eff_bytes"] for r in r_res)
        kb = sum(r.report.device["poly_bytes"] for r in r_res)
        kms = sum(r.report.device["poly_ms"] for r in r_res)
        kl, kname = poly_launches, ("SpMM fused with the GMRES-polynomial steps (structured mesh, TMA 3-D tiles, "
                                    "z-marching: spmm_mesh_poly2_kernel, two steps per pass on 5/7-point meshes "
                                    "on one GPU; spmm_mesh_kernel, one step, otherwise)")
    else:
        kb, kms, kl, kname = spmm_bytes, spmm_ms, spmm_launches, "spmm (CSR SpMM + fused epilogues)"
        keff = sum(r.report.device["spmm_eff_bytes"] for r in r_res)
    achieved = kb / (kms / 1e3) / 1e9 if kms > 0 else 0.0
    peak, peak_src = measured_peak()
    traffic = traffic_from_profiles(args.config)
    line = {
        "metric": METRIC, "value": round(value, 6), "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(value * 1e3, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: " + c["desc"] + " (reference generator semantics, unit weights)",
        "config": config_dict(args, c, g, world),
        "e2e": {"value": round(e2e, 6), "unit": "s", "h2d_bytes_per_step": int(h2d_bytes),
                "d2h_bytes_per_step": int(d2h_bytes)},
        "roofline": {"kernel": kname, "bound": "hbm",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": (traffic or {}).get("dram_bytes_per_launch") if traffic else None,
                     "peak_source": peak_src,
                     "bytes_per_launch": round(kb / max(kl, 1)),
                     "ms_per_launch": round(kms / max(kl, 1), 5),
                     "bytes_basis": ("the operator's own stored format: none for a recognised structured mesh "
                                     "(implicit stencil), 1 B/row for pattern ELL, 4 B/nnz + offsets for CSR; "
                                     "X and Y once per launch, H read+write on the steps that update it; the "
                                     "two-step kernel reads p_i and writes p_{i+2} and H, p_{i+1} stays on chip"),
                     "effective": {"basis": "same launches counted as pattern CSR (4 B/nnz + 8 B/row offsets)",
                                   "gbs": round(keff / (kms / 1e3) / 1e9, 1) if kms > 0 else 0.0,
                                   "bytes_per_launch": round(keff / max(kl, 1))},
                     "launches_per_step": kl // max(len(r_res), 1),
                     "kernel_share_of_step": round((kms / 1e3) / max(sum(t_res), 1e-12), 4),
                     "all_spmm": {"achieved": round(spmm_bytes / (spmm_ms / 1e3) / 1e9, 1) if spmm_ms > 0 else 0.0,
                                  "launches_per_step": spmm_launches // max(len(r_res), 1)}},
        "halo": ({"exchanges_per_step": sum(r.report.device["halo_launches"] for r in r_res) // max(len(r_res), 1),
                  "us_per_exchange": round(1e3 * sum(r.report.device["halo_ms"] for r in r_res)
                                           / max(1, sum(r.report.device["halo_launches"] for r in r_res)), 2),
                  "bytes_per_exchange": round(sum(r.report.device["halo_bytes"] for r in r_res)
                                              / max(1, sum(r.report.device["halo_launches"] for r in r_res))),
                  "path": "nccl" if os.environ.get("SPB_P2P", "1") == "0" else "p2p (NVLink peer writes)"}
                 if world > 1 else None),
        "step_s": [round(x, 5) for x in t_res], "e2e_step_s": [round(x, 5) for x in t_e2e],
        "clocks": clocks, "gpu_launches": int(launches),
        "result": {"cut": rep.cutsize, "imbalance": rep.imbalance, "iterations": rep.iterations,
                   "converged": all(rep.converged), "times": rep.times,
                   "e2e_cut": r_e2e[-1].report.cutsize},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            thr, sw = best_threads()
            s = cpu_sample(args.config, 3, thr)
            st = summarize_runs(s)
            line["cpu_baseline"] = {
                "value": st["median"], "unit": "s", "cores": s["cores"], "kind": s["kind"],
                "min": st["min"], "median": st["median"], "runs_s": st["runs_s"],
                "iterations": s["runs"][-1]["iterations"], "cut": s["runs"][-1]["cut"],
                "imbalance": s["runs"][-1]["imbalance"],
                "threads_from": "profiles/cpu_thread_sweep.json" if sw else "all cores (no sweep for this host)",
                "sample": (f"3 full runs of the reference partition_graph (oracle/_ref, max_iters 1000, "
                           f"OMP_WAIT_POLICY=active, {s['cores']} of {os.cpu_count()} host threads) on this "
                           f"workload; value = median")}
        except Exception as e:  # noqa: BLE001 - reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)[:300]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dg.free()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def reference_arm(args, c, rank, world):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    /root/reference/proj/src compiled in-tree) timed on this host: every timed step
    is one full partition_graph (max_iters 1000) of the workload; warm-up steps run
    max_iters=1 (untimed). Rank 0 only."""
    if rank != 0:
        return
    thr, sw = best_threads()
    s = cpu_sample(args.config, args.steps, thr, warmup=args.warmup, timeout=6 * 3600)
    st = summarize_runs(s)
    value = st["mean"]
    from paper_2105_00578_b200 import generators  # noqa: F401 (graph sizes for the config dict)
    g = make_graph(c["gen"])
    last = s["runs"][-1]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value * 1e3, 1),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: " + c["desc"] + " (reference generator semantics, unit weights)",
            "config": config_dict(args, c, g, world),
            "cpu_baseline": {"value": value, "unit": "s", "cores": s["cores"], "kind": s["kind"],
                             "min": st["min"], "median": st["median"], "runs_s": st["runs_s"],
                             "threads_from": "profiles/cpu_thread_sweep.json" if sw else "all cores",
                             "sample": (f"each timed step = one full reference partition_graph (max_iters 1000, "
                                        f"OMP_WAIT_POLICY=active, {s['cores']} of {os.cpu_count()} host "
                                        f"threads); warm-up steps ran max_iters=1")},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "result": {"cut": last["cut"], "imbalance": last["imbalance"], "iterations": last["iterations"],
                       "times": last["times"]}}
    print(json.dumps(line), flush=True)


def config_dict(args, c, g, world):
    return {"workload": f"{args.config}: {c['desc']}", "n": int(g.n), "nnz_A": int(g.row_offsets[-1]),
            "K": c["K"], "problem": c["problem"], "precond": c["precond"], "seed": 42,
            "parallelism": f"rows1d x{world}" if world > 1 else "single",
            "l2": "flushed between steps (256 MiB write)"}


if __name__ == "__main__":
    main()
