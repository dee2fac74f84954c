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
  cpu_baseline : the compiled reference (oracle/_ref) on this host, bounded sample

`--impl reference` times the reference's own CPU implementation instead (rank 0
only), one bounded sample per step.
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
                 K=4, problem="combinatorial", precond="jacobi", ref_iters=448),
    "cfg2": dict(desc="3D 7-point mesh 128^3, K=64, combinatorial, GMRES polynomial (degree 25)",
                 gen=("stencil3d", 128, 128, 128, 7), K=64, problem="combinatorial", precond="polynomial",
                 ref_iters=18),
    "cfg3": dict(desc="R-MAT scale 22 ef16 (LCC), K=64, normalized, Jacobi", gen=("rmat", 22, 16, 1),
                 K=64, problem="normalized", precond="jacobi", ref_iters=20),
    "cfg4": dict(desc="3D 27-point Brick mesh 256^3, K=256, generalized, GMRES polynomial",
                 gen=("stencil3d", 256, 256, 256, 27), K=256, problem="generalized", precond="polynomial",
                 ref_iters=12),
    # diagnostics: the per-GPU row block of cfg2 at 4 and 8 GPUs, on one GPU
    "cfg2q": dict(desc="3D 7-point mesh 128x128x32 (cfg2 / 4), K=64, combinatorial, GMRES polynomial",
                  gen=("stencil3d", 128, 128, 32, 7), K=64, problem="combinatorial", precond="polynomial",
                  ref_iters=18),
    "cfg2h": dict(desc="3D 7-point mesh 128x128x64 (cfg2 / 2), K=64, combinatorial, GMRES polynomial",
                  gen=("stencil3d", 128, 128, 64, 7), K=64, problem="combinatorial", precond="polynomial",
                  ref_iters=18),
    "cfg2e": dict(desc="3D 7-point mesh 128x128x16 (cfg2 / 8), K=64, combinatorial, GMRES polynomial",
                  gen=("stencil3d", 128, 128, 16, 7), K=64, problem="combinatorial", precond="polynomial",
                  ref_iters=18),
    "cfg5": dict(desc="R-MAT scale 24 ef16 (LCC), K=256, normalized, Jacobi", gen=("rmat", 24, 16, 1),
                 K=256, problem="normalized", precond="jacobi", ref_iters=20),
}


def make_graph(spec):
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
def cpu_sample_main(args):
    """Runs in a subprocess: the reference pipeline with max_iters in {1, 3, 2...}."""
    from oracle.ref import RefLib
    c = CONFIGS[args.config]
    g = make_graph(c["gen"])
    ref = RefLib()
    out = {"kind": ref.kind, "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))}
    times = {}
    for mi in args.cpu_iters:
        t0 = time.perf_counter()
        r = ref.partition_graph(g, run_config(c, max_iters=mi))
        times[mi] = {"wall": time.perf_counter() - t0, "total_s": r.report.times["total_s"],
                     "iterations": r.report.iterations, "cut": r.report.cutsize}
    out["times"] = times
    print("CPU_SAMPLE " + json.dumps(out), flush=True)


def cpu_sample(config, iters, timeout=900):
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    env.setdefault("OMP_WAIT_POLICY", "active")
    env["OMP_PROC_BIND"] = env.get("OMP_PROC_BIND", "false")
    cmd = [sys.executable, str(Path(__file__).resolve()), "--cpu-sample", "--config", config,
           "--cpu-iters", *map(str, iters)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    for ln in r.stdout.splitlines():
        if ln.startswith("CPU_SAMPLE "):
            return json.loads(ln[len("CPU_SAMPLE "):])
    raise RuntimeError(f"cpu sample failed: {r.stderr[-2000:]}")


def extrapolate(sample, ref_iters):
    """time(full) = T(1) + (ref_iters - 1) * t_iter, t_iter = (T(3) - T(1)) / 2."""
    t = sample["times"]
    t1, t3 = t["1"]["total_s"], t["3"]["total_s"]
    t_iter = max(0.0, (t3 - t1) / 2.0)
    return t1 + (ref_iters - 1) * t_iter, t_iter, t1 - t_iter


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
    ap.add_argument("--cpu-iters", type=int, nargs="*", default=[1, 3])
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
        kl, kname = poly_launches, "SpMM fused with the GMRES-polynomial step (spmm_ell_kernel on meshes)"
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
        "config": {"workload": f"{args.config}: {c['desc']}", "n": g.n, "nnz_A": int(g.row_offsets[-1]),
                   "K": c["K"], "seed": 42, "parallelism": f"rows1d x{world}" if world > 1 else "single",
                   "l2": "flushed between steps (256 MiB write)"},
        "e2e": {"value": round(e2e, 6), "unit": "s", "h2d_bytes_per_step": int(h2d_bytes),
                "d2h_bytes_per_step": int(d2h_bytes)},
        "roofline": {"kernel": kname, "bound": "hbm",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": (traffic or {}).get("dram_bytes_per_launch") if traffic else None,
                     "peak_source": peak_src,
                     "bytes_per_launch": round(kb / max(kl, 1)),
                     "ms_per_launch": round(kms / max(kl, 1), 5),
                     "bytes_basis": "the operator's own stored format (pattern ELL on meshes: 1 B/row)",
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
            s = cpu_sample(args.config, [1, 3])
            full, t_iter, setup = extrapolate(s, c["ref_iters"])
            line["cpu_baseline"] = {
                "value": round(full, 3), "unit": "s", "cores": s["cores"], "kind": s["kind"],
                "sample": (f"reference partition_graph with max_iters=1 and 3 on this host "
                           f"(setup {setup:.2f} s, {t_iter:.2f} s/iter), extrapolated to the reference's "
                           f"{c['ref_iters']} iterations (SURVEY §6, seed 42)")}
        except Exception as e:  # noqa: BLE001 - reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)[:300]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dg.free()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def reference_arm(args, c, rank, world):
    if rank != 0:
        return
    s = cpu_sample(args.config, [1, 3])
    full, t_iter, setup = extrapolate(s, c["ref_iters"])
    vals = []
    for _ in range(args.steps):
        s2 = cpu_sample(args.config, [2])
        t2 = s2["times"]["2"]["total_s"]
        vals.append(t2 + (c["ref_iters"] - 2) * t_iter)
    value = statistics.mean(vals)
    cores = s["cores"]
    sample = (f"each step: reference partition_graph with max_iters=2 on {cores} host threads, extrapolated "
              f"to {c['ref_iters']} iterations at {t_iter:.2f} s/iter (calibrated with max_iters=1,3)")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value * 1e3, 1),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: " + c["desc"], "config": {"workload": f"{args.config}: {c['desc']}"},
            "cpu_baseline": {"value": round(value, 3), "unit": "s", "cores": cores, "kind": s["kind"],
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
