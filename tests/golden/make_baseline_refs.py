"""Reference results at the BASELINE configs, on this repo's exact graph bytes.

TEST INFRASTRUCTURE ONLY. Runs the unmodified reference (oracle/_ref, the
compiled /root/reference/proj/src, `partition_graph` at src/pipeline.cpp:47-167)
on cfg1..cfg5 exactly as bench.py builds them (paper_2105_00578_b200.generators,
RunConfig seed 42, max_iters 1000, explicit problem/precond per BASELINE.json)
and writes tests/golden/baseline/<cfg>.json:

  csr_sha256        sha256 of row_offsets (int64) || col_indices (int32) bytes, so
                    the GPU-side test proves it partitions the same graph
  iterations, theta, residual_norms, converged, breakdown_retries, poly_degree,
  tol/problem/precond/init (resolved), cutsize, imbalance, part_weights,
  assignment_sha256 (int32 bytes), trace (per-iteration min/max residual), times
  cores / OMP settings / host the run used

cfg1 and cfg2 also store the assignment itself (uint8, compressed npz) so a GPU
test can feed the reference's partition to the device cut/imbalance kernels.

Usage (build container, needs oracle/_ref/libspecpart_ref.so):
    OMP_NUM_THREADS=6 OMP_WAIT_POLICY=active python tests/golden/make_baseline_refs.py cfg2 [cfg3 ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

OUT = ROOT / "tests" / "golden" / "baseline"


def csr_sha(g) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(g.row_offsets, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(g.col_indices, dtype=np.int32).tobytes())
    return h.hexdigest()


def main(names):
    from bench import CONFIGS, make_graph, run_config
    from oracle.ref import RefLib

    ref = RefLib()
    assert ref.kind == "reference", "baseline fixtures must come from the compiled reference"
    OUT.mkdir(parents=True, exist_ok=True)
    for name in names:
        c = CONFIGS[name]
        t0 = time.perf_counter()
        g = make_graph(c["gen"])
        tgen = time.perf_counter() - t0
        cfg = run_config(c)
        cfg.record_trace = True
        t0 = time.perf_counter()
        r = ref.partition_graph(g, cfg)
        wall = time.perf_counter() - t0
        rep = r.report
        a = np.ascontiguousarray(r.partition.assignment, dtype=np.int32)
        d = {
            "config": name, "desc": c["desc"], "gen": list(c["gen"]), "K": c["K"],
            "n": int(g.n), "nnz_A": int(g.row_offsets[-1]), "csr_sha256": csr_sha(g),
            "run_config": {"num_parts": cfg.num_parts, "problem": cfg.problem, "precond": cfg.precond,
                           "seed": cfg.seed, "max_iters": cfg.max_iters, "epsilon": cfg.epsilon},
            "resolved": {"problem": rep.problem, "precond": rep.precond, "tol": rep.tol, "init": rep.init,
                         "eigenvectors": rep.eigenvectors, "regular": rep.regular,
                         "max_degree": rep.max_degree, "avg_degree": rep.avg_degree},
            "iterations": rep.iterations, "breakdown_retries": rep.breakdown_retries,
            "poly_degree": rep.poly_degree,
            "theta": list(map(float, rep.theta)), "residual_norms": list(map(float, rep.residual_norms)),
            "converged": list(map(bool, rep.converged)),
            "cutsize": float(rep.cutsize), "imbalance": float(rep.imbalance),
            "part_weights": list(map(float, r.partition.part_weights)),
            "assignment_sha256": hashlib.sha256(a.tobytes()).hexdigest(),
            "warnings": list(rep.warnings),
            "trace": [{"iter": t.iter, "min_residual": float(t.min_residual), "max_residual": float(t.max_residual),
                       "theta": list(map(float, t.theta))} for t in rep.trace],
            "times": rep.times, "wall_s": wall, "generate_s": tgen,
            "host": {"cpu": platform.processor() or platform.machine(), "nproc": os.cpu_count(),
                     "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
                     "OMP_WAIT_POLICY": os.environ.get("OMP_WAIT_POLICY")},
            "oracle": str(ref.path.relative_to(ROOT)),
        }
        (OUT / f"{name}.json").write_text(json.dumps(d, indent=1, default=float) + "\n")
        if g.n <= 4_000_000 and c["K"] <= 256:
            np.savez_compressed(OUT / f"{name}_assignment.npz", assignment=a.astype(np.uint8))
        print(f"{name}: n={g.n} iters={rep.iterations} cut={rep.cutsize} imb={rep.imbalance} "
              f"total_s={rep.times.get('total_s')} wall={wall:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
