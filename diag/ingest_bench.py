"""Diagnostic: device ingestion (sp_ingest: symmetrize + largest_connected_component)
on raw R-MAT edge lists vs the compiled reference on the host cores.

    python tests/ingest_bench.py [scale ...]      (default: 22 24)

Prints one JSON line per scale: GPU time through the C-ABI with host buffers
(H2D inside, result left in HBM), the result sizes, a bit-exact check against the
reference at scales <= 22, and the reference's own time for the same call.
Algorithmic bytes (HBM): read 8(n+1) + 4 nnz_raw, write/read the 2 nnz_raw packed
keys through the radix sort (8 B each, ~2 passes of 8 bytes per digit), CSR and
relabel passes over nnz_sym.
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2105_00578_b200 import Context  # noqa: E402
from paper_2105_00578_b200 import generators as gen  # noqa: E402


def raw_csr(n, rows, cols):
    order = np.argsort(rows, kind="stable")
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offs[1:])
    return offs, np.ascontiguousarray(cols[order], dtype=np.int32)


def main():
    scales = [int(a) for a in sys.argv[1:]] or [22, 24]
    ctx = Context(0)
    ref = None
    try:
        from oracle.ref import REF_LIB, RefLib
        if REF_LIB.exists():
            ref = RefLib(REF_LIB)
    except Exception:
        ref = None
    for scale in scales:
        n, s, d = gen.rmat_edges(scale, 16, seed=1)
        offs, cols = raw_csr(n, s, d)
        del s, d
        w = gen.grid2d(64, 64)
        ctx.ingest(w.row_offsets, w.col_indices).free()  # warm-up (pool, module load)
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            dg = ctx.ingest(offs, cols)
            times.append(time.perf_counter() - t0)
            info = dg.info()
            if _ < 2:
                dg.free()
        line = dict(stage="ingest", scale=scale, n_raw=n, nnz_raw=int(offs[-1]), n_lcc=info.n, nnz_lcc=info.nnz,
                    nnz_symmetrized=info.nnz_symmetrized, gpu_s=min(times), gpu_s_all=times,
                    regular=info.regular, max_degree=info.max_degree)
        if ref is not None and scale <= int(os.environ.get("SPB_INGEST_REF_MAX", "22")):
            t0 = time.perf_counter()
            want, want_old = ref.symmetrize_lcc(n, offs, cols)
            line["ref_s"] = time.perf_counter() - t0
            line["ref_threads"] = 1  # symmetrize / LCC are serial in the reference
            got, old = dg.download()
            line["bit_exact"] = bool(np.array_equal(got.row_offsets, want.row_offsets)
                                     and np.array_equal(got.col_indices, want.col_indices)
                                     and np.array_equal(old, want_old))
        dg.free()
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
