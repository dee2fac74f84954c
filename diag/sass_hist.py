"""SASS instruction histogram of the hot kernels in libspecpart_b200.so (cuobjdump, no GPU).

    python diag/sass_hist.py > profiles/r02_sass_hist.md

Per kernel family: instruction count, the opcodes that prove the data path (UTMALDG = TMA
tensor loads, UBLKCP = bulk copies, SYNCS = mbarrier ops, DMMA = fp64 tensor-core MMA,
LDG/STG/LDS/STS, DADD/DMUL/DFMA) and the top opcodes.
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2105_00578_b200" / "libspecpart_b200.so"
FAMILIES = ["spmm_ell_kernel", "spmm_mesh_kernel", "spmm_mesh_poly2_kernel", "spmm_col_kernel", "spmm_rowcols_kernel", "long_chunk_cols_kernel",
            "spmm_group_kernel", "ts_bulk_kernel", "ts_mma_kernel", "mt_fill_kernel", "halo_push_kernel",
            "cheb_step_kernel", "spgemm_expand_kernel", "hook_kernel"]
KEY = ["UTMALDG", "UBLKCP", "SYNCS", "DMMA", "LDG", "STG", "LDS", "STS", "DADD", "DMUL", "DFMA", "SHFL", "BAR"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs = collections.defaultdict(collections.Counter)
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            funcs[cur][m.group(1)] += 1
    print("# SASS instruction histogram (cuobjdump -sass libspecpart_b200.so, sm_100a)\n")
    print("Summed over every template instantiation of each kernel family.\n")
    print("| family | instantiations | instructions | " + " | ".join(KEY) + " | top opcodes |")
    print("|---|---|---|" + "---|" * len(KEY) + "---|")
    for fam in FAMILIES:
        c = collections.Counter()
        k = 0
        for name, cnt in funcs.items():
            if fam in name:
                c.update(cnt)
                k += 1
        if not k:
            continue
        top = ", ".join(f"{op} {n}" for op, n in c.most_common(6))
        row = " | ".join(str(sum(v for op, v in c.items() if op.startswith(kk))) for kk in KEY)
        print(f"| `{fam}` | {k} | {sum(c.values())} | {row} | {top} |")


if __name__ == "__main__":
    sys.exit(main())
