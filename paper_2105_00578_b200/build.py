"""Builds libspecpart_b200.so in-tree with nvcc for sm_100a (no JIT, no torch).

Every .cu/.cpp under csrc/ is compiled to an object under build/ and linked
into paper_2105_00578_b200/libspecpart_b200.so against the CUDA runtime and
NCCL. Objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "obj"
GEN = ROOT / "build" / "gen"
TOOLS = PKG / "tools"
LIB = PKG / "libspecpart_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-ffp-contract=off",
          "-I", str(ROOT / "include"), "-I", str(CSRC), "-I", str(GEN), "--expt-relaxed-constexpr"]


def _sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers_mtime():
    hs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, hdr_mtime: float, verbose: bool) -> Path:
    obj = BUILD / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":
        cmd = [NVCC, *COMMON, "-x", "cu", *ARCH, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    return obj


def _gen_tables(verbose: bool) -> None:
    """MT19937-64 jump polynomials (tools/mt_jump_gen.cpp) -> build/gen/mt_jump_table.inc."""
    GEN.mkdir(parents=True, exist_ok=True)
    inc = GEN / "mt_jump_table.inc"
    src = TOOLS / "mt_jump_gen.cpp"
    if inc.exists() and inc.stat().st_mtime >= src.stat().st_mtime:
        return
    exe = GEN / "mt_jump_gen"
    subprocess.run(["g++", "-O2", "-std=c++20", "-o", str(exe), str(src)], check=True)
    # chunk of 2^18 draws, jumps for chunk indices < 2^16 (17 G draws)
    subprocess.run([str(exe), str(inc), "18", "16"], check=True)
    if verbose:
        print(f"generated {inc}")


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    _gen_tables(verbose)
    hm = max(_headers_mtime(), (GEN / "mt_jump_table.inc").stat().st_mtime)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    _build_shim_test(verbose)
    _build_cli(verbose)
    return LIB


NLOHMANN = Path(os.environ.get(
    "NLOHMANN_DIR", "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"))
CLI = ROOT / "build" / "specpart_b200"


def _build_cli(verbose: bool) -> None:
    """build/specpart_b200: the reference CLI (tools/specpart.cpp) on the C-ABI
    (paper_2105_00578_b200/tools/specpart_cli.cpp); nlohmann/json serializes the report as in
    pipeline.cpp:169-215."""
    src = PKG / "tools" / "specpart_cli.cpp"
    if CLI.exists() and CLI.stat().st_mtime >= max(src.stat().st_mtime, LIB.stat().st_mtime,
                                                   (ROOT / "include" / "specpart_b200.h").stat().st_mtime):
        return
    CLI.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), "-I", str(NLOHMANN), str(src), "-L", str(PKG),
           "-lspecpart_b200", "-Wl,-rpath,$ORIGIN/../paper_2105_00578_b200", "-o", str(CLI)]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)


def _build_shim_test(verbose: bool) -> None:
    """tests/cpp/{shim,caller}_test.cpp against include/specpart_b200.hpp + the library (reference-style
    C++ callers that compile unchanged against the shim; nlohmann/json for RunReport::to_json)."""
    for name in ("shim_test", "caller_test"):
        src = ROOT / "tests" / "cpp" / f"{name}.cpp"
        exe = ROOT / "build" / name
        if not src.exists():
            continue
        if exe.exists() and exe.stat().st_mtime >= max(src.stat().st_mtime, LIB.stat().st_mtime,
                                                       (ROOT / "include" / "specpart_b200.hpp").stat().st_mtime):
            continue
        exe.parent.mkdir(parents=True, exist_ok=True)
        cmd = ["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), "-I", str(NLOHMANN), str(src), "-L", str(PKG),
               "-lspecpart_b200", "-Wl,-rpath,$ORIGIN/../paper_2105_00578_b200", "-o", str(exe)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
    print(LIB)
