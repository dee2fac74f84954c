"""CPU: the C-ABI library loads, exports every declared symbol, and its structs
match the ctypes mirror (no compute: there is no GPU here)."""
import re
import subprocess
import tempfile
from pathlib import Path

import ctypes
import pytest

from paper_2105_00578_b200 import abi

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "specpart_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(sp_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = abi.load_library()
    names = declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in abi.SIGNATURES, f"{name} missing from the ctypes mirror"


def test_struct_layouts_match_header():
    src = """
#include <stdio.h>
#include <stddef.h>
#include "specpart_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu\\n", sizeof(sp_graph), sizeof(sp_config), sizeof(sp_report), sizeof(sp_trace_record));
  printf("%zu %zu %zu\\n", offsetof(sp_report, cutsize), offsetof(sp_report, part_weights), offsetof(sp_report, poly_ms));
  printf("%zu %zu\\n", sizeof(sp_graph_info), offsetof(sp_graph_info, regular));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = Path(d) / "t.c"
        c.write_text(src)
        exe = Path(d) / "t"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(c), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = list(map(int, out))
    assert sizes[0] == ctypes.sizeof(abi.SpGraph)
    assert sizes[1] == ctypes.sizeof(abi.SpConfig)
    assert sizes[2] == ctypes.sizeof(abi.SpReport)
    assert sizes[3] == ctypes.sizeof(abi.SpTraceRecord)
    assert sizes[4] == abi.SpReport.cutsize.offset
    assert sizes[5] == abi.SpReport.part_weights.offset
    assert sizes[6] == abi.SpReport.poly_ms.offset
    assert sizes[7] == ctypes.sizeof(abi.SpGraphInfo)
    assert sizes[8] == abi.SpGraphInfo.regular.offset


def test_enums_follow_reference_order():
    # pipeline.hpp:16-18 — numeric values let a C++ shim static_cast between the enums
    assert abi.PROBLEM == {"auto": 0, "combinatorial": 1, "generalized": 2, "normalized": 3}
    assert abi.PRECOND == {"auto": 0, "jacobi": 1, "polynomial": 2, "amg": 3, "none": 4}
    assert abi.INIT == {"auto": 0, "random": 1, "piecewise": 2}


def test_context_creation_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2105_00578_b200 import Context, SpecpartError
    with pytest.raises(SpecpartError):
        Context(0)


@pytest.mark.parametrize("name", ["shim_test", "caller_test"])
def test_shim_test_binary_links(name):
    exe = ROOT / "build" / name
    assert exe.exists(), f"build() compiles tests/cpp/{name}.cpp against include/specpart_b200.hpp"
    out = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
    assert "libspecpart_b200.so" in out and "not found" not in out.split("libspecpart_b200.so")[1].split("\n")[0]
