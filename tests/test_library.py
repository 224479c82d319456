"""The C-ABI library builds, loads without a GPU, and exports exactly what
include/srdl.h declares; the ctypes descriptors match the C layout."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2604_20073_b200 import build as builder
from paper_2604_20073_b200 import device as dev

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "srdl.h")


@pytest.fixture(scope="module")
def lib():
    builder.build()
    return dev.load_library()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|void|uint64_t|const char \*)\s*(srdl_\w+)\(", text, re.M)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(dev._SIGNATURES), "ctypes signatures out of sync with srdl.h"


def test_version_without_gpu(lib):
    assert lib.srdl_version() == 1


def test_descriptor_layout_matches_c(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "srdl.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(srdl_segment),"
        " sizeof(srdl_atom), sizeof(srdl_plan), sizeof(srdl_exec), offsetof(srdl_plan, atom),"
        " offsetof(srdl_exec, bitmap)); return 0;}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()))
    want = [
        ctypes.sizeof(dev.Segment),
        ctypes.sizeof(dev.AtomDesc),
        ctypes.sizeof(dev.PlanDesc),
        ctypes.sizeof(dev.ExecDesc),
        dev.PlanDesc.atom.offset,
        dev.ExecDesc.bitmap.offset,
    ]
    assert got == want
    assert ctypes.sizeof(dev.PlanDesc) + ctypes.sizeof(dev.ExecDesc) < 4096  # kernel parameter space


def test_engine_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2604_20073_b200 import DeviceUnavailable, Engine, parse

    with pytest.raises(DeviceUnavailable):
        Engine(parse(".decl R(a:symbol)\n"))


def test_col_ptrs_single_row_any_stride():
    """A one-row set produced by a transpose (strides (1, arity)) is a valid
    row set: column c starts c words after the first (regression: the
    distributed all-gather of a single staged tuple)."""
    import torch

    t = torch.arange(2, dtype=torch.int32).view(1, 2).t().contiguous()  # (2, 1), strides (1, 2)
    ptrs = dev.col_ptrs(t)
    assert ptrs[1] - ptrs[0] == 4
    wide = torch.zeros((3, 5), dtype=torch.int32)
    ptrs = dev.col_ptrs(wide)
    assert ptrs[2] - ptrs[0] == 2 * 5 * 4
    with pytest.raises(Exception):
        dev.col_ptrs(torch.zeros((5, 3), dtype=torch.int32).t())


def test_per_rule_kernels_compile_for_sm100a(lib):
    """The generated per-plan kernel source compiles with NVRTC for sm_100a
    (no GPU needed): the triangle's depth-3 plan and DOOP's deepest rule."""
    from paper_2604_20073_b200 import compile_program, parse, suites
    from paper_2604_20073_b200.wcoj import encode_shape

    tri = compile_program(parse(suites.TRIANGLE_PROGRAM)).strata[-1].plans[0]
    doop = compile_program(parse(suites.BASELINE_PROGRAMS["doop"][0]))
    deep = max((p for st in doop.strata for p in st.plans), key=lambda p: p.depth)
    for plan, mode in ((tri, 2), (deep, 2), (tri, 1)):
        nb = ctypes.c_uint64(0)
        rc = lib.srdl_wcoj_jit_compile_check(ctypes.byref(encode_shape(plan)), mode, ctypes.byref(nb))
        if rc == 2:
            pytest.skip("NVRTC unavailable")
        assert rc == 0, lib.srdl_last_error().decode()
        assert nb.value > 10_000
