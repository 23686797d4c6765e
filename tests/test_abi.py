"""C-ABI library: loads on a CPU-only host and exports every symbol that
include/cvz_b200.h declares (no compute calls -- there is no GPU here)."""

import ctypes
import os
import re

from conftest import ROOT
from paper_2108_00529_b200 import _native


def header_symbols():
    text = open(os.path.join(ROOT, "include", "cvz_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*|long long)\s*\*?\s*(cvz_\w+)\s*\(",
                                 text, flags=re.M)))


def test_library_exports_header():
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, s


def test_version_and_counters_callable_without_gpu():
    lib = _native.load()
    assert lib.cvz_version() == 1
    assert lib.cvz_launch_count() >= 0


def test_built_for_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_native.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out[:400]
