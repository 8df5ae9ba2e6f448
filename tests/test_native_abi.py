"""The C-ABI library loads and exports every symbol declared in include/bddc.h."""
import ctypes
import os
import re

import pytest

from paper_1901_02090_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "bddc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bddc_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_loads():
    _native.build_native()
    lib = _native.load()
    assert lib.bddc_version() >= 1
    assert lib.bddc_geom_size() == ctypes.sizeof(_native.Geom)


def test_every_declared_symbol_exported():
    _native.build_native()
    lib = ctypes.CDLL(_native.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares exactly those entry points
    assert set(declared) <= set(_native.EXPORTED)


def test_sm100a_cubin_embedded():
    import subprocess
    _native.build_native()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _native.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "DMMA" in sass   # FP64 tensor-core path present
