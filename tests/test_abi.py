"""The C-ABI library builds, loads, exports every symbol include/rfd.h declares,
and validates arguments on the host (no GPU needed: no compute calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2302_00942_b200 import build as rfd_build
from paper_2302_00942_b200 import rfd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    text = open(os.path.join(ROOT, "include", "rfd.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rfd_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    rfd_build.build()
    return rfd.load_library()


def test_header_symbols_exported(lib):
    declared = _declared_functions()
    assert declared, "no functions parsed from include/rfd.h"
    assert sorted(rfd.EXPORTED) == declared
    for name in declared:
        assert hasattr(lib, name), name


def test_sm100a_code_in_library():
    import subprocess
    import shutil
    rfd_build.build()
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", rfd.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _create(lib, pts, n, eps=0.1, lam=-1.0, m=16):
    h = ctypes.c_void_p()
    ptr = ctypes.c_void_p(pts.ctypes.data) if pts is not None else None
    st = lib.rfd_plan_create(ptr, n, eps, lam, m, 0, None, ctypes.byref(h))
    return st, h


def test_argument_validation_is_host_side(lib):
    pts = np.zeros((4, 3), np.float32)
    assert _create(lib, None, 4)[0] == rfd.RFD_EINVAL
    assert _create(lib, pts, 0)[0] == rfd.RFD_EINVAL
    assert _create(lib, pts, 4, m=0)[0] == rfd.RFD_EINVAL
    assert _create(lib, pts, 4, m=rfd.RFD_MAX_M + 1)[0] == rfd.RFD_EINVAL
    assert _create(lib, pts, 4, eps=0.0)[0] == rfd.RFD_EINVAL
    assert _create(lib, pts, 4, eps=float("inf"))[0] == rfd.RFD_EINVAL
    assert _create(lib, pts, 4, lam=float("nan"))[0] == rfd.RFD_EINVAL
    st, h = _create(lib, pts, 4, eps=-1.0)
    assert st == rfd.RFD_EINVAL and not h.value
    assert b"eps" in lib.rfd_last_error()
    assert lib.rfd_integrate(None, None, 1, None, None) == rfd.RFD_EINVAL
    lib.rfd_destroy(None)  # NULL-safe


def test_no_fallback_when_library_missing(tmp_path, monkeypatch):
    monkeypatch.setattr(rfd, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rfd.load_library(str(tmp_path / "missing.so"))
