"""The C-ABI library loads without a GPU and exports exactly the symbols
include/mglp_cuda.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2601_09026_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mglp_cuda.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mglp_[a-z_0-9]+)\s*\(", src)))


def test_library_built_in_tree():
    assert os.path.exists(N.LIB_PATH), "run __graft_entry__.build() first"


def test_loads_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    names = declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert sorted(N.EXPORTS) == declared()


def test_version_string_no_gpu_needed():
    assert b"sm_100a" in N.lib().mglp_version()


def test_sm100a_tensor_core_sass():
    """The shipped kernels are tcgen05 + TMA (UTC*MMA / UTMALDG in SASS)."""
    out = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in out.stdout
    assert "UTMALDG" in out.stdout
    assert "LDTM" in out.stdout
    assert "HGMMA" not in out.stdout  # no Hopper wgmma
