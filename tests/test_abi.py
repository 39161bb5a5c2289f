"""The C-ABI boundary: libspgcm.so loads without a GPU and exports every
function include/spgcm.h declares; the Python binding knows all of them."""
from __future__ import annotations

import ctypes
import os
import re

from paper_2411_03357_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header: str) -> set[str]:
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    lib = _native.load_spgcm()
    names = declared("spgcm.h")
    assert names, "no declarations parsed"
    for n in sorted(names):
        assert hasattr(lib, n), f"libspgcm.so does not export {n}"
    assert set(_native.SPGCM_SYMBOLS) == names


def test_version_and_errors_without_gpu():
    lib = _native.load_spgcm()
    assert b"sm_100a" in lib.sp_version()
    # argument validation happens before any CUDA call
    assert lib.sp_ctx_create(None, None) == _native.SP_EINVAL
    assert lib.sp_seal_batch(None, None, 1, None) == _native.SP_EINVAL


def test_desc_layout_matches_header():
    assert ctypes.sizeof(_native.SpDesc) == 56
    assert _native.SpDesc.iv.offset == 8 and _native.SpDesc.src.offset == 24 and _native.SpDesc.status.offset == 48


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2411_03357_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
