"""The C-ABI boundary on CPU: libwavekv.so loads (no GPU needed to load it)
and exports every entry point include/wavekv.h declares; the ctypes binding
declares the same set."""
import ctypes
import os
import re

from paper_2505_02922_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "wavekv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*int\s+(wk_\w+)\s*\(", src, flags=re.M))


def test_header_declares_the_binding_set():
    names = header_functions()
    assert len(names) >= 19
    assert names == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2505_02922_b200 import _build
    _build.build()
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in header_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert _lib.lib().wk_version() >= 3
