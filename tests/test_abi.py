"""CPU checks of the C-ABI boundary: the library builds, loads, and exports every
symbol include/tt.h declares; calls that need no GPU fail cleanly."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "tt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*([a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "while", "sizeof")))


def test_library_builds_and_exports_all_declared_symbols():
    from __graft_entry__ import _build_module
    build = _build_module()
    lib_path = build.build()
    lib = C.CDLL(lib_path)
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/tt.h but not exported"
    from paper_2309_03347_b200 import _lib
    assert sorted(_lib.SIG) == names


def test_binding_rejects_bad_arguments_without_gpu():
    from paper_2309_03347_b200 import _lib
    lib = _lib.lib()
    assert lib.tt_version().startswith(b"libtt-b200")
    # NULL descriptors are host-detectable errors
    st = lib.tt_matvec(None, None, None, None)
    assert st == 1
    assert b"NULL" in lib.tt_last_error()
    assert lib.als_local_apply(0, 1, 1, 1, 1, 1, 1, 1, None, None, None, None, None, None, 0, None) == 1
    assert lib.als_workspace(4, 2, 4, 2, 2, 4, 2, 4) > 0


def test_package_import_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_2309_03347_b200 import _lib
    with pytest.raises(ImportError):
        _lib.load(str(tmp_path / "missing.so"))
