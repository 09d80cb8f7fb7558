"""The C-ABI library loads and exports every symbol include/shiro.h declares
(no compute calls: this runs on CPU-only boxes)."""
import ctypes
import os
import re

import paper_2512_20178_b200 as sh
from paper_2512_20178_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "shiro.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(shiro_[a-z_]+)\s*\(", src)) - {"shiro_alltoallv_fn"})


def test_library_exports_every_declared_symbol():
    lib = sh.load()
    names = declared_symbols()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_binding_covers_header():
    lib = sh.load()
    for name in declared_symbols():
        f = getattr(lib, name)
        assert f.restype is not None or name == "shiro_last_error", name


def test_error_path_and_last_error():
    lib = sh.load()
    rc = lib.shiro_plan_info(None, None)
    assert rc == 1 and b"NULL" in lib.shiro_last_error()
    assert lib.shiro_free(None) == 0


def test_no_fallback_without_library(tmp_path, monkeypatch):
    monkeypatch.setattr(binding, "_lib", None)
    monkeypatch.setattr(binding, "LIB_PATH", str(tmp_path / "missing.so"))
    import pytest
    with pytest.raises(ImportError):
        binding.load()
