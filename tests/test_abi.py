"""The C-ABI library loads on CPU and exports every symbol include/tissuesim_b200.h declares."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2503_18616_b200 import _native as N
from paper_2503_18616_b200.errors import NativeLibraryError


def declared_functions():
    text = open(os.path.join(ROOT, "include", "tissuesim_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int32_t|int64_t|char\s*\*|const char\s*\*)\s*\*?\s*(ts_\w+)\s*\(",
                                  text, flags=re.M)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "ts_env_step" in names and "ts_create" in names and len(names) >= 14


def test_library_exports_every_declared_symbol():
    lib = N.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert sorted(declared_functions()) == N.exported_symbols()


def test_nm_exports():
    out = os.popen(f"nm -D --defined-only {N.LIB_PATH}").read()
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_abi_version_and_errors():
    lib = N.load()
    assert lib.ts_abi_version() == 3
    h = ctypes.c_void_p()
    rc = lib.ts_create(None, None, 0, ctypes.byref(h))
    assert rc == N.TS_ERR_INVALID
    assert b"null" in lib.ts_last_error()


def test_graph_launch_rejects_null_graph():
    """The step_numpy launch helpers validate before touching CUDA (safe on a CPU-only host)."""
    lib = N.load()
    for fn in (lib.ts_graph_launch, lib.ts_graph_launch_sync):
        assert fn(None, None) == N.TS_ERR_INVALID
        assert b"null graph" in lib.ts_last_error()


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {N.LIB_PATH}").read()
    assert "sm_100a" in out


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(NativeLibraryError):
        N.load()
