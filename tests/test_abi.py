"""CPU checks of the C-ABI boundary: libgoat.so builds, loads and exports
every symbol include/goat.h declares.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2111_05366_b200", "libgoat.so")


@pytest.fixture(scope="module")
def lib_path():
    from paper_2111_05366_b200 import build
    return build.build()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "goat.h")).read()
    return sorted(set(re.findall(r"\b(goat_[a-z_0-9]+)\s*\(", hdr)))


def test_header_declares_expected_surface():
    from paper_2111_05366_b200._lib import EXPORTS
    assert declared_symbols() == sorted(EXPORTS)


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (goat_[a-z_0-9]+)$", out, flags=re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_binds(lib_path):
    from paper_2111_05366_b200 import _lib
    lib = _lib.load()
    assert b"sm_100a" in lib.goat_version()
    for name in _lib.EXPORTS:
        assert hasattr(lib, name)


def test_library_is_sm100a_only(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_tensor_core_path_is_tcgen05(lib_path):
    """The fp32 gradient GEMM must be tcgen05/TMA/TMEM (not mma.sync/wmma)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib_path], capture_output=True,
                         text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in out, mnemonic
    assert "HMMA" not in out.replace("UTCHMMA", "")
