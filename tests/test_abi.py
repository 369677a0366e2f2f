"""The C-ABI library loads on a CPU-only host and exports every entry point
include/filterkit_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "filterkit_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(fk_[a-z_0-9]+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2212_09005_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2212_09005_b200 import _build
        _build.build()
    return _lib.load()


def test_header_declares_entry_points():
    names = _declared()
    assert "fk_tcf_insert" in names and "fk_tcf_query" in names and "fk_tcf_delete" in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2212_09005_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fk_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    assert set(_lib.exported_symbols()) <= exported


def test_version_calls_without_gpu(lib):
    assert b"sm_100a" in lib.fk_version()
    assert lib.fk_abi_version() == 1


def test_library_is_sm100a_only(lib):
    from paper_2212_09005_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2212_09005_b200 import Tcf
    with pytest.raises(RuntimeError):
        Tcf(num_blocks=8)
