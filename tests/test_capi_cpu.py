"""The C-ABI library loads without a GPU and exports every symbol that
include/bsparse.h declares, with the argument counts the ctypes binding
uses; workspace-size functions are pure host code."""

import os
import re

import pytest

from paper_1805_03380_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "bsparse.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:int|int64_t|size_t|const char \*)\s*\*?\s*(as_\w+)\s*\(([^)]*)\)\s*;", src):
        args = [a for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        out[m.group(1)] = len(args)
    return out


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    decl = _declared()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name


def test_binding_matches_header(lib):
    decl = _declared()
    assert set(decl) == set(_lib.SIGNATURES), set(decl) ^ set(_lib.SIGNATURES)
    for name, nargs in decl.items():
        assert len(_lib.SIGNATURES[name][1]) == nargs, name


def test_version_and_workspace_sizes_host_only(lib):
    assert lib.as_abi_version() == 1
    assert lib.as_build_workspace_bytes(1_000_000, 10_000) > 16 * 1_000_000
    assert lib.as_transpose_workspace_bytes(0, 0) > 0
    assert lib.as_trace_workspace_bytes(100, 10, 10) >= 256
    assert lib.as_spgemm_workspace_bytes(5, 0, 0) > 0
