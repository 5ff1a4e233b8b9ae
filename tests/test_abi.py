"""libhbfs.so loads without a GPU and exports every symbol include/hbfs.h declares."""

from __future__ import annotations

import ctypes as C
import os
import re

from conftest import REPO


def declared_symbols():
    with open(os.path.join(REPO, "include", "hbfs.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(hbfs_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("hbfs_graph_from_csr", "hbfs_graph_build", "hbfs_bfs", "hbfs_validate",
              "hbfs_sample_sources", "hbfs_graph_generate", "hbfs_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1704_02259_b200 import _lib
    from paper_1704_02259_b200._build import build

    build()
    lib = C.CDLL(_lib.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_version_and_error_plumbing_without_gpu():
    from paper_1704_02259_b200 import _lib

    lib = _lib.load()
    assert lib.hbfs_version() >= 100
    # invalid-argument paths return status codes, never crash, no device needed
    rc = lib.hbfs_graph_info(None, None, None, None, None, None)
    assert rc == _lib.HBFS_EINVAL
    assert b"null" in lib.hbfs_last_error()


def test_struct_layouts_match_header():
    from paper_1704_02259_b200 import _lib

    assert C.sizeof(_lib.hbfs_params) == 4 + 4 + 8 + 8 + 4 + 4 + 4 + 4
    assert C.sizeof(_lib.hbfs_layer_row) == 4 + 4 + 7 * 8 + 8
