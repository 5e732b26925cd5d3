"""CPU-side checks of the C ABI: the in-tree library loads and exports every
entry point include/qgs_b200.h declares (no device calls)."""

import os
import re

from paper_2411_16392_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "qgs_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qgs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared()
    for n in ("qgs_preprocess", "qgs_bin", "qgs_forward", "qgs_backward", "qgs_chain"):
        assert n in names


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for n in declared():
        assert hasattr(L, n), n
    assert sorted(_lib.EXPORTS) == declared()


def test_host_only_queries():
    L = _lib.load()
    assert L.qgs_version() >= 1
    assert L.qgs_prep_bytes(1000) >= 1000 * (256 + 128 + 16 + 4 + 8)
    assert L.qgs_bin_workspace_bytes(10, 1000, 64) >= 16 * 1000
    assert isinstance(L.qgs_last_error(), bytes)
