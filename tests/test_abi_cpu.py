"""The C ABI: the shared library loads without a GPU and exports every entry
point include/b200huff.h declares; the Python binding covers all of them."""

import re
from pathlib import Path

from paper_2201_09118_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "b200huff.h"


def declared():
    return sorted(set(re.findall(r"\b(bh_[a-z0-9_]+)\s*\(", HEADER.read_text())))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert missing == []
    assert lib.bh_version() >= 100


def test_binding_covers_header():
    assert sorted(_lib.SIGNATURES) == declared()


def test_status_codes_and_strings():
    lib = _lib.load()
    for code in range(0, 10):
        assert lib.bh_status_string(code)
    assert lib.bh_table_bytes(1024) > 0 and lib.bh_report_bytes() >= 128
    assert lib.bh_scan_workspace_bytes(1 << 20) > 0


def test_status_maps_to_reference_exceptions():
    import paper_2201_09118_b200 as ph
    import pytest
    for code, exc in ((1, ph.InvalidCode), (2, ph.Truncated), (3, ph.BadGap), (4, ph.NoFixpoint),
                      (5, ph.NotPresent), (6, ph.GapOverflow)):
        with pytest.raises(exc):
            _lib.check(code, "x")
    with pytest.raises(ValueError):
        _lib.check(7, "x")
