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


def test_report_struct_matches_device_report():
    """ctypes Report mirrors bh_report (same size as the device-side report)."""
    import ctypes as C
    assert C.sizeof(_lib.Report) == _lib.load().bh_report_bytes()


def test_split_phases_reference_names_and_wall_sum():
    """timings carry the reference's phase names (gap_decoder.py:82-92,
    sync_decoder.py:185-211) and add up to the call's wall time
    (tests/test_container_cli.py:253-266)."""
    import pytest
    from paper_2201_09118_b200._timing import split_phases
    st = [1_000_000, 1_000_000, 1_400_000, 1_600_000, 1_600_000, 2_000_000]  # ns
    t = {}
    split_phases(t, True, st, 0.002, 0.010, tuned=False)
    assert list(t) == ["entries_from_gap", "count_pass", "decode_write"]
    assert sum(t.values()) == pytest.approx(0.012)
    assert t["count_pass"] == pytest.approx(600e-6)
    t = {}
    split_phases(t, False, st, 0.001, 0.005, tuned=True)
    assert list(t) == ["intra_sync", "inter_sync", "output_index", "tune", "decode_write"]
    assert t["inter_sync"] == pytest.approx(400e-6) and t["tune"] == 0.0
    assert sum(t.values()) == pytest.approx(0.006)
    t = {}
    split_phases(t, True, [2 ** 64 - 1, 0, 0, 0, 0, 0], 0.001, 0.003, tuned=False)  # no stamps
    assert sum(t.values()) == pytest.approx(0.004)
