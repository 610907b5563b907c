"""ctypes binding to libb200huff.so (the C ABI in include/b200huff.h).

The library is built in-tree (``__graft_entry__.build()`` or ``make -C
paper_2201_09118_b200/csrc``).  There is no fallback: if the shared object is
missing, or no CUDA device is present, every decode entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libb200huff.so"

BH_OK, BH_INVALID, BH_TRUNCATED, BH_BADGAP, BH_NOFIXPOINT = 0, 1, 2, 3, 4
BH_NOTPRESENT, BH_GAPOVERFLOW, BH_BAD_ARGUMENT, BH_CUDA_ERROR, BH_NEED_STAGED = 5, 6, 7, 8, 9
BH_LENGTHOVERFLOW, BH_EMPTY = 10, 11
VARIANT_GAP, VARIANT_SYNC, VARIANT_COARSE = 1, 2, 3
STREAM_COUNT_IS_CAPACITY = 1
WORD_PAD = 8

P = C.c_void_p
U64 = C.c_uint64
U32 = C.c_uint32
I32 = C.c_int
SZ = C.c_size_t


class Stream(C.Structure):
    _fields_ = [
        ("words_dev", P), ("total_bits", U64), ("symbol_count", U64),
        ("subseq_bits", U32), ("subseqs_per_seq", U32), ("symbol_width", U32),
        ("max_codes", U32), ("gap_dev", P), ("table_dev", P),
        ("first_entry", U32), ("flags", U32),
    ]


class Tune(C.Structure):
    _fields_ = [
        ("t_high", U32), ("capacity", U32), ("capacity_table", U32 * 64),
        ("early_exit", U32), ("collect_stats", U32), ("fused", U32), ("seam_passes", U32),
        ("max_len", U32), ("ctas", U32), ("min_len", U32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("pad0", C.c_int32), ("fail_slot", U64),
        ("bits_sync", U64), ("bits_count", U64), ("bits_write", U64),
        ("write_rounds", U64), ("staged_slots", U64), ("bypass_slots", U64),
        ("total_symbols", U64), ("stale_seams", U64), ("seam_passes", U64),
        ("repair_needed", U64), ("pad", U64 * 4), ("phase_ns", U64 * 6),
    ]


# name -> (restype, argtypes); every symbol declared in include/b200huff.h
SIGNATURES = {
    "bh_version": (I32, []),
    "bh_status_string": (C.c_char_p, [I32]),
    "bh_device_sm_count": (I32, []),
    "bh_table_bytes": (SZ, [U32]),
    "bh_table_build": (I32, [P, U32, P, U32, P]),
    "bh_table_build_explicit": (I32, [P, P, U32, P, U32, P]),
    "bh_canonical_codes": (I32, [P, U32, P, P]),
    "bh_workspace_bytes": (SZ, [P, I32, P]),
    "bh_decode_async": (I32, [P, I32, P, P, P, SZ, P, P]),
    "bh_decode": (I32, [P, I32, P, P, P, SZ, P, P]),
    "bh_report_bytes": (SZ, []),
    "bh_report_init": (I32, [P, P]),
    "bh_report_read": (I32, [P, P, P]),
    "bh_decode_workspace_bytes": (SZ, [P, I32, P]),
    "bh_intra_sync": (I32, [P, I32, P, P, P, P, P, P, SZ, P, P]),
    "bh_intra_sync_ex": (I32, [P, P, U32, P, P, P, P, P, P, P, SZ, P, P]),
    "bh_seam_check": (I32, [P, P, P, P, P, P]),
    "bh_inter_sync_pass": (I32, [P, P, P, P, P, P, P, SZ, P, P, P]),
    "bh_entries_from_gap": (I32, [P, P, P]),
    "bh_count_windows": (I32, [P, I32, P, P, P, P, P]),
    "bh_output_index": (I32, [P, U64, P, P, SZ, P]),
    "bh_scan_workspace_bytes": (SZ, [U64]),
    "bh_decode_write": (I32, [P, P, P, P, P, U64, U32, P, U64, P, P]),
    "bh_decode_write_classes": (I32, [P, P, P, P, P, U64, U32, U32, P, P, P, U64, P, I32, P]),
    "bh_check_total": (I32, [P, P, I32, P, P]),
    "bh_tuner_plan": (I32, [P, P, U32, P, P, P, P, P, SZ, P]),
    "bh_tuner_workspace_bytes": (SZ, [U64, U32]),
    "bh_sequence_counts": (I32, [P, P, P, P]),
    "bh_encode_workspace_bytes": (SZ, [U64]),
    "bh_encode_size": (I32, [P, U64, P, U32, P, SZ, P, P, P]),
    "bh_encode_pack": (I32, [P, U64, P, P, U64, U32, P, P, U64, P, P, SZ, P]),
    "bh_repack_units": (I32, [P, U64, U32, P, U64, P]),
    "bh_sequential_decode": (I32, [P, U64, U64, I32, P, P, P, P]),
    "bh_start_histogram": (I32, [P, U64, U32, P, U64, P]),
    "bh_coarse_decode": (I32, [P, P, U64, P, P, P]),
    "bh_profile_enable": (I32, [I32]),
    "bh_profile_read": (I32, [C.c_char_p, SZ, P, P, I32]),
    "bh_fill_caps": (I32, [P, P, U32, P]),
    "bh_workspace_reset": (I32, [P, SZ, P]),
    "bh_book_workspace_bytes": (SZ, [U32]),
    "bh_symbol_histogram": (I32, [P, U64, U32, P, P]),
    "bh_build_lengths": (I32, [P, U32, P, P, P]),
    "bh_tuner_class_freq": (I32, [P, P, P, P, U32, P]),
    "bh_fused_supported": (I32, [P, I32]),
    "bh_dequant_workspace_bytes": (SZ, [U64]),
    "bh_dequantize": (I32, [P, U64, P, P, P, U64, C.c_double, U32, I32, P, P, SZ, P, P]),
}

_lib = None


def load():
    """Load the shared library (no GPU needed); raises if it is not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_2201_09118_b200/csrc` (there is no CPU fallback)"
            )
        # BH_LIB: load an alternative build of the same library (A/B experiments)
        lib = C.CDLL(os.environ.get("BH_LIB") or str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_EXC = {
    BH_INVALID: errors.InvalidCode,
    BH_TRUNCATED: errors.Truncated,
    BH_BADGAP: errors.BadGap,
    BH_NOFIXPOINT: errors.NoFixpoint,
    BH_NOTPRESENT: errors.NotPresent,
    BH_GAPOVERFLOW: errors.GapOverflow,
    BH_LENGTHOVERFLOW: errors.LengthOverflow,
    BH_EMPTY: errors.EmptyInput,
}


def check(status: int, what: str = "", slot: int | None = None) -> None:
    """Translate a library status into the reference's exception classes."""
    if status == BH_OK:
        return
    msg = load().bh_status_string(status).decode()
    if what:
        msg = f"{what}: {msg}"
    if slot is not None and slot != 2 ** 64 - 1:
        msg += f" (subsequence {slot})"
    exc = _EXC.get(status)
    if exc is not None:
        raise exc(msg)
    if status == BH_BAD_ARGUMENT:
        raise ValueError(msg)
    raise RuntimeError(msg)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2201_09118_b200 decodes on a CUDA device (B200); none is visible")
    load()
    return torch


def stream_handle(torch_stream=None) -> int:
    import torch
    st = torch_stream or torch.cuda.current_stream()
    return st.cuda_stream


def profile_enable(on: bool = True) -> None:
    check(load().bh_profile_enable(1 if on else 0), "profile")


def profile_read() -> dict:
    """{phase: (total_ms, intervals)} accumulated since profile_enable()."""
    import numpy as np
    names = C.create_string_buffer(4096)
    ms = np.zeros(64, np.float32)
    cnt = np.zeros(64, np.uint32)
    n = load().bh_profile_read(names, 4096, ms.ctypes.data, cnt.ctypes.data, 64)
    if n < 0:
        raise RuntimeError("profile read failed")
    keys = names.value.decode().split("\n")[:n]
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys)}
