"""Gap-array decoder on the GPU (reference gap_decoder.py).

Entry bits come straight from the per-subsequence forward skips, so there is
no speculation: the fused kernel counts each subsequence's codewords, obtains
its output offset through a decoupled look-back, and writes the staged symbols
in the same pass.  The sub-steps keep the reference's arrays.
"""

from __future__ import annotations

import time

import numpy as np

from . import _lib
from ._lib import check, load, ptr, stream_handle
from ._pipeline import run_decode
from .device import DeviceReport, d2h, device_stream, empty, h2d
from .errors import BadGap, NotPresent
from .staging import DEFAULT_CAPACITY, DecodeStats
from .state import SyncState, output_index_device

__all__ = ["entries_from_gap", "count_pass", "decode"]


def entries_from_gap(stream) -> SyncState:
    """All-synced state with entry = boundary + gap (gap_decoder.py:24-33)."""
    if stream.gap is None:
        raise NotPresent("the stream carries no gap array")
    ns = stream.num_subseqs
    st = SyncState.empty(ns, stream.num_seqs)
    if ns:
        ds = device_stream(stream)
        e = empty(ns, np.int64, ds.device)
        check(load().bh_entries_from_gap(ds.ref, ptr(e), stream_handle()), "entries_from_gap")
        st.entry_bits[:] = d2h(e, np.int64)[:ns]
    st.synced[:] = True
    return st


def count_pass(stream, state: SyncState, workers: int = 1, stats: DecodeStats | None = None) -> np.ndarray:
    """Count each slot's codewords between consecutive entries; returns the output index."""
    ns = stream.num_subseqs
    if ns == 0:
        if stats is not None:
            stats.add_bits("count_pass", 0)
        if stream.symbol_count:
            raise BadGap(f"gap entries give 0 symbols; the header says {stream.symbol_count}")
        return np.zeros(1, np.int64)
    ds = device_stream(stream)
    dev = ds.device
    e = h2d(np.ascontiguousarray(state.entry_bits, np.int64), dev)
    c = empty(ns, np.int64, dev)
    x = empty(ns, np.int64, dev)
    rep = DeviceReport(dev).init()
    check(load().bh_count_windows(ds.ref, 1, ptr(e), ptr(c), ptr(x), rep.ptr, stream_handle()), "count_pass")
    r = rep.read()
    check(r.status, "count_pass", r.fail_slot)
    if stats is not None:
        stats.add_bits("count_pass", r.bits_count)
    oi_d = output_index_device(c, ns, dev)
    state.counts[:] = d2h(c, np.int64)[:ns]
    state.exit_bits[:] = d2h(x, np.int64)[:ns]
    oi = d2h(oi_d, np.int64)[: ns + 1]
    if int(oi[-1]) != stream.symbol_count:
        raise BadGap(f"gap entries give {int(oi[-1])} symbols; the header says {stream.symbol_count}")
    return oi


def decode(stream, workers: int = 1, capacity: int = DEFAULT_CAPACITY, tuner_config=None,
           stats: DecodeStats | None = None, timings: dict | None = None, device_out: bool = False):
    """Decode a stream using its gap array; returns uint16 symbols."""
    t_enter = time.perf_counter()  # timings cover the whole call
    if stream.gap is None:
        raise NotPresent("the stream carries no gap array")
    return run_decode(stream, _lib.VARIANT_GAP, capacity, tuner_config, stats, timings,
                      return_device=device_out, t_enter=t_enter)
