"""Self-synchronization decoder on the GPU (reference sync_decoder.py).

Phases: intra-sequence synchronization (K2: one warp per sequence, one lane
per subsequence, exits handed to the right neighbour with warp shuffles and
convergence detected with ballots), inter-sequence seam passes (K3), the
output-index scan (K5) and the staged decode-and-write (K7).  ``decode``
runs the fused single-pass kernels; the sub-steps keep the reference's
SyncState arrays so intermediate states can be compared bit-for-bit.
"""

from __future__ import annotations

import time

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, load, ptr, stream_handle
from ._pipeline import run_decode
from .device import DeviceReport, Workspace, d2h, device_stream, empty, h2d
from .errors import NoFixpoint
from .staging import DEFAULT_CAPACITY, DecodeStats
from .state import SyncState, output_index

__all__ = ["SyncState", "output_index", "intra_sync", "inter_sync", "synchronize", "decode"]


class _DevState:
    """SyncState arrays on the device for the duration of a sub-step."""

    def __init__(self, stream, state: SyncState | None, device):
        ns, nq = stream.num_subseqs, stream.num_seqs
        st = state or SyncState.empty(ns, nq)
        self.host = st
        self.entries = h2d(_pad(st.entry_bits, np.int64), device)
        self.exits = h2d(_pad(st.exit_bits, np.int64), device)
        self.counts = h2d(_pad(st.counts, np.int64), device)
        self.synced = h2d(_pad(st.synced.astype(np.uint8), np.uint8), device)
        self.iters = h2d(_pad(st.iterations, np.int32), device)

    def args(self):
        return ptr(self.entries), ptr(self.exits), ptr(self.counts), ptr(self.synced), ptr(self.iters)

    def download(self, stream) -> SyncState:
        ns, nq = stream.num_subseqs, stream.num_seqs
        st = self.host
        st.entry_bits[:] = d2h(self.entries, np.int64)[:ns]
        st.exit_bits[:] = d2h(self.exits, np.int64)[:ns]
        st.counts[:] = d2h(self.counts, np.int64)[:ns]
        st.synced[:] = d2h(self.synced, np.uint8)[:ns].astype(bool)
        st.iterations[:] = d2h(self.iters, np.int32)[:nq]
        return st


def _pad(a, dt):
    a = np.ascontiguousarray(a, dtype=dt)
    return a if a.size else np.zeros(1, dt)


def _ws(stream, device):
    nbytes = (2 * stream.num_subseqs + 15) // 16 * 16 + 8 * stream.num_seqs + 256
    return Workspace.get(nbytes, device, "sync"), nbytes


def intra_sync(stream, s: int, state: SyncState | None = None, seed: int | None = None,
               early_exit: bool = True, stats: DecodeStats | None = None) -> SyncState:
    """Synchronize sequence ``s`` (sync_decoder.py:39-59)."""
    ds = device_stream(stream)
    dev = ds.device
    dst = _DevState(stream, state, dev)
    if stream.num_seqs:
        seeds = np.full(stream.num_seqs, -1, np.int64)
        seeds[s] = -2 if seed is None else int(seed)
        sd = h2d(seeds, dev)
        ws, wsb = _ws(stream, dev)
        rep = DeviceReport(dev).init()
        check(load().bh_intra_sync_ex(ds.ref, ptr(sd), 0, None, *dst.args(), ptr(ws), wsb, rep.ptr,
                                      stream_handle()), "intra_sync")
        r = rep.read()
        check(r.status, "intra_sync", r.fail_slot)
        if stats is not None:
            stats.add_bits("sync", r.bits_sync)
    return dst.download(stream)


def _seam_passes(stream, ds, dst, stats):
    lib = load()
    ws, wsb = _ws(stream, ds.device)
    for _ in range(max(stream.num_seqs, 1)):
        rep = DeviceReport(ds.device).init()
        stale = _lib.U64(0)
        check(lib.bh_inter_sync_pass(ds.ref, *dst.args(), ptr(ws), wsb, rep.ptr, C.byref(stale),
                                     stream_handle()), "inter_sync")
        r = rep.read()
        check(r.status, "inter_sync", r.fail_slot)
        if stats is not None:
            stats.add_bits("sync", r.bits_sync)
        if stale.value == 0:
            return
    raise NoFixpoint(f"sequence seams did not stabilize within {stream.num_seqs} passes")


def inter_sync(stream, state: SyncState, workers: int = 1, stats: DecodeStats | None = None) -> SyncState:
    """Seam passes until no sequence's seed changes (sync_decoder.py:116-149)."""
    if stream.num_seqs <= 1:
        return state
    ds = device_stream(stream)
    dst = _DevState(stream, state, ds.device)
    _seam_passes(stream, ds, dst, stats)
    return dst.download(stream)


def synchronize(stream, workers: int = 1, early_exit: bool = True,
                stats: DecodeStats | None = None) -> SyncState:
    """Intra-sequence sync of every sequence, then the seam passes."""
    ds = device_stream(stream)
    dst = _DevState(stream, None, ds.device)
    if stream.num_seqs:
        ws, wsb = _ws(stream, ds.device)
        rep = DeviceReport(ds.device).init()
        check(load().bh_intra_sync(ds.ref, int(early_exit), *dst.args(), ptr(ws), wsb, rep.ptr,
                                   stream_handle()), "intra_sync")
        r = rep.read()
        check(r.status, "intra_sync", r.fail_slot)
        if stats is not None:
            stats.add_bits("sync", r.bits_sync)
        if stream.num_seqs > 1:
            _seam_passes(stream, ds, dst, stats)
    return dst.download(stream)


def decode(stream, workers: int = 1, capacity: int = DEFAULT_CAPACITY, tuner_config=None,
           early_exit: bool = True, stats: DecodeStats | None = None, timings: dict | None = None,
           device_out: bool = False):
    """Decode a stream without using its gap array; returns uint16 symbols."""
    t_enter = time.perf_counter()  # timings cover the whole call
    return run_decode(stream, _lib.VARIANT_SYNC, capacity, tuner_config, stats, timings,
                      return_device=device_out, t_enter=t_enter)
