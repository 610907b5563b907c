"""Whole-decoder driver shared by sync_decoder.decode and gap_decoder.decode.

Calls ``bh_decode`` (include/b200huff.h) on the caller's current CUDA stream.
With ``stats`` requested it runs the reference-structured kernel pipeline so
the counters match the reference's DecodeStats; otherwise the fused
single-pass kernels.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from ._lib import check, load, ptr, require_cuda, stream_handle
from ._timing import split_phases
from .device import Workspace, d2h, device_stream, empty
from .staging import DEFAULT_CAPACITY


def make_tune(capacity: int = DEFAULT_CAPACITY, tuner_config=None, collect_stats: bool = False,
              fused: bool = True, seam_passes: int = 2, max_len: int = 0, min_len: int = 0) -> _lib.Tune:
    if capacity < 1:
        raise ValueError("staging capacity must be >= 1")
    t = _lib.Tune()
    t.capacity = int(capacity)
    if tuner_config is not None:
        if tuner_config.t_high > 255:
            raise ValueError("the device tuner supports t_high <= 255")
        t.t_high = int(tuner_config.t_high)
        for cls, cap in (tuner_config.capacity_table or {}).items():
            if 1 <= cls <= 64:
                t.capacity_table[cls - 1] = int(cap)
    t.early_exit = 1
    t.collect_stats = 1 if collect_stats else 0
    t.fused = 1 if fused else 0
    t.seam_passes = seam_passes
    t.max_len = int(max_len)
    t.min_len = int(min_len)
    return t


def run_decode(stream, variant: int, capacity: int = DEFAULT_CAPACITY, tuner_config=None,
               stats=None, timings=None, return_device: bool = False, fused: bool | None = None,
               t_enter: float | None = None):
    if t_enter is None:
        t_enter = time.perf_counter()
    torch = require_cuda()
    lib = load()
    ds = device_stream(stream)
    n = int(stream.symbol_count)
    if fused is None:
        fused = stats is None
    tune = make_tune(capacity, tuner_config, stats is not None, fused, max_len=stream.codebook.max_len,
                     min_len=stream.codebook.min_len)
    out = empty(n, np.uint16, ds.device)
    wsb = lib.bh_decode_workspace_bytes(ds.ref, variant, C.byref(tune))
    ws = Workspace.get(wsb, ds.device)
    rep = _lib.Report()
    if timings is not None:
        torch.cuda.current_stream(ds.device).synchronize()  # uploads belong to the first phase
    t_call = time.perf_counter()
    status = lib.bh_decode(ds.ref, variant, C.byref(tune), ptr(out), ptr(ws), wsb, C.byref(rep),
                           stream_handle())
    check(status, "decode", rep.fail_slot)
    if stats is not None:
        if variant == _lib.VARIANT_SYNC:
            stats.add_bits("sync", rep.bits_sync)
        else:
            stats.add_bits("count_pass", rep.bits_count)
        stats.absorb_write(rep)
    res = (out[:n] if n else out[:0]) if return_device else d2h(out, np.uint16)[:n]
    if timings is not None:
        if return_device:
            torch.cuda.current_stream(ds.device).synchronize()
        t_end = time.perf_counter()
        split_phases(timings, variant == _lib.VARIANT_GAP, list(rep.phase_ns), t_call - t_enter,
                     t_end - t_call, tuner_config is not None)
    return res
