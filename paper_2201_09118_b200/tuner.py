"""Compression-ratio tuner (reference tuner.py, Algorithm 2) on the GPU.

``plan`` classifies sequences by compression ratio, histograms the classes,
stable-sorts sequence ids by class and prefixes the class counts -- all in
device kernels (K6, csrc/decode.cu), integer-exact: class = min(ceil(count *
width / seq_bits), t_high + 1), zero-count sequences in class 1.
``decode_partitioned`` runs the staged write with each class's capacity in a
single launch (classes write disjoint output ranges, tuner.py:150-191).
The scalar helpers (classify, histogram, ...) keep the reference signatures.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from ._lib import check, load, ptr, stream_handle
from .device import DeviceReport, Workspace, d2h, device_stream, empty, h2d
from .errors import NonPositiveRatio
from .staging import DecodeStats

OVERFLOW_CAPACITY = 3584
SYMBOLS_PER_CLASS = 1024
MAX_T_HIGH = 255


@dataclass(frozen=True)
class TunerConfig:
    t_high: int = 8
    capacity_table: dict | None = None

    def __post_init__(self):
        if self.t_high < 1:
            raise ValueError("t_high must be >= 1")
        if self.capacity_table and any(v < 1 for v in self.capacity_table.values()):
            raise ValueError(f"capacities must be >= 1 (got {self.capacity_table})")


@dataclass
class PartitionPlan:
    t_high: int
    comp_ratio: np.ndarray
    comp_class: np.ndarray
    class_freq: np.ndarray
    permutation: np.ndarray
    class_start: np.ndarray
    capacity: np.ndarray

    def class_sequences(self, cls: int) -> np.ndarray:
        i = cls - 1
        lo = int(self.class_start[i])
        return self.permutation[lo: lo + int(self.class_freq[i])]


def classify(ratio: float, t_high: int) -> int:
    if ratio <= 0:
        raise NonPositiveRatio(f"compression ratio must be positive (got {ratio})")
    return t_high + 1 if ratio > t_high else math.ceil(ratio)


def histogram(classes, t_high: int) -> np.ndarray:
    c = np.asarray(classes, dtype=np.int64)
    return np.bincount(c - 1, minlength=t_high + 1).astype(np.int64)


def sort_by_class(classes) -> np.ndarray:
    return np.argsort(np.asarray(classes), kind="stable").astype(np.int64)


def class_starts(class_freq) -> np.ndarray:
    f = np.asarray(class_freq, dtype=np.int64)
    out = np.zeros(max(len(f), 1), dtype=np.int64)
    if len(f) > 1:
        out[1:] = np.cumsum(f[:-1])
    return out


def capacity(cls: int, config: TunerConfig) -> int:
    if not 1 <= cls <= config.t_high + 1:
        raise ValueError(f"class {cls} is outside 1..{config.t_high + 1}")
    if config.capacity_table and cls in config.capacity_table:
        return int(config.capacity_table[cls])
    return OVERFLOW_CAPACITY if cls > config.t_high else cls * SYMBOLS_PER_CLASS


def sequence_counts(stream, subseq_counts) -> np.ndarray:
    """Per-sequence symbol counts (GPU reduction)."""
    if stream.num_seqs == 0:
        return np.zeros(0, np.int64)
    ds = device_stream(stream)
    c = h2d(np.ascontiguousarray(subseq_counts, np.int64), ds.device)
    out = empty(stream.num_seqs, np.int64, ds.device)
    check(load().bh_sequence_counts(ds.ref, ptr(c), ptr(out), stream_handle()), "sequence_counts")
    return d2h(out, np.int64)[: stream.num_seqs]


def _ratios(stream, seq_counts: np.ndarray) -> np.ndarray:
    nq = stream.num_seqs
    bits = np.full(nq, stream.layout.seq_bits, dtype=np.int64)
    if nq:
        bits[-1] = stream.total_bits - (nq - 1) * stream.layout.seq_bits
    return (seq_counts * stream.codebook.symbol_width) / bits


def plan(stream, seq_counts, config: TunerConfig) -> PartitionPlan:
    if config.t_high > MAX_T_HIGH:
        raise ValueError(f"the device tuner supports t_high <= {MAX_T_HIGH}")
    lib = load()
    ds = device_stream(stream)
    dev = ds.device
    nq = stream.num_seqs
    C = config.t_high + 1
    sc = np.ascontiguousarray(seq_counts, np.int64)
    sc_d = h2d(sc if nq else np.zeros(1, np.int64), dev)
    cls_d, perm_d = empty(nq, np.int64, dev), empty(nq, np.int64, dev)
    freq_d, start_d = empty(C, np.int64, dev), empty(C, np.int64, dev)
    wsb = lib.bh_tuner_workspace_bytes(nq, config.t_high)
    ws = Workspace.get(wsb, dev, "tuner")
    check(lib.bh_tuner_plan(ds.ref, ptr(sc_d), config.t_high, ptr(cls_d), ptr(freq_d), ptr(perm_d),
                            ptr(start_d), ptr(ws), wsb, stream_handle()), "tuner plan")
    caps = np.array([capacity(c, config) for c in range(1, C + 1)], dtype=np.int64)
    return PartitionPlan(
        t_high=config.t_high,
        comp_ratio=_ratios(stream, sc),
        comp_class=d2h(cls_d, np.int64)[:nq],
        class_freq=d2h(freq_d, np.int64)[:C],
        permutation=d2h(perm_d, np.int64)[:nq],
        class_start=d2h(start_d, np.int64)[:C],
        capacity=caps,
    )


def decode_partitioned(stream, plan_: PartitionPlan, state, out_index, workers: int = 1,
                       out=None, stats: DecodeStats | None = None) -> np.ndarray:
    """Staged write per class, all classes in one launch (empty classes cost nothing)."""
    lib = load()
    ds = device_stream(stream)
    dev = ds.device
    oi = np.ascontiguousarray(out_index, np.int64)
    n = int(oi[-1])
    nq = stream.num_seqs
    out_d = empty(n, np.uint16, dev)
    if out is not None and n:
        out_d[:n].copy_(h2d(np.ascontiguousarray(out[:n], np.uint16), dev))
    rep = DeviceReport(dev).init()
    if nq and stream.num_subseqs:
        e_d = h2d(np.ascontiguousarray(state.entry_bits, np.int64), dev)
        c_d = h2d(np.ascontiguousarray(state.counts, np.int64), dev)
        oi_d = h2d(oi, dev)
        perm_d = h2d(np.ascontiguousarray(plan_.permutation, np.int64), dev)
        cls_d = h2d(np.ascontiguousarray(plan_.comp_class, np.int64), dev)
        caps = np.ascontiguousarray(plan_.capacity, np.uint32)
        caps_d = h2d(caps, dev)
        check(lib.bh_decode_write_classes(ds.ref, ptr(e_d), ptr(c_d), ptr(oi_d), ptr(perm_d), nq, 0,
                                          int(caps.max()), ptr(cls_d), ptr(caps_d), ptr(out_d), n,
                                          rep.ptr, 1, stream_handle()), "decode_partitioned")
    r = rep.read()
    check(r.status, "decode_partitioned", r.fail_slot)
    if stats is not None:
        stats.absorb_write(r)
    res = d2h(out_d, np.uint16)[:n]
    if out is not None:
        out[:n] = res
        return out
    return res
