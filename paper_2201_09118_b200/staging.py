"""Staged decode-and-write (reference staging.py:65-147) on the GPU.

One warp per sequence stages its slots' symbols in shared memory and flushes
them with coalesced stores, with exactly the reference's window rule (the
slot containing the window limit straddles; an oversized slot bypasses the
buffer), so ``DecodeStats`` -- rounds, staged and bypass slots, bits -- match
the reference for any capacity (K7, csrc/decode.cu).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._lib import check, load, ptr, stream_handle
from .device import DeviceReport, d2h, device_stream, empty, h2d

DEFAULT_CAPACITY = 3584


@dataclass
class DecodeStats:
    phase_bits: dict = field(default_factory=dict)
    write_rounds: int = 0
    staged_slots: int = 0
    bypass_slots: int = 0

    def add_bits(self, phase: str, bits: int) -> None:
        self.phase_bits[phase] = self.phase_bits.get(phase, 0) + int(bits)

    @property
    def bits_decoded(self) -> int:
        return sum(self.phase_bits.values())

    def absorb_write(self, rep) -> None:
        self.add_bits("decode_write", rep.bits_write)
        self.write_rounds += int(rep.write_rounds)
        self.staged_slots += int(rep.staged_slots)
        self.bypass_slots += int(rep.bypass_slots)


def decode_write(stream, state, out_index, capacity: int = DEFAULT_CAPACITY, workers: int = 1,
                 sequences=None, out=None, stats: DecodeStats | None = None) -> np.ndarray:
    """Decode every slot's symbols to their output-index positions.

    ``workers`` is accepted for API compatibility (the GPU ignores it).
    """
    if capacity < 1:
        raise ValueError("staging capacity must be >= 1")
    lib = load()
    ds = device_stream(stream)
    dev = ds.device
    oi = np.ascontiguousarray(out_index, np.int64)
    n = int(oi[-1])
    e_d = h2d(np.ascontiguousarray(state.entry_bits, np.int64), dev)
    c_d = h2d(np.ascontiguousarray(state.counts, np.int64), dev)
    oi_d = h2d(oi, dev)
    seq_d, nids = None, stream.num_seqs
    if sequences is not None:
        seqs = np.ascontiguousarray(sequences, np.int64)
        nids = len(seqs)
        seq_d = h2d(seqs if nids else np.zeros(1, np.int64), dev)
    out_d = empty(n, np.uint16, dev)
    if out is not None and n:
        out_d[:n].copy_(h2d(np.ascontiguousarray(out[:n], np.uint16), dev))
    rep = DeviceReport(dev).init()
    if nids and stream.num_subseqs:
        check(lib.bh_decode_write(ds.ref, ptr(e_d), ptr(c_d), ptr(oi_d), ptr(seq_d), nids, int(capacity),
                                  ptr(out_d), n, rep.ptr, stream_handle()), "decode_write")
    r = rep.read()
    check(r.status, "decode_write", r.fail_slot)
    if stats is not None:
        stats.absorb_write(r)
    res = d2h(out_d, np.uint16)[:n]
    if out is not None:
        out[:n] = res
        return out
    return res
