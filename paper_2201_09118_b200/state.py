"""Synchronization state and the output-index scan (reference state.py:16-53).

``SyncState`` keeps the reference's host arrays (int64 entry/exit/count per
subsequence, bool synced, int32 iterations per sequence) so the sub-step API
is a drop-in; the arrays are produced by the GPU kernels.  ``output_index``
runs the decoupled look-back scan kernel (K5, csrc/decode.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import check, load, ptr, require_cuda, stream_handle
from .device import Workspace, d2h, empty, h2d


@dataclass
class SyncState:
    entry_bits: np.ndarray
    exit_bits: np.ndarray
    counts: np.ndarray
    synced: np.ndarray
    iterations: np.ndarray

    @staticmethod
    def empty(num_subseqs: int, num_seqs: int) -> "SyncState":
        return SyncState(np.zeros(num_subseqs, np.int64), np.zeros(num_subseqs, np.int64),
                         np.zeros(num_subseqs, np.int64), np.zeros(num_subseqs, bool),
                         np.zeros(num_seqs, np.int32))

    def copy(self) -> "SyncState":
        return SyncState(self.entry_bits.copy(), self.exit_bits.copy(), self.counts.copy(),
                         self.synced.copy(), self.iterations.copy())


def output_index_device(counts_dev, n: int, device):
    """Device tensor of n int64 counts -> device tensor of n+1 exclusive offsets."""
    lib = load()
    oi = empty(n + 1, np.int64, device)
    wsb = lib.bh_scan_workspace_bytes(n)
    ws = Workspace.get(wsb, device, "scan")
    check(lib.bh_output_index(ptr(counts_dev), n, ptr(oi), ptr(ws), wsb, stream_handle()), "output_index")
    return oi


def output_index(counts) -> np.ndarray:
    """Exclusive prefix sum of per-subsequence counts, length n+1 (GPU scan)."""
    torch = require_cuda()
    c = np.ascontiguousarray(counts, dtype=np.int64)
    dev = torch.device("cuda", torch.cuda.current_device())
    oi = output_index_device(h2d(c if c.size else np.zeros(1, np.int64), dev), len(c), dev)
    return d2h(oi, np.int64)[: len(c) + 1]
