"""ctypes front-end for the C oracle (huff_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg, never by the product package.  It restates the
reference decode path (parhuff, /root/reference/pkg/src/parhuff) on the CPU so
the CUDA path can be checked bit-for-bit; the restatement itself is pinned by
tests/test_oracle_golden.py against fixtures produced by the real reference
(tests/golden/make_golden.py).

Streams are duck-typed: anything with ``units``, ``layout`` (unit_bits,
units_per_subseq, subseqs_per_seq), ``total_bits``, ``symbol_count``, ``gap``
and ``codebook`` (kind, entries, symbol_width) works -- the reference's
EncodedStream and the B200 package's EncodedStream both qualify.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

OK, INVALID, TRUNCATED, NOFIXPOINT = 0, 1, 2, 4


class OracleError(Exception):
    def __init__(self, status: int, where: int):
        super().__init__(f"oracle status {status} at {where}")
        self.status = status
        self.where = where


def build() -> Path:
    src = HERE / "huff_oracle.c"
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


class _Src(C.Structure):
    _fields_ = [
        ("units", C.c_void_p), ("n_units", C.c_int64), ("ulog2", C.c_int32),
        ("unit_bits", C.c_int32), ("kind", C.c_int32), ("max_len", C.c_int32),
        ("first_code", C.c_void_p), ("len_count", C.c_void_p),
        ("first_index", C.c_void_p), ("symbols", C.c_void_p),
        ("trie_child", C.c_void_p), ("trie_symbol", C.c_void_p),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build()))
        P = C.c_void_p
        I = C.c_int64
        _lib.or_count_windows.argtypes = [P, P, P, I, I, I, P, P, P]
        _lib.or_decode_counted.argtypes = [P, P, P, P, P, I, I, P]
        _lib.or_oracle_decode.argtypes = [P, I, I, P, P, P]
        _lib.or_encode_pack.argtypes = [P, I, P, P, P, C.c_int32, C.c_int32, I, P, I]
        _lib.or_encode_pack.restype = I
        _lib.or_sync_sequence.argtypes = [P, I, I, I, I, I, I, C.c_int32, I, P, P, P, P, P, P]
        _lib.or_synchronize.argtypes = [P, I, I, I, I, I, C.c_int32, P, P, P, P, P, P]
        _lib.or_decode_write.argtypes = [P, I, I, P, P, P, P, I, I, P, P, P]
        _lib.or_canonical_table.argtypes = [P, I, P, P, P, P, P]
        _lib.or_canonical_table.restype = C.c_int32
        _lib.or_tuner_plan.argtypes = [P, I, I, I, I, I, P, P, P, P]
        _lib.or_dequantize.argtypes = [P, I, P, P, I, C.c_double, I, P]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class Table:
    """Canonical arrays (codebook.py:209-233) or a trie (codebook.py:235-260)."""

    kind: int
    max_len: int
    first_code: np.ndarray
    len_count: np.ndarray
    first_index: np.ndarray
    symbols: np.ndarray
    trie_child: np.ndarray
    trie_symbol: np.ndarray
    codes: np.ndarray  # dense canonical code per symbol value (encode side)
    lens: np.ndarray   # dense length per symbol value, 0 = absent


def lengths_array(entries: dict, symbol_width: int) -> np.ndarray:
    lens = np.zeros(1 << symbol_width, dtype=np.uint8)
    for s, (_, ln) in entries.items():
        lens[int(s)] = int(ln)
    return lens


def canonical_table(lengths: np.ndarray) -> Table:
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    fc = np.zeros(33, np.int64)
    lc = np.zeros(33, np.int64)
    fi = np.zeros(33, np.int64)
    syms = np.zeros(max(int(np.count_nonzero(lengths)), 1), np.uint16)
    codes = np.zeros(max(len(lengths), 1), np.int64)
    ml = lib().or_canonical_table(_p(lengths), len(lengths), _p(fc), _p(lc), _p(fi), _p(syms), _p(codes))
    empty = np.zeros(2, np.int32)
    return Table(0, int(ml), fc, lc, fi, syms, empty, empty, codes, lengths)


def explicit_table(entries: dict, symbol_width: int) -> Table:
    """Binary trie over explicit (code, length) pairs, restating
    codebook.py:235-260 (prefix-freeness is the caller's contract)."""
    child = [[-1, -1]]
    sym = [-1]
    for s, (code, ln) in sorted(entries.items()):
        node = 0
        for i in range(ln - 1, -1, -1):
            b = (code >> i) & 1
            if child[node][b] < 0:
                child[node][b] = len(child)
                child.append([-1, -1])
                sym.append(-1)
            node = child[node][b]
        sym[node] = int(s)
    z64 = np.zeros(33, np.int64)
    lens = lengths_array(entries, symbol_width)
    codes = np.zeros(1 << symbol_width, np.int64)
    for s, (code, _) in entries.items():
        codes[int(s)] = int(code)
    return Table(1, max(ln for _, ln in entries.values()), z64, z64, z64,
                 np.zeros(1, np.uint16), np.ascontiguousarray(child, np.int32).ravel(),
                 np.asarray(sym, np.int32), codes, lens)


def table_for(codebook) -> Table:
    if codebook.kind == "canonical":
        return canonical_table(lengths_array(codebook.entries, codebook.symbol_width))
    return explicit_table(codebook.entries, codebook.symbol_width)


class Source:
    """Keeps the numpy buffers alive behind an or_src struct."""

    def __init__(self, units: np.ndarray, unit_bits: int, table: Table):
        self.units = np.ascontiguousarray(units, dtype=np.uint32)
        self.table = table
        t = table
        self.src = _Src(
            _p(self.units) if self.units.size else None, len(self.units),
            {8: 3, 16: 4, 32: 5}[unit_bits], unit_bits, t.kind, t.max_len,
            _p(t.first_code), _p(t.len_count), _p(t.first_index), _p(t.symbols),
            _p(t.trie_child), _p(t.trie_symbol),
        )

    @property
    def ref(self):
        return C.byref(self.src)


def source_for(stream) -> Source:
    return Source(stream.units, stream.layout.unit_bits, table_for(stream.codebook))


def _nsub(stream) -> int:
    return -(-int(stream.total_bits) // stream.layout.subseq_bits)


def _nseq(stream) -> int:
    return -(-_nsub(stream) // stream.layout.subseqs_per_seq)


@dataclass
class OracleResult:
    symbols: np.ndarray
    starts: np.ndarray
    per_subseq_counts: np.ndarray


def oracle_decode(stream, src: Source | None = None) -> OracleResult:
    """kernels.py:102-122 / encoder.py:129-159."""
    src = src or source_for(stream)
    n = int(stream.symbol_count)
    out = np.empty(max(n, 1), np.uint16)
    starts = np.empty(max(n, 1), np.int64)
    ret = np.zeros(4, np.int64)
    lib().or_oracle_decode(src.ref, int(stream.total_bits), n, _p(out), _p(starts), _p(ret))
    if ret[0] != OK:
        raise OracleError(int(ret[0]), int(ret[1]))
    out, starts = out[:n], starts[:n]
    b = np.arange(_nsub(stream) + 1, dtype=np.int64) * stream.layout.subseq_bits
    return OracleResult(out, starts, np.diff(np.searchsorted(starts, b)))


@dataclass
class State:
    entry_bits: np.ndarray
    exit_bits: np.ndarray
    counts: np.ndarray
    synced: np.ndarray
    iterations: np.ndarray
    bits: int = 0
    seam_passes: int = 0


def synchronize(stream, early_exit: bool = True, src: Source | None = None) -> State:
    """sync_decoder.py:152-170 with inter_sync (:116-149)."""
    src = src or source_for(stream)
    ns, nq = _nsub(stream), _nseq(stream)
    st = State(np.zeros(ns, np.int64), np.zeros(ns, np.int64), np.zeros(ns, np.int64),
               np.zeros(ns, np.uint8), np.zeros(nq, np.int32))
    ret = np.zeros(4, np.int64)
    if ns:
        lay = stream.layout
        lib().or_synchronize(src.ref, int(stream.total_bits), lay.subseq_bits, lay.subseqs_per_seq,
                             ns, nq, int(early_exit), _p(st.entry_bits), _p(st.exit_bits),
                             _p(st.counts), _p(st.synced), _p(st.iterations), _p(ret))
        if ret[0] != OK:
            raise OracleError(int(ret[0]), int(ret[1]))
    st.bits, st.seam_passes = int(ret[2]), int(ret[3])
    st.synced = st.synced.astype(bool)
    return st


def gap_count_pass(stream, src: Source | None = None) -> tuple[State, np.ndarray]:
    """gap_decoder.py:24-68 (entries_from_gap + count_pass)."""
    src = src or source_for(stream)
    ns, nq = _nsub(stream), _nseq(stream)
    sb = stream.layout.subseq_bits
    entries = np.arange(ns, dtype=np.int64) * sb + np.asarray(stream.gap, np.int64)
    stops = np.empty(ns, np.int64)
    if ns:
        stops[:-1] = entries[1:]
        stops[-1] = int(stream.total_bits)
    st = State(entries, np.zeros(ns, np.int64), np.zeros(ns, np.int64),
               np.ones(ns, bool), np.zeros(nq, np.int32))
    ret = np.zeros(4, np.int64)
    if ns:
        lib().or_count_windows(src.ref, _p(entries), _p(stops), 0, ns, int(stream.total_bits),
                               _p(st.counts), _p(st.exit_bits), _p(ret))
        if ret[0] != OK:
            raise OracleError(int(ret[0]), int(ret[1]))
    st.bits = int(ret[2])
    return st, output_index(st.counts)


def output_index(counts) -> np.ndarray:
    """state.py:44-53."""
    counts = np.asarray(counts, np.int64)
    out = np.zeros(len(counts) + 1, np.int64)
    np.cumsum(counts, out=out[1:])
    return out


def decode_write(stream, entries, counts, oi, capacity: int, sequences=None,
                 src: Source | None = None):
    """staging.py:65-147; returns (out, stats[bits, rounds, staged, bypass])."""
    src = src or source_for(stream)
    n = int(oi[-1])
    out = np.zeros(max(n, 1), np.uint16)
    seqs = np.arange(_nseq(stream), dtype=np.int64) if sequences is None else np.asarray(sequences, np.int64)
    stats = np.zeros(4, np.int64)
    ret = np.zeros(4, np.int64)
    entries = np.ascontiguousarray(entries, np.int64)
    counts = np.ascontiguousarray(counts, np.int64)
    oi = np.ascontiguousarray(oi, np.int64)
    if len(seqs):
        lib().or_decode_write(src.ref, stream.layout.subseqs_per_seq, _nsub(stream), _p(entries),
                              _p(counts), _p(oi), _p(seqs), len(seqs), int(capacity), _p(out),
                              _p(stats), _p(ret))
        if ret[0] != OK:
            raise OracleError(int(ret[0]), int(ret[1]))
    return out[:n], stats


def encode(symbols, codebook, layout, with_gap: bool):
    """encoder.py:33-97 via kernels.py:151-179; returns (units, total_bits, gap)."""
    t = table_for(codebook)
    syms = np.ascontiguousarray(symbols, np.uint16)
    lens = t.lens
    total = int(lens[syms].sum(dtype=np.int64)) if syms.size else 0
    units = np.zeros(-(-total // layout.unit_bits), np.uint32)
    nsub = -(-total // layout.subseq_bits)
    gap = np.full(nsub if with_gap else 0, -1, np.int64)
    if with_gap and nsub:
        gap[0] = 0
    lib().or_encode_pack(_p(syms), len(syms), _p(t.codes), _p(lens), _p(units) if units.size else None,
                         {8: 3, 16: 4, 32: 5}[layout.unit_bits], layout.unit_bits,
                         layout.subseq_bits, _p(gap) if gap.size else None, len(gap))
    g = None
    if with_gap:
        idx = np.nonzero(gap < 0)[0]
        gap[idx] = total - idx * layout.subseq_bits
        g = gap.astype(np.uint8)
    return units, total, g


def tuner_plan(seq_counts, num_seqs: int, seq_bits: int, total_bits: int, symbol_width: int,
               t_high: int):
    """tuner.py:117-147 in integer arithmetic."""
    sc = np.ascontiguousarray(seq_counts, np.int64)
    classes = np.zeros(max(num_seqs, 1), np.int64)
    freq = np.zeros(t_high + 1, np.int64)
    perm = np.zeros(max(num_seqs, 1), np.int64)
    start = np.zeros(t_high + 1, np.int64)
    last_bits = total_bits - (num_seqs - 1) * seq_bits if num_seqs else seq_bits
    lib().or_tuner_plan(_p(sc), num_seqs, seq_bits, last_bits, symbol_width, t_high,
                        _p(classes), _p(freq), _p(perm), _p(start))
    return classes[:num_seqs], freq, perm[:num_seqs], start


def sequence_counts(stream, subseq_counts) -> np.ndarray:
    """tuner.py:109-114."""
    nq = _nseq(stream)
    if nq == 0:
        return np.zeros(0, np.int64)
    firsts = np.arange(nq, dtype=np.int64) * stream.layout.subseqs_per_seq
    return np.add.reduceat(np.asarray(subseq_counts, np.int64), firsts)


def gap_decode(stream, capacity: int = 3584):
    """gap_decoder.py:71-92 without the tuner: full CPU restatement."""
    src = source_for(stream)
    st, oi = gap_count_pass(stream, src)
    if int(oi[-1]) != int(stream.symbol_count):
        raise OracleError(TRUNCATED, -1)
    out, _ = decode_write(stream, st.entry_bits, st.counts, oi, capacity, src=src)
    return out


def sync_decode(stream, capacity: int = 3584):
    """sync_decoder.py:173-211 without the tuner: full CPU restatement."""
    src = source_for(stream)
    st = synchronize(stream, src=src)
    oi = output_index(st.counts)
    if int(oi[-1]) != int(stream.symbol_count):
        raise OracleError(TRUNCATED, -1)
    out, _ = decode_write(stream, st.entry_bits, st.counts, oi, capacity, src=src)
    return out


if __name__ == "__main__":  # pragma: no cover
    print(build())


def dequantize(codes, outlier_indices, outlier_values, twice_eb: float, midpoint: int) -> np.ndarray:
    """kernels.py:216-227 dequantize_chain (float32-rounded recurrence)."""
    c = np.ascontiguousarray(codes, dtype=np.uint16)
    oi = np.ascontiguousarray(outlier_indices, dtype=np.int64)
    ov = np.ascontiguousarray(outlier_values, dtype=np.float64)
    out = np.empty(c.size, dtype=np.float64)
    lib().or_dequantize(c.ctypes.data, c.size, oi.ctypes.data, ov.ctypes.data, oi.size, float(twice_eb),
                        int(midpoint), out.ctypes.data)
    return out
