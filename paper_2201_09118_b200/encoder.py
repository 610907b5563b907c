"""Encoding (GPU) and the ground-truth decode API.

``encode`` keeps the reference signature (encoder.py:33-97) and produces the
same bytes: codewords concatenated MSB-first into ``unit_bits`` units, plus
the forward-skip gap array, computed by a single-pass GPU kernel (tile scan +
decoupled look-back for bit offsets, shared-memory packing, csrc/encode.cu).
``oracle_decode`` / ``mis_sync_decode`` are the reference's single-cursor
ground-truth decoders, run as one sequential GPU thread (no CPU path).
``emit_gap`` / ``signed_gaps`` are host utilities over start sets.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, load, ptr, require_cuda, stream_handle
from .bitstream import DEFAULT_LAYOUT, EncodedStream, LayoutConfig
from .codebook import Codebook, build_lengths, canonize
from .device import Workspace, d2h, device_stream, empty, h2d, zeros
from .errors import GapOverflow, InvalidCode, Truncated, UnknownSymbol


@dataclass
class OracleResult:
    symbols: np.ndarray
    starts: np.ndarray
    per_subseq_counts: np.ndarray


def _words_to_units(words: np.ndarray, total_bits: int, unit_bits: int) -> np.ndarray:
    n_units = -(-total_bits // unit_bits)
    if unit_bits == 32:
        return np.ascontiguousarray(words[:n_units], dtype=np.uint32)
    be = words.astype(">u4").view(np.uint8 if unit_bits == 8 else ">u2")
    return be[:n_units].astype(np.uint32)


def symbol_histogram_device(symbols_dev, n: int, alphabet: int = 1 << 16):
    """Device u64 counts per symbol value (K_hist, csrc/book.cu)."""
    torch = require_cuda()
    lib = load()
    dev = symbols_dev.device
    cells = max(int(alphabet), 8192)
    counts = torch.empty(cells, dtype=torch.int64, device=dev)
    src = symbols_dev
    if src.data_ptr() % 16:
        src = src.clone()
    check(lib.bh_symbol_histogram(ptr(src), int(n), int(alphabet), ptr(counts), stream_handle()), "histogram")
    return counts


def book_for_device(symbols_dev, n: int, width: int = 16) -> Codebook:
    """Canonical codebook fitted to a device array of uint16 symbols, built on
    the GPU: histogram, then Huffman lengths identical to the reference
    build_lengths (codebook.py:38-83; csrc/book.cu), then the canonical
    numbering (codebook.py:86-112).  Up to 4096 distinct symbols on the
    device; larger alphabets take the host build_lengths on the device
    histogram.  An empty input gets the reference's {0: 1} book."""
    torch = require_cuda()
    lib = load()
    if n == 0:
        return canonize({0: 1}, symbol_width=width)
    alphabet = 1 << width
    counts = symbol_histogram_device(symbols_dev, n, alphabet)
    lens = torch.empty(alphabet, dtype=torch.uint8, device=counts.device)
    status = torch.zeros(1, dtype=torch.int32, device=counts.device)
    check(lib.bh_build_lengths(ptr(counts), alphabet, ptr(lens), ptr(status), stream_handle()), "build_lengths")
    rc = int(status.item())
    if rc == _lib.BH_BAD_ARGUMENT:  # > 4096 distinct symbols: host heap on the device histogram
        c = counts[:alphabet].cpu().numpy()
        nz = np.nonzero(c)[0]
        return canonize(build_lengths({int(s): int(c[s]) for s in nz}), symbol_width=width)
    check(rc, "build_lengths")
    ln = lens.cpu().numpy()
    nz = np.nonzero(ln)[0]
    return canonize({int(s): int(ln[s]) for s in nz}, symbol_width=width)


def encode_device(symbols_dev, n: int, codebook: Codebook, layout: LayoutConfig = DEFAULT_LAYOUT,
                  with_gap: bool = False, chunk: int = 0):
    """Encode a device tensor of uint16 symbols; returns device (words, gap,
    total_bits, chunk_offsets).  ``words`` is MSB-first 32-bit words + pad."""
    torch = require_cuda()
    lib = load()
    dev = symbols_dev.device
    codes, lens = codebook.encode_arrays()
    alphabet = len(lens)
    lens_d = h2d(lens, dev)
    codes_d = h2d(codes.astype(np.uint32), dev)
    wsb = lib.bh_encode_workspace_bytes(n)
    ws = Workspace.get(wsb, dev, "encode")
    tb = _lib.U64(0)
    bad = _lib.U64(0)
    st = stream_handle()
    check(lib.bh_encode_size(ptr(symbols_dev), n, ptr(lens_d), alphabet, ptr(ws), wsb, C.byref(tb),
                             C.byref(bad), st), "encode")
    if bad.value != 2 ** 64 - 1:
        sym = int(symbols_dev[int(bad.value)].item()) & 0xFFFF
        raise UnknownSymbol(f"symbol {sym} has no codeword")
    total = int(tb.value)
    nwords = -(-total // 32)
    words = empty(nwords + _lib.WORD_PAD, np.uint32, dev)
    nsub = -(-total // layout.subseq_bits)
    gap = empty(nsub, np.uint8, dev) if with_gap else None
    offs = empty(-(-n // chunk), np.uint64, dev) if chunk else None
    rc = lib.bh_encode_pack(ptr(symbols_dev), n, ptr(codes_d), ptr(lens_d), total, layout.subseq_bits,
                            ptr(words), ptr(gap) if with_gap else None, int(chunk), ptr(offs),
                            ptr(ws), wsb, st)
    if rc == _lib.BH_GAPOVERFLOW:
        raise GapOverflow("gap entry does not fit in one byte")
    check(rc, "encode")
    return words, gap, total, offs


def encode(symbols, codebook: Codebook, layout: LayoutConfig = DEFAULT_LAYOUT,
           with_gap: bool = False) -> EncodedStream:
    """Concatenate codewords MSB-first; optionally emit the gap array."""
    torch = require_cuda()
    syms = np.ascontiguousarray(symbols, dtype=np.uint16)
    _, lens = codebook.encode_arrays()
    if syms.size and int(syms.max()) >= len(lens):
        raise UnknownSymbol(f"symbol {int(syms.max())} is outside the {codebook.symbol_width}-bit alphabet")
    dev = torch.device("cuda", torch.cuda.current_device())
    n = int(syms.size)
    sd = h2d(syms if n else np.zeros(1, np.uint16), dev)
    words, gap, total, _ = encode_device(sd, n, codebook, layout, with_gap)
    units = _words_to_units(d2h(words, np.uint32), total, layout.unit_bits)
    g = d2h(gap, np.uint8)[: -(-total // layout.subseq_bits)] if with_gap else None
    return EncodedStream(layout=layout, units=units, total_bits=total, symbol_count=n,
                         codebook=codebook, gap=g)


def _sequential(stream, start_bit: int, n: int, mode: int):
    lib = load()
    ds = device_stream(stream)
    out = empty(max(n, 1), np.uint16, ds.device)
    starts = empty(max(n, 1), np.int64, ds.device) if mode == 0 else None
    res = zeros(2, np.uint64, ds.device)
    check(lib.bh_sequential_decode(ds.ref, start_bit, n, mode, ptr(out), ptr(starts), ptr(res),
                                   stream_handle()), "sequential decode")
    status, k = (int(v) for v in d2h(res, np.uint64)[:2])
    return ds, out, starts, status, k


def oracle_decode(stream) -> OracleResult:
    """Single-cursor decode from bit 0 (encoder.py:129-159) on one GPU thread."""
    n = int(stream.symbol_count)
    ds, out, starts, status, k = _sequential(stream, 0, n, 0)
    if status == _lib.BH_INVALID:
        raise InvalidCode(f"no codeword matches the bits of symbol {k}")
    if status == _lib.BH_TRUNCATED:
        raise Truncated(f"the stream ends after {k} of {n} symbols")
    ns = stream.num_subseqs
    cnt = empty(max(ns, 1), np.int64, ds.device)
    check(load().bh_start_histogram(ptr(starts), n, stream.layout.subseq_bits, ptr(cnt), max(ns, 1),
                                    stream_handle()), "start histogram")
    return OracleResult(d2h(out, np.uint16)[:n], d2h(starts, np.int64)[:n], d2h(cnt, np.int64)[:ns])


def mis_sync_decode(stream, start_bit: int) -> np.ndarray:
    """Decode from an arbitrary bit to the end, dropping a partial tail codeword."""
    if not 0 <= start_bit < max(int(stream.total_bits), 1):
        raise ValueError(f"start bit {start_bit} is outside the stream")
    cap = max(int(stream.total_bits) - start_bit, 1)
    ds, out, _, status, k = _sequential(stream, start_bit, cap, 1)
    if status != _lib.BH_OK:
        raise InvalidCode("no codeword matches the bits")
    return d2h(out, np.uint16)[:k]


def emit_gap(starts: np.ndarray, layout: LayoutConfig, total_bits: int) -> np.ndarray:
    """Forward-skip gaps from a start set (the stream end is a virtual start)."""
    nsub = -(-total_bits // layout.subseq_bits)
    b = np.arange(nsub, dtype=np.int64) * layout.subseq_bits
    s = np.append(np.asarray(starts, dtype=np.int64), total_bits)
    g = s[np.searchsorted(s, b)] - b
    if g.size and int(g.max()) >= 256:
        raise GapOverflow("gap entry does not fit in one byte")
    return g.astype(np.uint8)


def signed_gaps(starts: np.ndarray, layout: LayoutConfig, total_bits: int) -> np.ndarray:
    """Paper convention: start of the codeword overlapping each boundary, minus the boundary."""
    nsub = -(-total_bits // layout.subseq_bits)
    b = np.arange(nsub, dtype=np.int64) * layout.subseq_bits
    s = np.asarray(starts, dtype=np.int64)
    return s[np.searchsorted(s, b, side="right") - 1] - b
