"""HUF2 container -> device ingest.

The reference reads a whole container into host memory (container.py:75-135)
and its memcpy-inclusive numbers (Fig. 5) pay a full H2D
copy before decoding starts.  Here:

* ``load_container_device`` parses the header and lengths, then streams the
  gap bytes and the payload units from the file through two pinned staging
  buffers: while one buffer is being copied to the GPU (async H2D on a copy
  stream), the next file chunk is read into the other.  The returned
  EncodedStream carries its device mirror already (words, gap, K1 tables), and
  its host ``units`` are a read-only memory map of the file -- nothing is
  copied twice.
* ``decode_container`` = ingest + decode (device or host output).
* ``ingest_shard`` is the multi-GPU ingest: rank r of `world` reads only its
  contiguous span of sequences (payload bytes, gap bytes) from the file,
  decodes it as a chunk whose symbol count is not known in advance
  (bh_stream flag BH_STREAM_COUNT_IS_CAPACITY: the count comes back in the
  report), and -- with torch.distributed initialised -- gathers the 8-byte
  per-rank counts to place its output and to check the header count.  No
  rank reads another rank's bytes; the decode itself exchanges nothing.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, load, ptr, require_cuda, stream_handle
from .bitstream import EncodedStream, LayoutConfig
from .codebook import canonize
from .container import _HEAD, _U64, _UNIT, FLAG_GAP, MAGIC, VERSION
from .errors import BadGap, ContainerError, NotPresent, Truncated

CHUNK_BYTES = 64 << 20


@dataclass(frozen=True)
class ContainerInfo:
    """Header fields and section offsets of a HUF2 file (container.py:42-57)."""

    path: str
    symbol_width: int
    unit_bits: int
    units_per_subseq: int
    subseqs_per_seq: int
    symbol_count: int
    total_bits: int
    lengths: np.ndarray
    gap_off: int     # file offset of the gap bytes (-1: no gap)
    gap_count: int
    units_off: int   # file offset of the unit words
    unit_count: int

    @property
    def layout(self) -> LayoutConfig:
        return LayoutConfig(self.unit_bits, self.units_per_subseq, self.subseqs_per_seq)

    def codebook(self):
        lengths = {s: int(ln) for s, ln in enumerate(self.lengths) if ln}
        if lengths:
            return canonize(lengths, symbol_width=self.symbol_width)
        if self.symbol_count == 0:
            return canonize({0: 1}, symbol_width=self.symbol_width)
        raise ContainerError("the container has symbols but an empty codebook")


def read_info(path) -> ContainerInfo:
    """Parse the header, lengths and section offsets (no payload read)."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(_HEAD.size)
        if len(head) < _HEAD.size:
            raise ContainerError("file is shorter than the container header")
        magic, ver, width, unit_bits, flags, ups, sps, nsym, tb, alphabet = _HEAD.unpack(head)
        if magic != MAGIC:
            raise ContainerError(f"bad magic {magic!r}")
        if ver != VERSION:
            raise ContainerError(f"unsupported container version {ver}")
        if unit_bits not in _UNIT:
            raise ContainerError(f"bad unit width {unit_bits}")
        lens = np.frombuffer(f.read(alphabet), dtype=np.uint8)
        if lens.size != alphabet:
            raise ContainerError("codebook lengths are truncated")
        off = _HEAD.size + alphabet
        gap_off, ng = -1, 0
        if flags & FLAG_GAP:
            b = f.read(_U64.size)
            if len(b) < _U64.size:
                raise ContainerError("gap section is truncated")
            (ng,) = _U64.unpack(b)
            gap_off = off + _U64.size
            off = gap_off + ng
            if off > size:
                raise ContainerError("gap bytes are truncated")
            f.seek(off)
        b = f.read(_U64.size)
        if len(b) < _U64.size:
            raise ContainerError("unit section is truncated")
        (nu,) = _U64.unpack(b)
        units_off = off + _U64.size
        if units_off + nu * (unit_bits // 8) > size:
            raise ContainerError("unit words are truncated")
    return ContainerInfo(str(path), width, unit_bits, ups, sps, nsym, tb, lens.copy(), gap_off, ng, units_off, nu)


class _Stager:
    """Two pinned host buffers feeding async H2D copies on a copy stream."""

    def __init__(self, torch, dev, chunk: int):
        self.torch = torch
        self.chunk = chunk
        self.bufs = [torch.empty(chunk, dtype=torch.uint8).pin_memory() for _ in range(2)]
        self.done = [None, None]
        self.copy = torch.cuda.Stream(dev)
        self.k = 0

    def file_to_device(self, f, file_off: int, nbytes: int, dst_u8):
        """Copy file bytes [file_off, +nbytes) into the device byte tensor dst_u8.
        The copies wait for the work already queued on the caller's stream
        (dst_u8 was allocated -- and zero-filled -- there)."""
        self.copy.wait_stream(self.torch.cuda.current_stream(dst_u8.device))
        f.seek(file_off)
        pos = 0
        while pos < nbytes:
            i = self.k & 1
            if self.done[i] is not None:
                self.done[i].synchronize()  # the copy that last used this buffer has finished
            m = min(self.chunk, nbytes - pos)
            view = self.bufs[i].numpy()[:m]
            got = f.readinto(memoryview(view))
            if got != m:
                raise ContainerError("file ended inside the payload")
            with self.torch.cuda.stream(self.copy):
                dst_u8[pos:pos + m].copy_(self.bufs[i][:m], non_blocking=True)
                ev = self.torch.cuda.Event()
                ev.record(self.copy)
            self.done[i] = ev
            pos += m
            self.k += 1

    def finish(self, stream):
        stream.wait_stream(self.copy)


def _device_words(torch, lib, dev, info: ContainerInfo, stager, f, u0: int, nunits: int, stream):
    """Device MSB-first word buffer (+ BH_WORD_PAD zero words) of units [u0, u0+nunits)."""
    ub = info.unit_bits
    nbits = nunits * ub
    nwords = -(-nbits // 32)
    words = torch.zeros(nwords + _lib.WORD_PAD, dtype=torch.int32, device=dev)
    nbytes = nunits * (ub // 8)
    if ub == 32:
        stager.file_to_device(f, info.units_off + 4 * u0, nbytes, words.view(torch.uint8))
        stager.finish(stream)
        return words, nwords
    raw = torch.empty(nbytes + 4, dtype=torch.uint8, device=dev)
    stager.file_to_device(f, info.units_off + (ub // 8) * u0, nbytes, raw)
    stager.finish(stream)
    # little-endian 8/16-bit units on disk -> one u32 per unit -> MSB-first words
    dt = torch.int16 if ub == 16 else torch.uint8
    u = raw[:nbytes].view(dt).to(torch.int32) & ((1 << ub) - 1)
    check(lib.bh_repack_units(u.data_ptr(), nunits, ub, words.data_ptr(), nwords, stream_handle(stream)),
          "repack units")
    return words, nwords


def load_container_device(path, device=None, chunk_bytes: int = CHUNK_BYTES) -> EncodedStream:
    """Read a HUF2 file straight into device memory (pinned, double-buffered,
    file reads overlapped with H2D); returns the stream with its device mirror."""
    torch = require_cuda()
    lib = load()
    from .device import DeviceStream
    info = read_info(path)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    book = info.codebook()
    main = torch.cuda.current_stream(dev)
    stager = _Stager(torch, dev, chunk_bytes)
    with open(path, "rb") as f:
        gap_d = None
        if info.gap_off >= 0:
            gap_d = torch.zeros(max(info.gap_count, 1), dtype=torch.uint8, device=dev)
            stager.file_to_device(f, info.gap_off, info.gap_count, gap_d)
        words, _ = _device_words(torch, lib, dev, info, stager, f, 0, info.unit_count, main)
    units = np.memmap(path, dtype=np.dtype(_UNIT[info.unit_bits]), mode="r", offset=info.units_off,
                      shape=(info.unit_count,)) if info.unit_count else np.zeros(0, np.uint32)
    gap = None
    if info.gap_off >= 0:
        gap = np.memmap(path, dtype=np.uint8, mode="r", offset=info.gap_off, shape=(info.gap_count,)) \
            if info.gap_count else np.zeros(0, np.uint8)
    stream = EncodedStream(layout=info.layout, units=np.asarray(units, dtype=np.uint32)
                           if info.unit_bits != 32 else units, total_bits=info.total_bits,
                           symbol_count=info.symbol_count, codebook=book, gap=gap)
    ds = DeviceStream.from_device(stream, words, gap_d, dev)
    ds.ready = torch.cuda.Event()
    ds.ready.record(main)
    stream._device[str(dev)] = ds
    return stream


def decode_container(path, variant: str = "gap", device=None, device_out: bool = True, **kw):
    """Ingest a HUF2 file onto the device and decode it."""
    from . import gap_decoder, sync_decoder
    st = load_container_device(path, device)
    dec = gap_decoder if variant == "gap" else sync_decoder
    return dec.decode(st, device_out=device_out, **kw)


def ingest_shard(path, rank: int = 0, world: int = 1, variant: str = "gap", device=None, group=None):
    """Rank `rank`'s contiguous span of sequences, read from the file alone and
    decoded on this GPU.  Returns (symbols tensor, output offset, total symbols)
    -- the offset and total from the gathered per-rank counts when
    torch.distributed is initialised (else offset None, total this shard's)."""
    torch = require_cuda()
    lib = load()
    from ._pipeline import make_tune
    from .device import DeviceReport, empty
    from .shard import sequence_ranges
    info = read_info(path)
    if info.gap_off < 0:
        raise NotPresent("sharded ingest needs the container's gap array")
    lay = info.layout
    sb, sps = lay.subseq_bits, lay.subseqs_per_seq
    if (sb * sps) % 128 or (sb * sps) % info.unit_bits:
        raise ValueError("sharded ingest needs sequences of a whole number of 128-bit blocks")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream(dev)
    book = info.codebook()
    nsub = -(-info.total_bits // sb)
    nseq = -(-nsub // sps)
    q0, q1 = sequence_ranges(nseq, world)[rank]
    if q0 >= q1:  # more ranks than sequences: this rank holds nothing
        n, out0, total = 0, None, 0
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            from .shard import gather_totals, shard_offsets
            totals = gather_totals(0, group)
            out0, total = shard_offsets(totals)[rank], sum(totals)
        return torch.empty(0, dtype=torch.int16, device=dev), out0, total
    s0, s1 = q0 * sps, min(q1 * sps, nsub)
    b0 = q0 * sb * sps
    stager = _Stager(torch, dev, CHUNK_BYTES)
    with open(path, "rb") as f:
        # this span's gap bytes plus the next span's first (where this span ends)
        f.seek(info.gap_off + s0)
        g = np.frombuffer(f.read(s1 - s0 + (1 if s1 < nsub else 0)), dtype=np.uint8)
        end = info.total_bits if s1 >= nsub else min(s1 * sb + int(g[-1]), info.total_bits)
        tb = max(end - b0, 0)
        ns = -(-tb // sb) if tb else 0
        gap_d = torch.zeros(max(ns, 1), dtype=torch.uint8, device=dev)
        if ns:
            gap_d[:ns].copy_(torch.from_numpy(g[:ns].copy()).to(dev))
        u0 = b0 // info.unit_bits
        nun = min(-(-end // info.unit_bits), info.unit_count) - u0 if tb else 0
        words, _ = _device_words(torch, lib, dev, info, stager, f, u0, max(nun, 0), main)
    lens = torch.from_numpy(book.length_bytes().copy()).to(dev)
    max_codes = max(len(book.entries), 1)
    table = torch.empty(lib.bh_table_bytes(max_codes), dtype=torch.uint8, device=dev)
    check(lib.bh_table_build(lens.data_ptr(), lens.numel(), table.data_ptr(), max_codes, stream_handle(main)),
          "table")
    cap = tb // max(book.min_len, 1) + 1  # codewords starting in the span
    c = _lib.Stream(words.data_ptr(), tb, cap, sb, sps, book.symbol_width, max_codes, gap_d.data_ptr(),
                    table.data_ptr(), int(g[0]) if s0 else 0, _lib.STREAM_COUNT_IS_CAPACITY)
    from .shard import kraft_complete
    # incomplete books: the fused self-sync kernel declines them and a chunk
    # has no staged fallback -- enter through the gap bytes (same symbols)
    var = _lib.VARIANT_SYNC if variant != "gap" and kraft_complete(book) else _lib.VARIANT_GAP
    tune = make_tune(max_len=book.max_len, min_len=book.min_len)
    out = empty(cap, np.uint16, dev)
    n = 0
    if tb:
        wsb = lib.bh_workspace_bytes(C.byref(c), var, C.byref(tune))
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
        check(lib.bh_workspace_reset(ws.data_ptr(), ws.numel(), stream_handle(main)), "workspace")
        rep = DeviceReport(dev).init()
        check(lib.bh_decode_async(C.byref(c), var, C.byref(tune), out.data_ptr(), ws.data_ptr(), wsb, rep.ptr,
                                  stream_handle(main)), "shard decode")
        r = rep.read()
        check(r.status, "shard decode")
        n = int(r.total_symbols)
    out0, total = None, n
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        from .shard import gather_totals, shard_offsets
        totals = gather_totals(n, group)
        out0, total = shard_offsets(totals)[rank], sum(totals)
        if total != info.symbol_count:
            exc = BadGap if variant == "gap" else Truncated
            raise exc(f"shards decode {total} symbols; the header says {info.symbol_count}")
    elif world == 1 and n != info.symbol_count:
        raise (BadGap if variant == "gap" else Truncated)(
            f"decoded {n} symbols; the header says {info.symbol_count}")
    return out[:n], out0, total


__all__ = ["ContainerInfo", "read_info", "load_container_device", "decode_container", "ingest_shard"]
