"""Device mirror of an EncodedStream, and small host<->device helpers.

A ``DeviceStream`` owns the stream's device buffers (torch tensors used purely
as allocations): the payload as MSB-first 32-bit words plus BH_WORD_PAD zero
words, the gap bytes, and the decode-table blob built on the GPU by K1
(csrc/table.cu).  It is cached on the EncodedStream per device, so repeated
decodes of one stream upload nothing.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from ._lib import check, load, ptr, require_cuda, stream_handle


def h2d(arr: np.ndarray, device, pinned: bool = False):
    """numpy -> device tensor (uint16/uint32 travel as int16/int32 views)."""
    torch = require_cuda()
    a = np.ascontiguousarray(arr)
    if not a.flags.writeable:
        a = a.copy()
    view = {np.dtype(np.uint16): np.int16, np.dtype(np.uint32): np.int32,
            np.dtype(np.uint64): np.int64}.get(a.dtype)
    if view is not None:
        a = a.view(view)
    t = torch.from_numpy(a)
    if pinned:
        t = t.pin_memory()
    return t.to(device, non_blocking=pinned)


def d2h(t, dtype) -> np.ndarray:
    a = t.cpu().numpy()
    return a.view(dtype) if a.dtype != np.dtype(dtype) else a


def empty(n: int, dtype, device):
    torch = require_cuda()
    tdt = {np.uint8: torch.uint8, np.int64: torch.int64, np.int32: torch.int32,
           np.uint16: torch.int16, np.uint32: torch.int32, np.uint64: torch.int64}[dtype]
    return torch.empty(max(int(n), 1), dtype=tdt, device=device)


def zeros(n: int, dtype, device):
    t = empty(n, dtype, device)
    t.zero_()
    return t


class Workspace:
    """Grow-only device scratch, one buffer per (device, CUDA stream, tag).

    The C ABI is safe per (workspace, stream) pair (include/b200huff.h): calls
    on one stream are ordered, so they may share a workspace; calls on
    different streams -- e.g. two host threads, each on its own stream -- get
    different buffers.  The reference decoders are safe for concurrent callers
    (staging.py:48-62), and so is this mirror.  The map is guarded by a lock;
    a buffer that grows is replaced, and the old one stays alive until the
    work already queued on its stream has finished with it (torch's caching
    allocator orders its reuse on that stream)."""

    _bufs: dict = {}
    _lock = threading.Lock()

    @classmethod
    def get(cls, nbytes: int, device, tag: str = "main"):
        torch = require_cuda()
        dev = torch.device(device)
        st = torch.cuda.current_stream(dev)
        key = (str(dev), st.cuda_stream, tag)
        with cls._lock:
            buf = cls._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.empty(max(int(nbytes), 256) + 256, dtype=torch.uint8, device=dev)
                # fused-kernel descriptors are epoch-tagged: zero once per allocation
                check(load().bh_workspace_reset(buf.data_ptr(), buf.numel(), stream_handle(st)), "workspace")
                cls._bufs[key] = buf
            return buf


class DeviceStream:
    """Device buffers of one stream plus the ``bh_stream`` struct that names them."""

    def __init__(self, stream, device=None, pinned: bool = False):
        torch = require_cuda()
        lib = load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream
        lay = stream.layout
        tb = int(stream.total_bits)
        nwords = -(-tb // 32)
        st = stream_handle()
        self.words = zeros(nwords + _lib.WORD_PAD, np.uint32, self.device)
        if len(stream.units):
            if lay.unit_bits == 32:
                self.words[:nwords].copy_(h2d(stream.units, self.device, pinned))
            else:
                units = h2d(stream.units, self.device, pinned)
                check(lib.bh_repack_units(ptr(units), len(stream.units), lay.unit_bits,
                                          ptr(self.words), nwords, st), "repack units")
        self.gap = None
        if stream.gap is not None:
            g = stream.gap if len(stream.gap) else np.zeros(1, np.uint8)
            self.gap = h2d(g, self.device, pinned)
        book = stream.codebook
        self.max_codes = max(len(book.entries), 1)
        self.table = empty(lib.bh_table_bytes(self.max_codes), np.uint8, self.device)
        if book.kind == "canonical":
            lens = book.length_bytes()
            lt = h2d(lens if lens.size else np.zeros(1, np.uint8), self.device)
            check(lib.bh_table_build(ptr(lt), len(lens), ptr(self.table), self.max_codes, st), "table")
        else:
            codes, lens = book.encode_arrays()
            alphabet = max(book.entries) + 1 if book.entries else 1
            ct = h2d(codes[:alphabet].astype(np.uint32), self.device)
            lt = h2d(lens[:alphabet], self.device)
            check(lib.bh_table_build_explicit(ptr(ct), ptr(lt), alphabet, ptr(self.table),
                                              self.max_codes, st), "table")
            self._keep = (ct, lt)
        self.c = _lib.Stream(ptr(self.words), tb, int(stream.symbol_count), lay.subseq_bits,
                             lay.subseqs_per_seq, book.symbol_width, self.max_codes,
                             ptr(self.gap), ptr(self.table))

    @classmethod
    def from_device(cls, stream, words, gap, device) -> "DeviceStream":
        """Mirror over device buffers that already hold the payload words (+ pad)
        and gap bytes (container ingest); builds the K1 tables."""
        lib = load()
        ds = cls.__new__(cls)
        ds.device = device
        ds.stream = stream
        ds.words = words
        ds.gap = gap
        book = stream.codebook
        lay = stream.layout
        ds.max_codes = max(len(book.entries), 1)
        ds.table = empty(lib.bh_table_bytes(ds.max_codes), np.uint8, device)
        lens = book.length_bytes()
        ds._lens = h2d(lens if lens.size else np.zeros(1, np.uint8), device)
        check(lib.bh_table_build(ptr(ds._lens), len(lens), ptr(ds.table), ds.max_codes, stream_handle()), "table")
        ds.c = _lib.Stream(ptr(words), int(stream.total_bits), int(stream.symbol_count), lay.subseq_bits,
                           lay.subseqs_per_seq, book.symbol_width, ds.max_codes, ptr(gap), ptr(ds.table))
        return ds

    @property
    def ref(self):
        return C.byref(self.c)

    @property
    def num_subseqs(self) -> int:
        return self.stream.num_subseqs

    @property
    def num_seqs(self) -> int:
        return self.stream.num_seqs


_ds_lock = threading.Lock()


def device_stream(stream, device=None) -> DeviceStream:
    """The stream's device mirror on `device`, built once and cached on the
    EncodedStream.  Its uploads and table build are queued on the stream that
    built it; a caller on another CUDA stream waits for them (an event)."""
    torch = require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    cache = getattr(stream, "_device", None)
    key = str(dev)
    with _ds_lock:
        ds = cache.get(key) if isinstance(cache, dict) else None
        if ds is None:
            ds = DeviceStream(stream, dev)
            ds.ready = torch.cuda.Event()
            ds.ready.record(torch.cuda.current_stream(dev))
            if isinstance(cache, dict):
                cache[key] = ds
    torch.cuda.current_stream(dev).wait_event(ds.ready)
    return ds


class DeviceReport:
    """Device-side report buffer (bh_report_bytes) with a host reader."""

    def __init__(self, device):
        self.buf = empty(load().bh_report_bytes(), np.uint8, device)

    @property
    def ptr(self) -> int:
        return ptr(self.buf)

    def init(self):
        check(load().bh_report_init(self.ptr, stream_handle()), "report init")
        return self

    def read(self) -> _lib.Report:
        r = _lib.Report()
        check(load().bh_report_read(self.ptr, C.byref(r), stream_handle()), "report read")
        return r
