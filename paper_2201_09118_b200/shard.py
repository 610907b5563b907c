"""Multi-GPU sharding of the decode path.

Decoding shards with no collective on the data path:

* a batch of independent fields (the multi-field config) is cut into `world`
  equal contiguous spans of sequences (``balanced_pieces``: payload bits per
  sequence are constant, and decode time follows payload bits), each rank
  decoding its pieces concurrently into its own outputs (``decode_shard``);
  ``lpt_assign`` spreads whole fields instead;
* one long stream is cut at sequence boundaries, so every shard's entry bits
  are known (boundary + gap byte) and shards are independent; the only
  exchange is the per-shard symbol totals (8 bytes per rank) that place each
  shard's output, done off the timed path.

Timing over ranks is the max of the per-rank device times (``max_over_ranks``).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np


def lpt_assign(sizes, world: int) -> list[list[int]]:
    """Indices of `sizes` per rank, greedy longest-processing-time first."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(sizes)), key=lambda i: (-sizes[i], i)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + sizes[i], r))
    for lst in out:
        lst.sort()
    return out


def sequence_ranges(num_seqs: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, sequence-aligned [q0, q1) per rank (sizes differ by <= 1)."""
    base, extra = divmod(num_seqs, world)
    out, q = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((q, q + n))
        q += n
    return out


def shard_offsets(totals) -> list[int]:
    """Exclusive prefix of per-shard symbol totals (where each shard's output starts)."""
    acc, out = 0, []
    for t in totals:
        out.append(acc)
        acc += int(t)
    return out


def gather_totals(total: int, group=None) -> list[int]:
    """All ranks' symbol totals (a tiny collective, outside the timed region)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([int(total)], dtype=torch.int64, device=dev)
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return [int(p.item()) for p in parts]


def max_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


@dataclass(frozen=True)
class Chunk:
    """A sequence-aligned piece of one stream, decodable on its own.

    ``word0`` is its first 32-bit payload word, ``total_bits`` its bit span
    (it ends at the next chunk's first codeword start, so codewords belong to
    the chunk they start in, exactly like gap windows), ``sub0``/``nsub`` its
    slice of the gap array, ``first_entry`` the bit offset of its first
    codeword (the first gap byte; 0 for the stream's first chunk), ``n`` the
    symbols it decodes and ``out0`` where they go in the stream's output.
    """

    q0: int
    q1: int
    word0: int
    total_bits: int
    sub0: int
    nsub: int
    first_entry: int
    n: int
    out0: int


def _chunk(q0: int, q1: int, total_bits: int, subseq_bits: int, subseqs_per_seq: int, gap, oi) -> "Chunk":
    nsub = -(-total_bits // subseq_bits)
    seq_bits = subseq_bits * subseqs_per_seq
    s0, s1 = q0 * subseqs_per_seq, min(q1 * subseqs_per_seq, nsub)
    b0 = q0 * seq_bits
    end = total_bits if s1 >= nsub else min(s1 * subseq_bits + int(gap[s1]), total_bits)
    tb = end - b0
    ns = -(-tb // subseq_bits)
    return Chunk(q0, q1, b0 // 32, tb, s0, ns, int(gap[s0]) if s0 else 0, int(oi[s1] - oi[s0]), int(oi[s0]))


def _check_chunkable(subseq_bits: int, subseqs_per_seq: int) -> None:
    if (subseq_bits * subseqs_per_seq) % 128:
        # a chunk's payload pointer (words + word0) must stay 16-byte aligned:
        # the fused kernel stages words with 16-byte cp.async
        raise ValueError("chunking needs sequences that are a whole number of 128-bit (16-byte) blocks")


def chunk_stream(total_bits: int, subseq_bits: int, subseqs_per_seq: int, gap, subseq_counts,
                 nchunks: int) -> list[Chunk]:
    """Cut a stream into `nchunks` sequence-aligned chunks.

    `gap` is the stream's forward-skip array and `subseq_counts` the symbols
    per subsequence (the gap count pass), both recorded at encode time; they
    give every chunk's entry bit and symbol count without decoding.
    """
    _check_chunkable(subseq_bits, subseqs_per_seq)
    gap = np.asarray(gap, dtype=np.int64)
    cnt = np.asarray(subseq_counts, dtype=np.int64)
    nsub = -(-total_bits // subseq_bits)
    nseq = -(-nsub // subseqs_per_seq)
    oi = np.concatenate([[0], np.cumsum(cnt)])
    return [_chunk(q0, q1, total_bits, subseq_bits, subseqs_per_seq, gap, oi)
            for q0, q1 in sequence_ranges(nseq, max(1, min(nchunks, nseq))) if q0 < q1]


def balanced_pieces(num_seqs, world: int) -> list[list[tuple[int, int, int]]]:
    """Strong-scaling split of a batch of fields over `world` ranks.

    The fields' sequences are laid end to end and cut into `world` contiguous
    spans of equal sequence count (every sequence holds the same number of
    payload bits, and decode time follows payload bits across the batch's
    compression ratios); each span becomes at most one piece per field it
    touches.  Returns, per rank, [(field, q0, q1)] -- far fewer launches per
    rank than an LPT spread of many small chunks.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    starts = np.concatenate([[0], np.cumsum(np.asarray(num_seqs, dtype=np.int64))])
    total = int(starts[-1])
    out: list[list[tuple[int, int, int]]] = []
    for r in range(world):
        g0, g1 = total * r // world, total * (r + 1) // world
        mine = []
        for f in range(len(num_seqs)):
            lo, hi = max(g0, int(starts[f])), min(g1, int(starts[f + 1]))
            if lo < hi:
                mine.append((f, lo - int(starts[f]), hi - int(starts[f])))
        out.append(mine)
    return out


def piece_chunk(total_bits: int, subseq_bits: int, subseqs_per_seq: int, gap, subseq_counts,
                q0: int, q1: int) -> Chunk:
    """The sequence range [q0, q1) of one stream as a decodable Chunk."""
    _check_chunkable(subseq_bits, subseqs_per_seq)
    gap = np.asarray(gap, dtype=np.int64)
    oi = np.concatenate([[0], np.cumsum(np.asarray(subseq_counts, dtype=np.int64))])
    return _chunk(q0, q1, total_bits, subseq_bits, subseqs_per_seq, gap, oi)


def kraft_complete(book) -> bool:
    """Kraft sum exactly 1 (every bit pattern decodes)."""
    return sum(1 << (32 - ln) for _, ln in book.entries.values()) == 1 << 32


def decode_shard(streams, rank: int = 0, world: int = 1, variant: str = "gap", device=None):
    """Decode this rank's share of a batch of streams (BASELINE
    config 5): the batch's sequences cut into `world` equal contiguous spans
    (`balanced_pieces`), each piece a sequence-aligned chunk entered at its
    first gap byte.  The pieces run as concurrent fused decodes on one CUDA
    stream each, their CTA counts proportional to their payload, so the rank's
    whole share takes one wave of the GPU.  No collective: the result is, per
    piece, (stream index, output offset in that stream, device uint16 tensor).
    Streams need their gap arrays (every piece's entry bit and symbol count
    come from them and the encode-side count pass)."""
    import ctypes as C

    import torch

    from . import _lib
    from ._lib import check, stream_handle
    from ._pipeline import make_tune
    from .device import DeviceReport, device_stream, empty
    from .gap_decoder import count_pass, entries_from_gap
    from .errors import NotPresent
    lib = _lib.load()
    for st in streams:
        if st.gap is None:
            raise NotPresent("sharded decode needs every stream's gap array")
    spans = balanced_pieces([st.num_seqs for st in streams], world)[rank]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream(dev)
    total_bits = 0
    plan = []
    for fi, q0, q1 in spans:
        st = streams[fi]
        ds = device_stream(st, dev)
        lay = st.layout
        if q0 == 0 and q1 == st.num_seqs:
            c = _lib.Stream(ds.c.words_dev, st.total_bits, st.symbol_count, lay.subseq_bits, lay.subseqs_per_seq,
                            st.codebook.symbol_width, ds.max_codes, ds.c.gap_dev, ds.c.table_dev, 0, 0)
            n, out0, tb = st.symbol_count, 0, st.total_bits
        else:
            s = entries_from_gap(st)
            count_pass(st, s)
            ch = piece_chunk(st.total_bits, lay.subseq_bits, lay.subseqs_per_seq, st.gap, s.counts, q0, q1)
            c = _lib.Stream(ds.c.words_dev + 4 * ch.word0, ch.total_bits, ch.n, lay.subseq_bits, lay.subseqs_per_seq,
                            st.codebook.symbol_width, ds.max_codes, ds.c.gap_dev + ch.sub0, ds.c.table_dev,
                            ch.first_entry, 0)
            n, out0, tb = ch.n, ch.out0, ch.total_bits
        plan.append((fi, out0, n, tb, c, st.codebook))
        total_bits += tb
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    results, keep = [], []
    for k, (fi, out0, n, tb, c, book) in enumerate(plan):
        # the self-sync decoder's fused kernel declines incomplete books (a
        # single-symbol book) and a chunk cannot take the staged
        # pipeline: such pieces are entered through their gap bytes instead
        # (same symbols -- the synchronised state is the unique fixpoint)
        sync_ok = variant != "gap" and kraft_complete(book)
        var = _lib.VARIANT_SYNC if sync_ok else _lib.VARIANT_GAP
        if not lib.bh_fused_supported(C.byref(c), var):
            raise ValueError("sharded decode needs the fused decoder, which does not take this layout "
                             "(sequences of more than 16384 bits per tile, or forced knobs)")
        tune = make_tune(max_len=book.max_len, min_len=book.min_len)
        if len(plan) > 1:
            tune.ctas = max(1, round(sms * tb / max(total_bits, 1)))
        s = torch.cuda.Stream(dev) if k else main
        if k:
            s.wait_stream(main)
        with torch.cuda.stream(s):
            out = empty(n, np.uint16, dev)
            wsb = lib.bh_workspace_bytes(C.byref(c), var, C.byref(tune))
            ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)  # this call's scratch
            check(lib.bh_workspace_reset(ws.data_ptr(), ws.numel(), stream_handle(s)), "workspace")
            rep = DeviceReport(dev).init()
            check(lib.bh_decode_async(C.byref(c), var, C.byref(tune), out.data_ptr(), ws.data_ptr(), wsb, rep.ptr,
                                      stream_handle(s)), "shard decode")
        keep.append((s, rep, c, tune, ws))
        results.append((fi, out0, out[:n]))
    for s, rep, *_ in keep:
        main.wait_stream(s)
        with torch.cuda.stream(s):
            check(rep.read().status, "shard decode")
    return results
