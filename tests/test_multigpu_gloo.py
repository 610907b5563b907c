"""Multi-process (world_size 2, gloo on CPU) coverage of the N>1 host path:
field assignment, sequence ranges, per-shard output offsets from gathered
totals and max-over-ranks timing -- the only exchanges sharding needs."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2201_09118_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sizes, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        assign = shard.lpt_assign(sizes, world)
        mine = assign[rank]
        total = sum(sizes[i] for i in mine)               # stands in for decoded symbols
        totals = shard.gather_totals(total)
        offs = shard.shard_offsets(totals)
        t = shard.max_over_ranks(1.0 + rank)
        q.put((rank, assign, totals, offs, t))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    sizes = [170, 34, 129, 11, 95, 95, 40, 300]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sizes, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, t0, o0, m0), (r1, a1, t1, o1, m1) = res
    assert a0 == a1 and sorted(a0[0] + a0[1]) == list(range(len(sizes)))
    assert t0 == t1 and sum(t0) == sum(sizes)
    assert o0 == o1 == [0, t0[0]]
    assert m0 == m1 == 2.0


def test_sequence_ranges_cover_stream():
    for nseq in (0, 1, 7, 9958, 349_500):
        for world in (1, 2, 4, 8):
            rs = shard.sequence_ranges(nseq, world)
            assert rs[0][0] == 0 and rs[-1][1] == nseq
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def _pieces_worker(rank, world, port, nseqs, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard.balanced_pieces(nseqs, world)[rank]
        totals = shard.gather_totals(sum(q1 - q0 for _, q0, q1 in mine))
        q.put((rank, mine, totals))
    finally:
        dist.destroy_process_group()


def test_two_rank_balanced_pieces_gloo():
    """Strong-scaling split of a batch (BASELINE config 5) over 2 ranks: every
    sequence of every field on exactly one rank, equal shares (+-1)."""
    nseqs = [67_123, 22_240, 251_255]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pieces_worker, args=(r, world, port, nseqs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    totals = res[0][2]
    assert res[1][2] == totals and sum(totals) == sum(nseqs) and abs(totals[0] - totals[1]) <= 1
    seen = {f: [] for f in range(len(nseqs))}
    for _, mine, _ in res:
        for f, q0, q1 in mine:
            seen[f].append((q0, q1))
    for f, n in enumerate(nseqs):
        spans = sorted(seen[f])
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_balanced_pieces_many_worlds():
    nseqs = [5, 0, 17, 3]
    for world in (1, 2, 3, 4, 8, 30):
        parts = shard.balanced_pieces(nseqs, world)
        assert len(parts) == world
        assert sum(q1 - q0 for p in parts for _, q0, q1 in p) == sum(nseqs)
        sizes = [sum(q1 - q0 for _, q0, q1 in p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
