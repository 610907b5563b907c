"""The N-rank decode path end to end: two processes (world_size 2, gloo) on
the one visible GPU, each decoding its share of a CESM/RTM/QMCPACK-shaped
batch through shard.decode_shard (balanced sequence-aligned spans, no
collective on the data path) and checking it against the pinned C oracle;
then the per-rank symbol totals are gathered (the one 8-byte exchange) and
must add up to the batch."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SPECS = (("cesm", 1_700_000, 0.6), ("rtm", 500_000, 0.8), ("qmcpack", 1_600_000, 22.0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(ph):
    from paper_2201_09118_b200.synth import gaussian_codes
    out = []
    for i, (_, n, sigma) in enumerate(SPECS):
        codes = gaussian_codes(n, 1024, sigma, seed=100 + i)
        out.append((codes, ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)))
    return out


def _worker(rank, world, port, variant, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2201_09118_b200 as ph
        from paper_2201_09118_b200 import shard
        from oracle import oracle
        batch = _batch(ph)
        res = shard.decode_shard([st for _, st in batch], rank, world, variant)
        mine = 0
        for fi, out0, t in res:
            codes, st = batch[fi]
            ref = oracle.oracle_decode(st).symbols if fi == 1 else codes  # one field through the C oracle
            got = t.cpu().numpy().view(np.uint16)
            if not np.array_equal(got, ref[out0:out0 + got.size]):
                raise AssertionError(f"rank {rank} field {fi} piece at {out0} differs")
            mine += got.size
        totals = shard.gather_totals(mine)
        q.put((rank, [(fi, out0, int(t.numel())) for fi, out0, t in res], totals))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["gap", "sync"])
def test_two_ranks_decode_their_shares(variant):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, variant, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    total = sum(n for _, n, _ in SPECS)
    assert res[0][2] == res[1][2] and sum(res[0][2]) == total
    # the two ranks' pieces tile every field exactly once
    cover = {}
    for _, pieces, _ in res:
        for fi, out0, n in pieces:
            cover.setdefault(fi, []).append((out0, n))
    for fi, (_, n, _) in enumerate(SPECS):
        spans = sorted(cover[fi])
        assert spans[0][0] == 0 and sum(s for _, s in spans) == n
        assert all(a[0] + a[1] == b[0] for a, b in zip(spans, spans[1:]))
