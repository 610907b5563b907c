"""GPU: damaged streams behave exactly like the reference.

tests/golden/corrupt.npz (made by tests/golden/make_corrupt.py with the real
reference) holds small cuSZ-shaped streams with one edit each -- a gap byte
set or stepped, a payload bit flipped, a wrong symbol count -- and what the
reference's sync and gap decoders did with it: the CodecError class, or the
sha256 of the output when the damaged stream still decodes.  Both B200
decoders (fused fast path, and the reference-structured pipeline with stats)
must reproduce every outcome.
"""

import hashlib
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

Z = np.load(Path(__file__).resolve().parent / "golden" / "corrupt.npz")
KINDS = ("gap_set", "gap_step", "bit_flip", "count", "truncate")
CASES = list(range(len(Z["cases"])))


@pytest.fixture(scope="module")
def ph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    return ph


def damaged(ph, i):
    bi, kind, a, b = (int(x) for x in Z["cases"][i])
    tb, cnt, ub, ups, sps = (int(x) for x in Z[f"b{bi}_meta"])
    units = Z[f"b{bi}_units"].astype(np.uint32).copy()
    gap = Z[f"b{bi}_gap"].astype(np.uint8).copy()
    lens = Z[f"b{bi}_lens"]
    nz = np.nonzero(lens)[0]
    book = ph.canonize({int(s): int(lens[s]) for s in nz}, symbol_width=16)
    k = KINDS[kind]
    if k == "gap_set":
        gap[a] = b
    elif k == "gap_step":
        gap[a] = (int(gap[a]) + b) % 256
    elif k == "bit_flip":
        units[a // ub] ^= np.uint32(1) << np.uint32(ub - 1 - a % ub)
    elif k == "count":
        cnt = max(0, cnt + b)
    else:
        tb -= b
        units = units[: -(-tb // ub)].copy()
        if tb % ub:
            units[-1] &= np.uint32(((1 << ub) - 1) ^ ((1 << (ub - tb % ub)) - 1))
        gap = gap[: -(-tb // (ub * ups))].copy()
    return ph.EncodedStream(layout=ph.LayoutConfig(ub, ups, sps), units=units, total_bits=tb, symbol_count=cnt,
                            codebook=book, gap=gap)


def outcome(ph, fn) -> str:
    try:
        out = fn()
    except ph.CodecError as e:
        return "E:" + type(e).__name__
    return "H:" + hashlib.sha256(np.ascontiguousarray(np.asarray(out, dtype=np.uint16)).tobytes()).hexdigest()


@pytest.mark.parametrize("i", CASES)
def test_damaged_stream_matches_reference(ph, i):
    st = damaged(ph, i)
    want_sync, want_gap = str(Z["o_sync"][i]), str(Z["o_gap"][i])
    assert outcome(ph, lambda: ph.sync_decoder.decode(st)) == want_sync
    assert outcome(ph, lambda: ph.gap_decoder.decode(st)) == want_gap
    assert outcome(ph, lambda: ph.sync_decoder.decode(st, stats=ph.DecodeStats())) == want_sync
    assert outcome(ph, lambda: ph.gap_decoder.decode(st, stats=ph.DecodeStats())) == want_gap
