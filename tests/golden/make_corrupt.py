"""Corruption corpus: what the REAL reference does on damaged streams.

Run in the build container only (imports parhuff from /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_corrupt.py

Output (committed): tests/golden/corrupt.npz -- a few small base streams
and, per case, one edit (gap byte, payload bit flip, symbol_count or
total_bits change) plus the outcome of the reference's sync and gap
decoders: the CodecError class name, or the sha256 of the decoded output
when the damaged stream still decodes (a flipped payload bit usually just
changes symbols).  tests/test_gpu_corrupt.py replays every case through the
B200 decoders and requires the same outcome.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import parhuff as ph  # noqa: E402
from parhuff import gap_decoder, sync_decoder  # noqa: E402

KINDS = ("gap_set", "gap_step", "bit_flip", "count", "truncate")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(fn) -> str:
    try:
        out = fn()
    except ph.CodecError as e:
        return "E:" + type(e).__name__
    return "H:" + sha(np.asarray(out, dtype=np.uint16))


def bases(rng):
    """(symbols, layout) pairs: short- and long-code books, three layouts, two
    streams large enough to span many CTAs of the fused kernel."""
    out = []
    for sigma, n, lay in ((0.6, 12_000, (32, 4, 32)), (3.0, 8_000, (32, 4, 32)), (22.0, 5_000, (32, 4, 32)),
                          (3.0, 6_000, (16, 3, 5)), (8.0, 4_000, (8, 5, 7)),
                          (0.6, 1_500_000, (32, 4, 32)), (22.0, 300_000, (32, 4, 32))):
        g = np.clip(np.rint(rng.normal(0, sigma, n)) + 512, 0, 1023).astype(np.uint16)
        out.append((g, ph.LayoutConfig(*lay)))
    return out


def main():
    rng = np.random.default_rng(0xBADC0DE)
    base_list = bases(rng)
    d = {}
    cases = []
    for bi, (syms, lay) in enumerate(base_list):
        v, c = np.unique(syms, return_counts=True)
        book = ph.canonize(ph.build_lengths({int(x): int(y) for x, y in zip(v, c)}), symbol_width=16)
        st = ph.encode(syms, book, lay, with_gap=True)
        codes, lens = book.encode_arrays()
        d[f"b{bi}_units"] = st.units
        d[f"b{bi}_gap"] = st.gap
        d[f"b{bi}_lens"] = lens
        d[f"b{bi}_meta"] = np.array([st.total_bits, st.symbol_count, lay.unit_bits, lay.units_per_subseq,
                                     lay.subseqs_per_seq], np.int64)
        for k in range(60):
            kind = KINDS[k % len(KINDS)]
            units, gap = st.units.copy(), st.gap.copy()
            tb, cnt = st.total_bits, st.symbol_count
            a = b = 0
            if kind == "gap_set":
                a = int(rng.integers(len(gap)))
                b = int(rng.integers(0, 40))
                gap[a] = b
            elif kind == "gap_step":
                a = int(rng.integers(len(gap)))
                b = int(rng.choice([-3, -2, -1, 1, 2, 3]))
                gap[a] = (int(gap[a]) + b) % 256
            elif kind == "bit_flip":
                a = int(rng.integers(tb))
                ub = lay.unit_bits
                units[a // ub] ^= np.uint32(1) << np.uint32(ub - 1 - a % ub)
            elif kind == "count":
                b = int(rng.choice([-7, -1, 1, 5]))
                cnt = max(0, cnt + b)
            else:  # a stream cut short: drop the tail units, zero the bits past the new end
                b = int(rng.integers(1, 40))
                tb = tb - b
                ub = lay.unit_bits
                units = units[: -(-tb // ub)].copy()
                if tb % ub:
                    units[-1] &= np.uint32(((1 << ub) - 1) ^ ((1 << (ub - tb % ub)) - 1))
                gap = gap[: -(-tb // (lay.unit_bits * lay.units_per_subseq))].copy()
            try:
                bad = ph.EncodedStream(layout=lay, units=units, total_bits=tb, symbol_count=cnt,
                                       codebook=book, gap=gap)
            except (ValueError, ph.CodecError):
                continue
            o_sync = outcome(lambda: sync_decoder.decode(bad))
            o_gap = outcome(lambda: gap_decoder.decode(bad))
            cases.append((bi, KINDS.index(kind), a, b, o_sync, o_gap))
            print(f"base {bi} {kind:9s} a={a:6d} b={b:4d} sync={o_sync[:30]} gap={o_gap[:30]}", flush=True)
    d["cases"] = np.array([c[:4] for c in cases], np.int64)
    d["o_sync"] = np.array([c[4] for c in cases])
    d["o_gap"] = np.array([c[5] for c in cases])
    np.savez_compressed(HERE / "corrupt.npz", **d)
    print(f"{len(cases)} cases -> {HERE / 'corrupt.npz'}")


if __name__ == "__main__":
    main()
