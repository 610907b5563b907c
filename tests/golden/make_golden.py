"""Generate golden fixtures by running the REAL reference package.

Run in the build container only (it imports parhuff from
/root/reference/pkg/src, which does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/cases/<name>.npz  -- stream + every reference output the tests pin
  tests/golden/quant.npz         -- reference quantize/dequantize fixtures (`--quant`)
  tests/golden/digests.json      -- sha256 digests for full-size synthetic fields
                                    (`--digests [keys]`: only these, every
                                    BASELINE config by default)

The cases mirror the reference's own tests: the Listing-1
worked streams, deep/long codes, trailing windows without a start, aligned
streams, several layouts (A4), synth/Zipf streams, the incomplete-book case
(A14), the empty stream, and corrupted headers/gaps with the exception class
the reference raises.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, REF)
sys.path.insert(0, str(REPO))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import parhuff as ph  # noqa: E402
from parhuff import gap_decoder, sync_decoder, tuner  # noqa: E402
from parhuff.staging import decode_write  # noqa: E402

from paper_2201_09118_b200.synth import FIELDS, field_codes  # noqa: E402

SYNC_BOOK = {ord("A"): "00", ord("B"): "10", ord("C"): "11", ord("D"): "010", ord("E"): "011"}
CAPS = (1, 2, 8, 1024, 3584, 8192)
T_HIGHS = (1, 4, 8)


def chars(t):
    return [ord(c) for c in t]


def zipf(rng, n, alphabet):
    w = 1.0 / np.arange(1, alphabet + 1, dtype=np.float64)
    w /= w.sum()
    return rng.choice(alphabet, size=n, p=w).astype(np.uint16)


def book_for(symbols, width):
    symbols = np.asarray(symbols)
    if symbols.size == 0:
        return ph.canonize({0: 1}, symbol_width=width)
    v, c = np.unique(symbols, return_counts=True)
    return ph.canonize(ph.build_lengths({int(a): int(b) for a, b in zip(v, c)}), symbol_width=width)


def geometric_book(levels, width=16):
    lengths = {i: i + 1 for i in range(levels - 1)}
    lengths[levels - 1] = levels - 1
    return ph.canonize(lengths, symbol_width=width)


def explicit_book():
    return ph.from_explicit(ph.codes_from_strings(SYNC_BOOK))


def _exc_name(fn):
    try:
        fn()
    except ph.CodecError as e:
        return type(e).__name__
    return ""


def record(name, symbols, book, layout, with_gap=True, out=None, header_delta=0, gap_edit=None):
    symbols = np.asarray(symbols, dtype=np.uint16)
    stream = ph.encode(symbols, book, layout, with_gap=with_gap)
    d = {}
    d["symbols_in"] = symbols
    d["unit_bits"] = layout.unit_bits
    d["ups"] = layout.units_per_subseq
    d["sps"] = layout.subseqs_per_seq
    d["symbol_width"] = book.symbol_width
    d["kind"] = 0 if book.kind == "canonical" else 1
    codes, lens = book.encode_arrays()
    d["codes"] = codes
    d["lens"] = lens
    d["units"] = stream.units
    d["total_bits"] = stream.total_bits
    d["symbol_count"] = stream.symbol_count
    d["has_gap"] = int(stream.gap is not None)
    d["gap"] = stream.gap if stream.gap is not None else np.zeros(0, np.uint8)
    if header_delta or gap_edit is not None:
        gap = stream.gap.copy() if stream.gap is not None else None
        if gap_edit is not None:
            gap_edit(gap)
        bad = ph.EncodedStream(layout=layout, units=stream.units, total_bits=stream.total_bits,
                               symbol_count=stream.symbol_count + header_delta,
                               codebook=book, gap=gap)
        d["symbol_count"] = bad.symbol_count
        d["gap"] = bad.gap if bad.gap is not None else np.zeros(0, np.uint8)
        d["err_sync"] = _exc_name(lambda: sync_decoder.decode(bad))
        d["err_gap"] = _exc_name(lambda: gap_decoder.decode(bad)) if bad.gap is not None else "NotPresent"
        d["err_oracle"] = _exc_name(lambda: ph.oracle_decode(bad))
        np.savez_compressed(out / f"{name}.npz", **d)
        return
    orc = ph.oracle_decode(stream)
    assert np.array_equal(orc.symbols, symbols)
    d["oracle_starts"] = orc.starts
    d["oracle_counts"] = orc.per_subseq_counts
    err_sync = _exc_name(lambda: sync_decoder.synchronize(stream))
    d["err_sync"] = err_sync
    d["err_gap"] = "" if stream.gap is not None else "NotPresent"
    if not err_sync:
        st = sync_decoder.synchronize(stream)
        slow = sync_decoder.synchronize(stream, early_exit=False)
        assert np.array_equal(slow.iterations, st.iterations)
        d["sync_entries"] = st.entry_bits
        d["sync_exits"] = st.exit_bits
        d["sync_counts"] = st.counts
        d["sync_iterations"] = st.iterations
        stats = ph.DecodeStats()
        sync_decoder.decode(stream, stats=stats)
        d["sync_phase_bits"] = np.array([stats.phase_bits.get("sync", 0),
                                         stats.phase_bits.get("decode_write", 0)], np.int64)
        # intra-only state (before seam passes) for the intra_sync sub-step
        intra = ph.SyncState.empty(stream.num_subseqs, stream.num_seqs)
        for s in range(stream.num_seqs):
            sync_decoder.intra_sync(stream, s, state=intra)
        d["intra_entries"] = intra.entry_bits
        d["intra_exits"] = intra.exit_bits
        d["intra_counts"] = intra.counts
        d["intra_iterations"] = intra.iterations
    if stream.gap is not None:
        gst = gap_decoder.entries_from_gap(stream)
        gstats = ph.DecodeStats()
        oi = gap_decoder.count_pass(stream, gst, stats=gstats)
        d["gap_entries"] = gst.entry_bits
        d["gap_exits"] = gst.exit_bits
        d["gap_counts"] = gst.counts
        d["gap_oi"] = oi
        d["gap_count_bits"] = gstats.phase_bits.get("count_pass", 0)
        assert np.array_equal(gap_decoder.decode(stream), symbols)
    base = gst if stream.gap is not None else (st if not err_sync else None)
    if base is not None:
        oi = ph.output_index(base.counts)
        rows = []
        for cap in CAPS:
            s2 = ph.DecodeStats()
            o = decode_write(stream, base, oi, capacity=cap, stats=s2)
            assert np.array_equal(o, symbols)
            rows.append([cap, s2.phase_bits.get("decode_write", 0), s2.write_rounds,
                         s2.staged_slots, s2.bypass_slots])
        d["dw_stats"] = np.array(rows, np.int64)
        seqc = tuner.sequence_counts(stream, base.counts)
        for th in T_HIGHS:
            plan = tuner.plan(stream, seqc, ph.TunerConfig(t_high=th))
            d[f"plan{th}_class"] = plan.comp_class
            d[f"plan{th}_freq"] = plan.class_freq
            d[f"plan{th}_perm"] = plan.permutation
            d[f"plan{th}_start"] = plan.class_start
            d[f"plan{th}_cap"] = plan.capacity
            st3 = ph.DecodeStats()
            o = tuner.decode_partitioned(stream, plan, base, oi, stats=st3)
            assert np.array_equal(o, symbols)
            d[f"plan{th}_stats"] = np.array([st3.write_rounds, st3.staged_slots, st3.bypass_slots],
                                            np.int64)
    np.savez_compressed(out / f"{name}.npz", **d)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = HERE / "cases"
    out.mkdir(parents=True, exist_ok=True)
    byte = ph.LayoutConfig(8, 1, 32)
    rng = np.random.default_rng(20240)

    record("worked", chars("BACACCBDBAAEBBA"), explicit_book(), byte, out=out)
    record("sync_text", chars("CBADCBA"), explicit_book(), byte, with_gap=False, out=out)
    record("worked_2seq", chars("BACACCBDBAAEBBA"), explicit_book(), ph.LayoutConfig(8, 1, 2), out=out)
    record("worked_16", chars("BACACCBDBAAEBBA"), explicit_book(), ph.LayoutConfig(16, 1, 4), out=out)

    r1 = np.random.default_rng(1)
    w = np.array([2.0 ** -(i + 1) for i in range(31)] + [2.0 ** -31])
    deep = r1.choice(32, size=4000, p=w / w.sum()).astype(np.uint16)
    deep[:64] = 31
    record("deep31", deep, geometric_book(32), ph.DEFAULT_LAYOUT, out=out)
    r2 = np.random.default_rng(2)
    record("deep15_8bit", r2.integers(10, 16, size=300).astype(np.uint16), geometric_book(16),
           ph.LayoutConfig(8, 1, 4), out=out)
    record("trailing", np.array([0] * 7 + [9], np.uint16), geometric_book(10, width=8),
           ph.LayoutConfig(8, 1, 8), out=out)
    al = np.tile(np.arange(16, dtype=np.uint16), 64)
    record("aligned", al, book_for(al, 8), byte, out=out)
    al2 = np.tile(np.arange(16, dtype=np.uint16), 128)
    record("aligned_128", al2, book_for(al2, 8), ph.DEFAULT_LAYOUT, out=out)
    st = np.tile(np.arange(16, dtype=np.uint16), 32)
    record("straddle", st, book_for(st, 8), ph.LayoutConfig(8, 2, 32), out=out)
    bs = np.zeros(400, dtype=np.uint16)
    bs[1::2] = np.arange(200) % 5
    record("seam_split", bs, book_for(bs, 8), ph.LayoutConfig(8, 2, 8), out=out)
    one = np.zeros(100, np.uint16)
    record("single_symbol", one, book_for(one, 16), ph.DEFAULT_LAYOUT, out=out)
    record("empty", np.zeros(0, np.uint16), book_for([], 16), ph.DEFAULT_LAYOUT, out=out)
    record("one_symbol_stream", np.array([7], np.uint16), book_for([7, 7, 3], 16), ph.DEFAULT_LAYOUT, out=out)
    record("three", np.array([7, 7, 3], np.uint16), book_for([7, 7, 3], 16), ph.DEFAULT_LAYOUT, out=out)

    layouts = [(16, 3, 5), (8, 5, 7), (32, 3, 33), (32, 4, 32), (8, 1, 32), (16, 1, 4),
               (32, 1, 64), (32, 8, 16), (8, 3, 3), (32, 2, 1)]
    for i, (ub, ups, sps) in enumerate(layouts):
        for width in (8, 16):
            alphabet = int(rng.integers(2, 250 if width == 8 else 3000))
            n = int(rng.integers(2000, 16000))
            syms = zipf(rng, n, alphabet)
            record(f"zipf_{ub}_{ups}_{sps}_w{width}", syms, book_for(syms, width),
                   ph.LayoutConfig(ub, ups, sps), out=out)
    for sharp in (0.3, 0.45, 0.75, 0.9, 0.98, 0.999):
        codes = ph.synth_codes(12000, sharp, seed=int(rng.integers(2 ** 31)))
        dev = codes.astype(np.int64) - 32768
        codes = (32768 + np.clip(dev, -2048, 2047)).astype(np.uint16)
        record(f"synth_{sharp}", codes, book_for(codes, 16), ph.DEFAULT_LAYOUT, out=out)
    two = np.concatenate([ph.synth_codes(20000, 0.45, seed=1), ph.synth_codes(20000, 0.999, seed=2)])
    record("two_regime", two, book_for(two, 16), ph.DEFAULT_LAYOUT, out=out)
    g = field_codes(FIELDS["1m"], n=100_000)
    record("gauss_1m_head", g, book_for(g, 16), ph.DEFAULT_LAYOUT, out=out)
    g2 = field_codes(FIELDS["hacc"], n=60_000)
    record("gauss_hacc_head", g2, book_for(g2, 16), ph.DEFAULT_LAYOUT, out=out)
    # A14: incomplete canonical book -- sync raises on valid streams
    inc = ph.canonize({0: 1, 1: 3, 2: 3}, symbol_width=8)
    record("incomplete_book", np.random.default_rng(5).choice(3, size=500).astype(np.uint16),
           inc, ph.LayoutConfig(8, 1, 32), out=out)
    # corrupted inputs
    cz = zipf(np.random.default_rng(9), 800, 30)
    record("bad_header", cz, book_for(cz, 16), ph.DEFAULT_LAYOUT, with_gap=False, out=out, header_delta=5)
    cg = zipf(np.random.default_rng(6), 3000, 40)

    def edit(gap):
        gap[1] = (gap[1] + 1) % 17
    record("bad_gap", cg, book_for(cg, 16), ph.DEFAULT_LAYOUT, out=out, gap_edit=edit)
    record("bad_header_gap", cg, book_for(cg, 16), ph.DEFAULT_LAYOUT, out=out, header_delta=-3)

    # HUF2 containers written by the reference (byte-compatibility fixtures)
    cdir = HERE / "containers"
    cdir.mkdir(exist_ok=True)
    for name in ("zipf_16_3_5_w8", "zipf_32_4_32_w16", "gauss_1m_head", "empty", "single_symbol",
                 "trailing", "deep31", "zipf_8_1_32_w8"):
        z = np.load(out / f"{name}.npz")
        lens = z["lens"]
        nz = np.nonzero(lens)[0]
        book = ph.canonize({int(s): int(lens[s]) for s in nz}, symbol_width=int(z["symbol_width"]))
        lay = ph.LayoutConfig(int(z["unit_bits"]), int(z["ups"]), int(z["sps"]))
        st = ph.EncodedStream(layout=lay, units=z["units"].astype(np.uint32), total_bits=int(z["total_bits"]),
                              symbol_count=int(z["symbol_count"]), codebook=book,
                              gap=z["gap"] if int(z["has_gap"]) else None)
        ph.write_container(st, cdir / f"{name}.huf2")

    make_digests(("1m", "hurricane"))


# every BASELINE.json config (SURVEY §8d shapes): the reference encoder's bytes
DIGEST_KEYS = ("1m", "hurricane", "nyx", "nyx256", "nyx4096", "hacc", "cesm", "rtm", "qmcpack")


def make_digests(keys=DIGEST_KEYS):
    """sha256 of the reference encoder's output (lengths, units, gap) and of the
    symbols for full-size synthetic fields; the reference gap decoder checks
    each stream round-trips.  Existing entries for other keys are kept."""
    path = HERE / "digests.json"
    digests = json.loads(path.read_text()) if path.exists() else {}
    for key in keys:
        spec = FIELDS[key]
        codes = field_codes(spec)
        book = book_for(codes, 16)
        stream = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
        _, lens = book.encode_arrays()
        dec = gap_decoder.decode(stream, workers=os.cpu_count() or 8)
        assert np.array_equal(dec, codes)
        digests[key] = {
            "n": spec.n, "total_bits": int(stream.total_bits), "max_len": int(book.max_len),
            "lengths": sha(lens), "units": sha(stream.units), "gap": sha(stream.gap),
            "symbols": sha(codes),
        }
        print(key, digests[key], flush=True)
        del codes, stream, dec
        path.write_text(json.dumps(digests, indent=1) + "\n")

def make_quant():
    """Reconstruction fixtures (quant.py:50-74, kernels.py:181-227): the real
    reference quantizes synthetic fields and dequantizes them; the decoded
    codes, outlier sidecar and float64 reconstruction are kept."""
    rng = np.random.default_rng(77)
    cases = {}

    def rec(name, data, eb, width=16):
        cfg = ph.QuantConfig(error_bound=eb, symbol_width=width)
        q = ph.quantize(data, cfg)
        out = ph.dequantize(q, cfg)
        cases[name] = dict(codes=q.codes, oidx=q.outlier_indices, oval=q.outlier_values, eb=np.float64(eb),
                           width=np.int64(width), expect=out)
        print(name, "n", len(data), "outliers", len(q.outlier_indices))

    walk = np.cumsum(rng.normal(0, 0.01, 60_000))
    rec("walk_pow2", walk, 2.0 ** -9)                      # exact regime, no outliers
    jumps = walk.copy()
    jumps[rng.choice(len(jumps), 40, replace=False)] += rng.normal(0, 500, 40)
    rec("jumps_pow2", jumps, 2.0 ** -9)                    # outliers with arbitrary values
    rec("walk_1e-3", walk, 1e-3)                           # 2eb not a power of two
    rec("walk_w8", np.cumsum(rng.normal(0, 0.002, 30_000)), 2.0 ** -10, width=8)
    ramp = np.arange(200_000, dtype=np.float64) * (2.0 ** -6) * 120.0  # running sums pass 2^24 units
    rec("ramp_pow2", ramp, 2.0 ** -7)
    sine = np.sin(np.arange(80_000) / 300.0) * 3.0
    rec("sine_pow2_small_eb", sine, 2.0 ** -20)
    np.savez_compressed(HERE / "quant.npz", **{f"{k}__{f}": v for k, d in cases.items() for f, v in d.items()})


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--digests":
        make_digests(tuple(sys.argv[2:]) or DIGEST_KEYS)
    elif len(sys.argv) > 1 and sys.argv[1] == "--quant":
        make_quant()
    else:
        main()
