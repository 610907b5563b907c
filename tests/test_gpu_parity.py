"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures) and the pinned C oracle.  Bit-exact throughout."""

import hashlib

import numpy as np
import pytest

from golden_cases import all_cases, case, digests

pytestmark = pytest.mark.gpu

CASES = all_cases()
GOOD = [c for c in CASES if not c.corrupt]
BAD = [c for c in CASES if c.corrupt]


@pytest.fixture(scope="module")
def ph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    return ph


def as_stream(ph, c):
    """Golden case -> the package's EncodedStream with an equivalent codebook."""
    if c.codebook.kind == "canonical":
        lens = {s: ln for s, (_, ln) in c.codebook.entries.items()}
        book = ph.canonize(lens, symbol_width=c.codebook.symbol_width)
        assert book.entries == c.codebook.entries
    else:
        book = ph.from_explicit(c.codebook.entries, symbol_width=c.codebook.symbol_width)
    lay = ph.LayoutConfig(c.layout.unit_bits, c.layout.units_per_subseq, c.layout.subseqs_per_seq)
    return ph.EncodedStream(layout=lay, units=c.units, total_bits=c.total_bits,
                            symbol_count=c.symbol_count, codebook=book, gap=c.gap)


@pytest.mark.parametrize("c", GOOD, ids=lambda c: c.name)
def test_encode_matches_reference(ph, c):
    st = as_stream(ph, c)
    enc = ph.encode(c.symbols, st.codebook, st.layout, with_gap=c.gap is not None)
    assert enc.total_bits == c.total_bits
    assert np.array_equal(enc.units, c.units)
    if c.gap is not None:
        assert np.array_equal(enc.gap, c.gap)


@pytest.mark.parametrize("c", GOOD, ids=lambda c: c.name)
def test_decoders_match_reference(ph, c):
    st = as_stream(ph, c)
    if c.gap is not None:
        assert np.array_equal(ph.gap_decoder.decode(st), c.symbols)
        assert np.array_equal(ph.gap_decoder.decode(st, stats=ph.DecodeStats()), c.symbols)
    if str(c["err_sync"]):
        with pytest.raises(getattr(ph, str(c["err_sync"]))):
            ph.sync_decoder.decode(st)
    else:
        assert np.array_equal(ph.sync_decoder.decode(st), c.symbols)
        stats = ph.DecodeStats()
        assert np.array_equal(ph.sync_decoder.decode(st, stats=stats), c.symbols)
        assert stats.phase_bits["decode_write"] == c.total_bits


@pytest.mark.parametrize("c", GOOD, ids=lambda c: c.name)
def test_sync_state_matches_reference(ph, c):
    st = as_stream(ph, c)
    if str(c["err_sync"]):
        with pytest.raises(ph.InvalidCode):
            ph.sync_decoder.synchronize(st)
        return
    s = ph.sync_decoder.synchronize(st)
    assert np.array_equal(s.entry_bits, c["sync_entries"])
    assert np.array_equal(s.exit_bits, c["sync_exits"])
    assert np.array_equal(s.counts, c["sync_counts"])
    assert np.array_equal(s.iterations, c["sync_iterations"])
    assert s.synced.all()
    intra = ph.SyncState.empty(st.num_subseqs, st.num_seqs)
    for q in range(st.num_seqs):
        ph.sync_decoder.intra_sync(st, q, state=intra)
    assert np.array_equal(intra.entry_bits, c["intra_entries"])
    assert np.array_equal(intra.counts, c["intra_counts"])
    assert np.array_equal(intra.iterations, c["intra_iterations"])
    assert np.array_equal(ph.output_index(s.counts), np.concatenate([[0], np.cumsum(c["sync_counts"])]))


@pytest.mark.parametrize("c", [c for c in GOOD if c.gap is not None], ids=lambda c: c.name)
def test_gap_count_pass_matches_reference(ph, c):
    st = as_stream(ph, c)
    s = ph.gap_decoder.entries_from_gap(st)
    assert np.array_equal(s.entry_bits, c["gap_entries"])
    stats = ph.DecodeStats()
    oi = ph.gap_decoder.count_pass(st, s, stats=stats)
    assert np.array_equal(s.counts, c["gap_counts"])
    assert np.array_equal(s.exit_bits, c["gap_exits"])
    assert np.array_equal(oi, c["gap_oi"])
    assert stats.phase_bits["count_pass"] == int(c["gap_count_bits"])


@pytest.mark.parametrize("c", [c for c in GOOD if c.has("dw_stats")], ids=lambda c: c.name)
def test_decode_write_stats_match_reference(ph, c):
    st = as_stream(ph, c)
    if c.gap is not None:
        entries, counts = c["gap_entries"], c["gap_counts"]
    else:
        entries, counts = c["sync_entries"], c["sync_counts"]
    state = ph.SyncState(entries.copy(), entries.copy(), counts.copy(),
                         np.ones(len(entries), bool), np.zeros(st.num_seqs, np.int32))
    oi = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for cap, bits, rounds, staged, bypass in c["dw_stats"]:
        stats = ph.DecodeStats()
        out = ph.decode_write(st, state, oi, capacity=int(cap), stats=stats)
        assert np.array_equal(out, c.symbols)
        assert [stats.phase_bits.get("decode_write", 0), stats.write_rounds, stats.staged_slots,
                stats.bypass_slots] == [bits, rounds, staged, bypass], f"capacity {cap}"


@pytest.mark.parametrize("c", [c for c in GOOD if c.has("plan8_class")], ids=lambda c: c.name)
def test_tuner_matches_reference(ph, c):
    st = as_stream(ph, c)
    counts = c["gap_counts"] if c.gap is not None else c["sync_counts"]
    entries = c["gap_entries"] if c.gap is not None else c["sync_entries"]
    seqc = ph.tuner.sequence_counts(st, counts)
    state = ph.SyncState(entries.copy(), entries.copy(), counts.copy(),
                         np.ones(len(entries), bool), np.zeros(st.num_seqs, np.int32))
    oi = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for th in (1, 4, 8):
        plan = ph.tuner.plan(st, seqc, ph.TunerConfig(t_high=th))
        assert np.array_equal(plan.comp_class, c[f"plan{th}_class"])
        assert np.array_equal(plan.class_freq, c[f"plan{th}_freq"])
        assert np.array_equal(plan.permutation, c[f"plan{th}_perm"])
        assert np.array_equal(plan.class_start, c[f"plan{th}_start"])
        assert np.array_equal(plan.capacity, c[f"plan{th}_cap"])
        stats = ph.DecodeStats()
        out = ph.tuner.decode_partitioned(st, plan, state, oi, stats=stats)
        assert np.array_equal(out, c.symbols)
        assert [stats.write_rounds, stats.staged_slots, stats.bypass_slots] == c[f"plan{th}_stats"].tolist()
        if c.gap is not None:
            assert np.array_equal(ph.gap_decoder.decode(st, tuner_config=ph.TunerConfig(t_high=th)), c.symbols)


@pytest.mark.parametrize("c", GOOD, ids=lambda c: c.name)
def test_oracle_api_on_device(ph, c):
    st = as_stream(ph, c)
    r = ph.oracle_decode(st)
    assert np.array_equal(r.symbols, c.symbols)
    assert np.array_equal(r.starts, c["oracle_starts"])
    assert np.array_equal(r.per_subseq_counts, c["oracle_counts"])


@pytest.mark.parametrize("c", BAD, ids=lambda c: c.name)
def test_corrupt_streams_raise_like_reference(ph, c):
    st = as_stream(ph, c)
    if str(c["err_sync"]):
        with pytest.raises(getattr(ph, str(c["err_sync"]))):
            ph.sync_decoder.decode(st)
        with pytest.raises(getattr(ph, str(c["err_sync"]))):
            ph.sync_decoder.decode(st, stats=ph.DecodeStats())
    if str(c["err_gap"]):
        with pytest.raises(getattr(ph, str(c["err_gap"]))):
            ph.gap_decoder.decode(st)
        with pytest.raises(getattr(ph, str(c["err_gap"]))):
            ph.gap_decoder.decode(st, stats=ph.DecodeStats())


def test_missing_gap_raises(ph):
    st = as_stream(ph, case("sync_text"))
    with pytest.raises(ph.NotPresent):
        ph.gap_decoder.decode(st)
    with pytest.raises(ph.NotPresent):
        ph.gap_decoder.entries_from_gap(st)


def test_mis_sync_worked_example(ph):
    st = as_stream(ph, case("sync_text"))
    assert "".join(chr(s) for s in ph.mis_sync_decode(st, 1)) == "CAABCBA"


FULL_KEYS = ("1m", "hurricane", "nyx", "nyx256", "nyx4096", "hacc", "cesm", "rtm", "qmcpack")


@pytest.mark.parametrize("key", FULL_KEYS)
def test_full_size_config_digests(ph, key):
    """Every BASELINE.json config at full size: the reference encoder's bytes
    (sha256 of lengths, units, gap written by make_golden.py --digests from the
    real parhuff), then both decoders bit-exact on the device (compared there,
    so the 562 MB HACC output never crosses PCIe)."""
    import torch
    from paper_2201_09118_b200.synth import FIELDS, field_codes
    d = digests()[key]
    codes = field_codes(FIELDS[key])
    assert codes.size == d["n"]
    assert hashlib.sha256(codes.tobytes()).hexdigest() == d["symbols"]
    book = ph.book_for(codes, 16)
    _, lens = book.encode_arrays()
    assert book.max_len == d["max_len"]
    assert hashlib.sha256(lens.tobytes()).hexdigest() == d["lengths"]
    st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    assert st.total_bits == d["total_bits"]
    assert hashlib.sha256(st.units.tobytes()).hexdigest() == d["units"]
    assert hashlib.sha256(st.gap.tobytes()).hexdigest() == d["gap"]
    want = torch.from_numpy(codes.view(np.int16)).cuda()
    for dec in (ph.gap_decoder, ph.sync_decoder):
        got = dec.decode(st, device_out=True)
        assert got.numel() == codes.size
        assert torch.equal(got, want), (key, dec.__name__)
        del got
    st._device = {}  # release the device copy before the next config


@pytest.mark.parametrize("key", ("1m", "hurricane", "hacc"))
def test_coarse_baseline_k8(ph, key):
    """K8, the in-run cuSZ-style coarse decoder (one thread per fixed-symbol
    chunk, encoder-recorded chunk offsets): bit-exact at every chunk size of
    the SURVEY §8d sweep (2^8 .. 2^14 symbols), against the codes and the
    single-cursor truth (encoder.py:129-159)."""
    import torch
    from paper_2201_09118_b200 import _lib
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty, h2d
    from paper_2201_09118_b200.encoder import encode_device
    from paper_2201_09118_b200.synth import FIELDS, field_codes
    codes = field_codes(FIELDS[key], n=min(FIELDS[key].n, 40_000_000))
    book = ph.book_for(codes, 16)
    st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    ds = device_stream(st)
    sd = h2d(codes, ds.device)
    want = torch.from_numpy(codes.view(np.int16)).cuda()
    lib = _lib.load()
    for lg in range(8, 15):
        chunk = 1 << lg
        words, _, total, offs = encode_device(sd, codes.size, book, ph.DEFAULT_LAYOUT, False, chunk)
        assert total == st.total_bits
        offs_h = offs.cpu().numpy().view(np.uint64)
        # chunk c starts at the bit where symbol c*chunk starts (oracle starts)
        lens = book.encode_arrays()[1][codes].astype(np.uint64)
        starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
        assert np.array_equal(offs_h[: -(-codes.size // chunk)], starts[::chunk])
        out = empty(codes.size, np.uint16, ds.device)
        rep = DeviceReport(ds.device).init()
        check(lib.bh_coarse_decode(ds.ref, offs.data_ptr(), chunk, out.data_ptr(), rep.ptr, stream_handle()),
              "coarse")
        check(rep.read().status, "coarse")
        assert torch.equal(out[: codes.size], want), (key, chunk)
