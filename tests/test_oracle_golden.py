"""Pin the C oracle (oracle/huff_oracle.c) to the reference's own outputs.

The fixtures in tests/golden were produced by the real parhuff package
(tests/golden/make_golden.py); the oracle is trusted as the GPU checker only
because every function here reproduces them exactly.
"""

import numpy as np
import pytest

from golden_cases import all_cases, digests

CASES = all_cases()
GOOD = [c for c in CASES if not c.corrupt]
BAD = [c for c in CASES if c.corrupt]


@pytest.mark.parametrize("c", GOOD, ids=lambda c: c.name)
def test_encode_pack_matches_reference(oracle_mod, c):
    units, total, gap = oracle_mod.encode(c.symbols, c.codebook, c.layout, with_gap=c.gap is not None)
    assert total == c.total_bits
    assert np.array_equal(units, c.units)
    if c.gap is not None:
        assert np.array_equal(gap, c.gap)


@pytest.mark.parametrize("c", GOOD, ids=lambda c: c.name)
def test_oracle_decode_matches_reference(oracle_mod, c):
    r = oracle_mod.oracle_decode(c)
    assert np.array_equal(r.symbols, c.symbols)
    assert np.array_equal(r.starts, c["oracle_starts"])
    assert np.array_equal(r.per_subseq_counts, c["oracle_counts"])


@pytest.mark.parametrize("c", GOOD, ids=lambda c: c.name)
def test_synchronize_matches_reference(oracle_mod, c):
    if str(c["err_sync"]):
        with pytest.raises(oracle_mod.OracleError):
            oracle_mod.synchronize(c)
        return
    st = oracle_mod.synchronize(c)
    assert np.array_equal(st.entry_bits, c["sync_entries"])
    assert np.array_equal(st.exit_bits, c["sync_exits"])
    assert np.array_equal(st.counts, c["sync_counts"])
    assert np.array_equal(st.iterations, c["sync_iterations"])
    slow = oracle_mod.synchronize(c, early_exit=False)
    assert np.array_equal(slow.iterations, st.iterations)


@pytest.mark.parametrize("c", [c for c in GOOD if c.gap is not None], ids=lambda c: c.name)
def test_gap_count_pass_matches_reference(oracle_mod, c):
    st, oi = oracle_mod.gap_count_pass(c)
    assert np.array_equal(st.entry_bits, c["gap_entries"])
    assert np.array_equal(st.counts, c["gap_counts"])
    assert np.array_equal(st.exit_bits, c["gap_exits"])
    assert np.array_equal(oi, c["gap_oi"])
    assert st.bits == int(c["gap_count_bits"])


@pytest.mark.parametrize("c", [c for c in GOOD if c.has("dw_stats")], ids=lambda c: c.name)
def test_decode_write_stats_match_reference(oracle_mod, c):
    if c.gap is not None:
        entries, counts = c["gap_entries"], c["gap_counts"]
    else:
        entries, counts = c["sync_entries"], c["sync_counts"]
    oi = oracle_mod.output_index(counts)
    for cap, bits, rounds, staged, bypass in c["dw_stats"]:
        out, stats = oracle_mod.decode_write(c, entries, counts, oi, int(cap))
        assert np.array_equal(out, c.symbols)
        assert stats.tolist() == [bits, rounds, staged, bypass]


@pytest.mark.parametrize("c", [c for c in GOOD if c.has("plan8_class")], ids=lambda c: c.name)
def test_tuner_plan_matches_reference(oracle_mod, c):
    counts = c["gap_counts"] if c.gap is not None else c["sync_counts"]
    seqc = oracle_mod.sequence_counts(c, counts)
    for th in (1, 4, 8):
        cls, freq, perm, start = oracle_mod.tuner_plan(seqc, c.num_seqs, c.layout.seq_bits,
                                                       c.total_bits, c.codebook.symbol_width, th)
        assert np.array_equal(cls, c[f"plan{th}_class"])
        assert np.array_equal(freq, c[f"plan{th}_freq"])
        assert np.array_equal(perm, c[f"plan{th}_perm"])
        assert np.array_equal(start, c[f"plan{th}_start"])


@pytest.mark.parametrize("c", BAD, ids=lambda c: c.name)
def test_corrupt_inputs_fail_like_reference(oracle_mod, c):
    if str(c["err_gap"]) and c.gap is not None:
        with pytest.raises(oracle_mod.OracleError):
            oracle_mod.gap_decode(c)
    if str(c["err_sync"]):
        with pytest.raises(oracle_mod.OracleError):
            oracle_mod.sync_decode(c)


def test_full_size_1m_field_digest(oracle_mod):
    """Reference encode of the 1M config regenerated here: same bytes."""
    import hashlib
    from paper_2201_09118_b200.synth import FIELDS, field_codes
    from paper_2201_09118_b200.codebook import book_for
    from paper_2201_09118_b200.bitstream import DEFAULT_LAYOUT
    dg = digests()["1m"]
    codes = field_codes(FIELDS["1m"])
    assert hashlib.sha256(codes.tobytes()).hexdigest() == dg["symbols"]
    book = book_for(codes, 16)
    units, total, gap = oracle_mod.encode(codes, book, DEFAULT_LAYOUT, True)
    assert total == dg["total_bits"]
    assert hashlib.sha256(units.tobytes()).hexdigest() == dg["units"]
    assert hashlib.sha256(gap.tobytes()).hexdigest() == dg["gap"]
