"""Host-side logic on the CPU: codebook construction, container bytes,
layout/bitstream utilities and the tuner's scalar helpers, each against the
reference's behaviour (golden fixtures written by the real reference)."""

import numpy as np
import pytest

import paper_2201_09118_b200 as ph
from paper_2201_09118_b200 import tuner
from golden_cases import CASES_DIR, GOLDEN, all_cases

GOOD = [c for c in all_cases() if not c.corrupt]


@pytest.mark.parametrize("c", [c for c in GOOD if c.codebook.kind == "canonical"], ids=lambda c: c.name)
def test_canonize_matches_reference_entries(c):
    lens = {s: ln for s, (_, ln) in c.codebook.entries.items()}
    book = ph.canonize(lens, symbol_width=c.codebook.symbol_width)
    assert book.entries == c.codebook.entries


@pytest.mark.parametrize("c", [c for c in GOOD if c.codebook.kind == "canonical" and c.symbol_count > 1
                               and c.name.startswith(("zipf", "synth", "gauss", "two", "aligned"))],
                         ids=lambda c: c.name)
def test_build_lengths_reproduces_reference_book(c):
    counts = np.bincount(c.symbols.astype(np.int64))
    lens = ph.build_lengths({int(s): int(counts[s]) for s in np.nonzero(counts)[0]})
    assert lens == {s: ln for s, (_, ln) in c.codebook.entries.items()}


def test_build_lengths_edge_rules():
    assert ph.build_lengths({5: 9}) == {5: 1}
    with pytest.raises(ph.EmptyInput):
        ph.build_lengths({1: 0})
    with pytest.raises(ph.KraftViolation):
        ph.canonize({0: 1, 1: 1, 2: 1})
    with pytest.raises(ph.LengthOverflow):
        ph.canonize({0: 33})
    # Listing-1 style canonical numbering (test_codebook.py:82-86)
    book = ph.canonize({0: 2, 1: 2, 2: 2, 3: 3, 4: 3})
    assert {s: format(c, f"0{l}b") for s, (c, l) in book.entries.items()} == \
        {0: "00", 1: "01", 2: "10", 3: "110", 4: "111"}


def test_explicit_prefix_violation():
    with pytest.raises(ph.NotPrefixFree):
        ph.from_explicit(ph.codes_from_strings({1: "0", 2: "01"}))


@pytest.mark.parametrize("path", sorted((GOLDEN / "containers").glob("*.huf2")), ids=lambda p: p.stem)
def test_container_bytes_match_reference(tmp_path, path):
    st = ph.read_container(path)
    from golden_cases import case
    c = case(path.stem)
    assert st.total_bits == c.total_bits and st.symbol_count == c.symbol_count
    assert np.array_equal(st.units, c.units)
    if c.symbol_count:
        assert st.codebook.entries == c.codebook.entries
    out = tmp_path / "x.huf2"
    ph.write_container(st, out)
    assert out.read_bytes() == path.read_bytes()


def test_container_corruption(tmp_path):
    src = sorted((GOLDEN / "containers").glob("zipf*.huf2"))[0].read_bytes()
    bad = bytearray(src)
    bad[0] ^= 0xFF
    (tmp_path / "m").write_bytes(bytes(bad))
    with pytest.raises(ph.ContainerError):
        ph.read_container(tmp_path / "m")
    bad = bytearray(src)
    bad[4] = 9
    (tmp_path / "v").write_bytes(bytes(bad))
    with pytest.raises(ph.ContainerError):
        ph.read_container(tmp_path / "v")
    (tmp_path / "t").write_bytes(src[:-3])
    with pytest.raises(ph.ContainerError):
        ph.read_container(tmp_path / "t")


def test_layout_and_bit_reads():
    assert ph.DEFAULT_LAYOUT.subseq_bits == 128 and ph.DEFAULT_LAYOUT.seq_bits == 4096
    with pytest.raises(ValueError):
        ph.LayoutConfig(unit_bits=12)
    from golden_cases import case
    c = case("worked")
    st = ph.EncodedStream(layout=ph.LayoutConfig(8, 1, 32), units=c.units, total_bits=c.total_bits,
                          symbol_count=c.symbol_count, codebook=ph.canonize({0: 1}), gap=c.gap)
    assert st.read_bits(0, 2) == 0b10 and st.read_bits(14, 3) == 0b010
    with pytest.raises(ph.OutOfRange):
        st.read_bits(st.storage_bits + 1, 1)
    # the 32-bit word view used on the device is the same bit sequence
    w = st.words32()
    assert int(w[0]) == 0x8CF940E8
    bw = ph.BitWriter(8)
    bw.write(0b101, 3)
    bw.write(0b11111, 5)
    bw.write(1, 1)
    assert bw.getvalue().tolist() == [0b10111111, 0b10000000] and bw.bit_length == 9


def test_tuner_scalar_helpers():
    assert tuner.classify(3.86, 8) == 4 and tuner.classify(12.3, 8) == 9 and tuner.classify(0.8, 8) == 1
    with pytest.raises(ph.NonPositiveRatio):
        tuner.classify(0.0, 8)
    assert tuner.histogram([1, 4, 4, 9, 4], 8).tolist() == [1, 0, 0, 3, 0, 0, 0, 0, 1]
    assert tuner.sort_by_class([2, 1, 2]).tolist() == [1, 0, 2]
    assert tuner.class_starts([2, 0, 3]).tolist() == [0, 2, 2]
    cfg = ph.TunerConfig(t_high=8, capacity_table={4: 5120})
    assert tuner.capacity(4, cfg) == 5120 and tuner.capacity(3, cfg) == 3072 and tuner.capacity(9, cfg) == 3584
    with pytest.raises(ValueError):
        tuner.capacity(0, cfg)


def test_emit_gap_host_utility():
    lay = ph.LayoutConfig(8, 1, 32)
    from golden_cases import case
    c = case("worked")
    assert ph.emit_gap(c["oracle_starts"], lay, c.total_bits).tolist() == [0, 0, 1, 2]
    assert ph.signed_gaps(c["oracle_starts"], lay, c.total_bits).tolist() == [0, 0, -2, -1]
    with pytest.raises(ph.GapOverflow):
        ph.emit_gap(np.array([0, 400]), ph.LayoutConfig(8, 1, 4), 420)


def test_decode_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from golden_cases import case
    c = case("zipf_32_4_32_w16")
    book = ph.canonize({s: ln for s, (_, ln) in c.codebook.entries.items()}, symbol_width=16)
    st = ph.EncodedStream(layout=ph.DEFAULT_LAYOUT, units=c.units, total_bits=c.total_bits,
                          symbol_count=c.symbol_count, codebook=book, gap=c.gap)
    with pytest.raises(RuntimeError, match="CUDA"):
        ph.gap_decoder.decode(st)
    with pytest.raises(RuntimeError, match="CUDA"):
        ph.sync_decoder.decode(st)


def test_chunk_stream_partitions_symbols_and_windows():
    """Sequence-aligned chunks (sharded decode): every symbol in exactly one
    chunk, chunk spans end at the next chunk's first codeword start."""
    import numpy as np
    from paper_2201_09118_b200 import shard
    rng = np.random.default_rng(3)
    sb, sps = 128, 4
    tb = 128 * 4 * 37 + 77
    nsub = -(-tb // sb)
    gap = rng.integers(0, 20, nsub).astype(np.uint8)
    gap[0] = 0
    counts = rng.integers(0, 60, nsub)
    for k in (1, 2, 5, 10, 37, 100):
        ch = shard.chunk_stream(tb, sb, sps, gap, counts, k)
        assert sum(c.n for c in ch) == counts.sum()
        assert [c.out0 for c in ch] == list(np.cumsum([0] + [c.n for c in ch])[:-1])
        assert ch[0].q0 == 0 and ch[-1].q1 == -(-nsub // sps)
        for a, b in zip(ch, ch[1:]):
            assert a.q1 == b.q0
            assert a.word0 * 32 + a.total_bits == b.word0 * 32 + b.first_entry  # ends at the next entry
            assert b.first_entry == gap[b.sub0]
        assert ch[-1].word0 * 32 + ch[-1].total_bits == tb
        assert all(c.sub0 + c.nsub <= nsub for c in ch)


def test_chunk_stream_rejects_unaligned_sequences():
    """A chunk's payload pointer must stay 16-byte aligned (the fused kernel
    stages words with 16-byte cp.async): sequences of a non-multiple of 128
    bits, e.g. layout (32, 3, 33), cannot be chunked."""
    import numpy as np
    import pytest
    from paper_2201_09118_b200 import shard
    sb, sps = 96, 33
    tb = sb * sps * 5
    nsub = -(-tb // sb)
    with pytest.raises(ValueError, match="128-bit"):
        shard.chunk_stream(tb, sb, sps, np.zeros(nsub, np.uint8), np.ones(nsub, np.int64), 2)
