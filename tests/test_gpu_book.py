"""Codebook construction on the device: the GPU histogram
and the two-queue Huffman length builder (csrc/book.cu) must give exactly the
reference build_lengths books (codebook.py:38-83) -- pinned against the
golden fixtures and full-size digests the real parhuff produced, and against
the host restatement on adversarial tie patterns."""

import hashlib

import numpy as np
import pytest

from golden_cases import all_cases, digests

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    return ph


def dev(a):
    import torch
    a = np.ascontiguousarray(a, dtype=np.uint16)
    return torch.from_numpy(a.view(np.int16).copy()).cuda()


def test_histogram_matches_bincount(ph):
    rng = np.random.default_rng(4)
    for n, hi in ((1, 5), (7, 3), (1000, 70000 // 2), (1_000_003, 9000), (3_000_000, 65536)):
        x = rng.integers(0, hi, n).astype(np.uint16)
        c = ph.symbol_histogram_device(dev(x), n).cpu().numpy()
        want = np.bincount(x, minlength=65536)
        assert np.array_equal(c[:65536], want)


def test_golden_books_from_device(ph):
    """Every golden case whose book the reference built from its symbols
    (book_for in make_golden.py) comes out identical on the device."""
    checked = 0
    for c in all_cases():
        if c.codebook.kind != "canonical" or c.symbols.size == 0:
            continue
        host = ph.book_for(c.symbols, c.codebook.symbol_width)
        if host.entries != c.codebook.entries:
            continue  # a hand-made book (geometric, incomplete, ...)
        got = ph.book_for_device(dev(c.symbols), c.symbols.size, c.codebook.symbol_width)
        assert got.entries == c.codebook.entries, c.name
        checked += 1
    assert checked >= 20


@pytest.mark.parametrize("key", ("1m", "hurricane", "nyx", "nyx256", "nyx4096", "hacc", "cesm", "rtm", "qmcpack"))
def test_full_size_books_from_device(ph, key):
    """The reference's length bytes for every BASELINE config (sha256 written
    by make_golden.py --digests), built from the codes on the device."""
    import torch
    from paper_2201_09118_b200.synth import FIELDS, field_codes
    d = digests()[key]
    codes = field_codes(FIELDS[key])
    book = ph.book_for_device(dev(codes), codes.size, 16)
    _, lens = book.encode_arrays()
    assert book.max_len == d["max_len"]
    assert hashlib.sha256(lens.tobytes()).hexdigest() == d["lengths"]
    torch.cuda.empty_cache()


def counts_book(ph, counts: dict, width=16):
    """Device book from an explicit histogram (symbols materialised)."""
    syms = np.concatenate([np.full(c, s, np.uint16) for s, c in counts.items()]) if counts else np.zeros(0, np.uint16)
    return ph.book_for_device(dev(syms), syms.size, width)


def test_tie_patterns_match_host_build_lengths(ph):
    rng = np.random.default_rng(9)
    cases = [
        {s: 5 for s in range(300)},                      # all counts equal
        {s: 1 + (s % 3) for s in range(1000)},           # few distinct counts, many ties
        {s: 2 ** (s % 7) for s in range(0, 4000, 3)},    # merged sums tie leaves often
        {3: 1, 9: 1},                                    # two symbols
        {65535: 4, 0: 4, 777: 8},                        # extreme symbol values
    ]
    for _ in range(10):
        k = int(rng.integers(2, 4096))
        syms = rng.choice(65536, size=k, replace=False)
        cases.append({int(s): int(c) for s, c in zip(syms, rng.integers(1, 50, k))})
    for cnt in cases:
        want = ph.canonize(ph.build_lengths(cnt), symbol_width=16)
        assert counts_book(ph, cnt).entries == want.entries


def test_single_symbol_and_empty(ph):
    assert counts_book(ph, {42: 17}).entries == {42: (0, 1)}
    assert ph.book_for_device(dev(np.zeros(0, np.uint16)), 0, 16).entries == {0: (0, 1)}


def test_length_overflow_raises(ph):
    """Fibonacci counts force a degenerate tree: codes longer than 32 bits."""
    fib = [1, 1]
    while len(fib) < 36:
        fib.append(fib[-1] + fib[-2])
    cnt = {s: c for s, c in enumerate(fib)}
    with pytest.raises(ph.LengthOverflow):
        ph.build_lengths(cnt)
    # materialising 39 M symbols is fine on the device
    with pytest.raises(ph.LengthOverflow):
        counts_book(ph, cnt)


def test_large_alphabet_uses_host_lengths_on_device_histogram(ph):
    rng = np.random.default_rng(1)
    x = rng.integers(0, 6000, 200_000).astype(np.uint16)  # > 4096 distinct symbols
    assert ph.book_for_device(dev(x), x.size, 16).entries == ph.book_for(x, 16).entries
