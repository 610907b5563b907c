"""Input generators for property tests (restated from the reference's test
helpers: Zipf draws, tests/conftest.py:65-69; synth_codes, quant.py:77-96;
the acceptance-suite case mix, tests/test_acceptance.py:67-79)."""

import numpy as np


def zipf(rng, n, alphabet):
    w = 1.0 / np.arange(1, alphabet + 1, dtype=np.float64)
    w /= w.sum()
    return rng.choice(alphabet, size=n, p=w).astype(np.uint16)


def synth_codes(n, sharpness, seed, width=16):
    rng = np.random.default_rng(seed)
    p = sharpness ** 4
    mag = rng.geometric(p, size=n).astype(np.int64) - 1
    sign = rng.integers(0, 2, size=n, dtype=np.int64) * 2 - 1
    mid = 1 << (width - 1)
    return np.clip(mid + sign * mag, 0, (1 << width) - 1).astype(np.uint16)


SHARP = (0.12, 0.3, 0.46, 0.6, 0.75, 0.9, 0.95, 0.98, 0.999)


def case_symbols(rng, index, n):
    """(symbols, width) for acceptance-style case `index`."""
    if index % 2 == 0:
        s = SHARP[index // 2 % len(SHARP)]
        codes = synth_codes(n, s, int(rng.integers(2 ** 31)))
        dev = codes.astype(np.int64) - 32768
        return (32768 + np.clip(dev, -2048, 2047)).astype(np.uint16), 16
    width = 8 if index % 4 == 1 else 16
    alphabet = int(rng.integers(2, 257 if width == 8 else 4097))
    return zipf(rng, n, alphabet), width


def case_lengths(rng, count=1000):
    lengths = [0, 1, 2, 3, 7]
    lengths += [int(x) for x in np.exp(rng.uniform(np.log(4), np.log(20_000), count - 45))]
    lengths += [100_000] * 36 + [250_000, 500_000, 750_000, 1_000_000]
    return lengths
