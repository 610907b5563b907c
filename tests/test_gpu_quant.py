"""Reconstruction after decode on the device: the one-pass
segmented scan in the provably exact regime and the on-device reference
recurrence otherwise, both bit-identical (as float64 bit patterns) to the
reference's dequantize (golden fixtures from the real parhuff) and, at scale,
to the pinned C restatement of dequantize_chain."""

import numpy as np
import pytest

from test_oracle_quant import quant_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    return ph


EXPECT_PATH = {"walk_pow2": "scan", "walk_w8": "scan", "sine_pow2_small_eb": "scan", "walk_1e-3": "chain",
               "jumps_pow2": "chain", "ramp_pow2": "chain"}


def test_reference_fixtures(ph):
    from paper_2201_09118_b200 import quant
    import torch
    for name, c in quant_cases().items():
        cfg = quant.QuantConfig(float(c["eb"]), int(c["width"]))
        got = quant.dequantize(quant.QuantResult(c["codes"], c["oidx"], c["oval"]), cfg)
        assert np.array_equal(got.view(np.uint64), c["expect"].view(np.uint64)), name
        st = {}
        codes = torch.from_numpy(c["codes"].astype(np.uint16).view(np.int16)).cuda()
        quant.dequantize_device(codes, c["codes"].size, c["oidx"], c["oval"], cfg, stats=st)
        assert st["path"] == EXPECT_PATH[name], (name, st)


@pytest.mark.parametrize("n,sigma,n_out", [(1, 3.0, 0), (4095, 3.0, 0), (4097, 3.0, 2), (3_000_001, 8.0, 0),
                                           (20_000_000, 3.0, 500), (50_000_000, 22.0, 3000)])
def test_scan_matches_chain_at_scale(ph, oracle_mod, n, sigma, n_out):
    """Exact regime at scale (outlier values multiples of 2eb, several per
    tile and across tile seams): scan == the reference recurrence."""
    import torch
    from paper_2201_09118_b200 import quant
    from paper_2201_09118_b200.synth import gaussian_codes
    rng = np.random.default_rng(n)
    codes = (gaussian_codes(n, 1024, sigma, seed=3).astype(np.int64) - 512 + 32768).astype(np.uint16)
    eb = 2.0 ** -12
    oidx = np.sort(rng.choice(n, size=min(n_out, n), replace=False)).astype(np.int64)
    oval = rng.integers(-2 ** 20, 2 ** 20, oidx.size).astype(np.float64) * (2 * eb)
    want = oracle_mod.dequantize(codes, oidx, oval, 2 * eb, 32768)
    st = {}
    got = quant.dequantize_device(torch.from_numpy(codes.view(np.int16)).cuda(), n, oidx, oval,
                                  quant.QuantConfig(eb), stats=st)
    assert st["path"] == "scan"
    assert np.array_equal(got.cpu().numpy().view(np.uint64), want.view(np.uint64))


def test_running_sum_past_2_24_falls_back(ph, oracle_mod):
    import torch
    from paper_2201_09118_b200 import quant
    n = 1_000_000
    codes = np.full(n, 32768 + 40, np.uint16)  # the running sum reaches 4e7 units
    st = {}
    got = quant.dequantize_device(torch.from_numpy(codes.view(np.int16)).cuda(), n, [], [],
                                  quant.QuantConfig(2.0 ** -5), stats=st)
    assert st["path"] == "chain"
    want = oracle_mod.dequantize(codes, [], [], 2.0 ** -4, 32768)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("variant", ["gap", "sync"])
def test_decode_then_dequantize_on_device(ph, oracle_mod, variant):
    """Decode a field and reconstruct it without the codes leaving the GPU."""
    from paper_2201_09118_b200 import quant
    from paper_2201_09118_b200.synth import gaussian_codes
    # quantization codes around the 16-bit midpoint (cuSZ-style)
    codes = (gaussian_codes(5_000_000, 1024, 3.0, seed=11).astype(np.int64) - 512 + 32768).astype(np.uint16)
    st = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
    cfg = quant.QuantConfig(2.0 ** -9, 16)
    oidx = np.array([0, 17, 4096, 4_999_999], np.int64)
    oval = np.array([3.0, -2.5, 1024.0, 7.0])
    stats = {}
    got = quant.decode_dequantize(st, oidx, oval, cfg, variant, stats=stats)
    assert stats["path"] == "scan"
    want = oracle_mod.dequantize(codes, oidx, oval, 2 * cfg.error_bound, cfg.midpoint)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
