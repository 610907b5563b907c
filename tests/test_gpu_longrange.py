"""The fused kernel's long-range branch (csrc/fused.cu k_fused2 with a CTA
range longer than its shared-memory tile arrays): tile totals and offsets
through the workspace with a block-wide scan, SYNC seam candidates and exit
descriptors in global memory, and the global exit-descriptor spins of the
seam fix-up.  Full-size HACC and QMCPACK take this branch naturally (about
1,200 tiles per CTA); here it is forced at small sizes with the test knobs
BH_FUSED_SMEM_TILES (shared-memory tile limit) and BH_FUSED_GRID (fewer CTAs),
both decoders, including streams whose seams depend on the seed (sigma 22)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    return ph


@pytest.fixture
def knobs():
    saved = {k: os.environ.get(k) for k in ("BH_FUSED_SMEM_TILES", "BH_FUSED_GRID")}

    def set_(tiles=None, grid=None):
        for k, v in (("BH_FUSED_SMEM_TILES", tiles), ("BH_FUSED_GRID", grid)):
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)
    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("sigma,n", [(0.6, 3_000_000), (8.0, 2_000_000), (22.0, 1_500_000), (3.0, 400_000)])
@pytest.mark.parametrize("tiles,grid", [(0, None), (0, 3), (16, 5), (None, 1), (None, 2)])
def test_long_range_branch_bit_exact(ph, knobs, sigma, n, tiles, grid):
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(n, 1024, sigma, seed=int(sigma * 10) + n % 7)
    book = ph.book_for(codes, 16)
    st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    knobs(tiles, grid)
    try:
        for dec in (ph.gap_decoder, ph.sync_decoder):
            got = dec.decode(st)
            assert np.array_equal(got, codes), (dec.__name__, sigma, tiles, grid)
    finally:
        knobs()


def test_long_range_corrupt_streams_still_raise(ph, knobs):
    """Damaged streams through the long-range branch raise like the reference."""
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(500_000, 1024, 8.0, seed=3)
    book = ph.book_for(codes, 16)
    st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    bad_count = ph.EncodedStream(layout=st.layout, units=st.units, total_bits=st.total_bits,
                                 symbol_count=st.symbol_count + 3, codebook=st.codebook, gap=st.gap)
    knobs(0, 2)
    try:
        with pytest.raises(ph.BadGap):
            ph.gap_decoder.decode(bad_count)
        with pytest.raises(ph.Truncated):
            ph.sync_decoder.decode(bad_count)
    finally:
        knobs()


@pytest.mark.parametrize("window", [0, 8, 24])
@pytest.mark.parametrize("sigma,n,tiles,grid", [(8.0, 2_000_000, None, None), (22.0, 1_500_000, 0, 3),
                                                (3.0, 3_000_000, None, 2), (0.6, 1_000_000, 16, 5)])
def test_seam_walk_serial_pass(ph, knobs, window, sigma, n, tiles, grid):
    """Self-sync seams inside a CTA's range are resolved by one walk from the
    predecessor's exit; walks that do not meet go to warp 0's ordered serial
    pass (csrc/fused.cu, BH_SEAMWALK), including successor chains when a
    re-synchronised exit changes and the ordered scan once more than FAIL_CAP
    (128) walks failed in one CTA.  BH_SEAMWALK_WINDOW narrows the walk window
    so that most seams take that pass (window 0: all whose seed differs from
    the slot's own entry)."""
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(n, 1024, sigma, seed=int(sigma * 10) + n % 11)
    book = ph.book_for(codes, 16)
    st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    knobs(tiles, grid)
    os.environ["BH_SEAMWALK_WINDOW"] = str(window)
    try:
        got = ph.sync_decoder.decode(st)
        assert np.array_equal(got, codes), (sigma, window, tiles, grid)
    finally:
        os.environ.pop("BH_SEAMWALK_WINDOW", None)
        knobs()


@pytest.mark.parametrize("bits", [0, 32, 128])
def test_presync_lengths_bit_exact(ph, bits):
    """Every pre-synchronisation length (BH_PRESYNC_BITS) decodes the same
    symbols: the entry guess only decides how often the intra-sequence rounds
    re-decode.  Narrow (short-code) and wide books, 16-bit units."""
    from paper_2201_09118_b200.synth import gaussian_codes
    os.environ["BH_PRESYNC_BITS"] = str(bits)
    try:
        for sigma, n in ((0.8, 1_000_000), (8.0, 1_000_000), (22.0, 700_000)):
            codes = gaussian_codes(n, 1024, sigma, seed=n % 13 + int(sigma))
            book = ph.book_for(codes, 16)
            for lay in (ph.DEFAULT_LAYOUT, ph.LayoutConfig(16, 8, 16)):
                st = ph.encode(codes, book, lay, with_gap=True)
                assert np.array_equal(ph.sync_decoder.decode(st), codes), (sigma, bits, lay)
    finally:
        os.environ.pop("BH_PRESYNC_BITS", None)
