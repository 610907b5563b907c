"""Randomized equivalence on the GPU (the reference's acceptance criteria 4/5,
tests/test_acceptance.py:82-141): for 1,000 seeded streams the GPU sync,
gap and tuner-partitioned decoders all equal the pinned CPU oracle, with
layouts, capacities and t_high varied across cases."""

import numpy as np
import pytest

from streams import case_lengths, case_symbols

pytestmark = pytest.mark.gpu

CAPS = (1, 8, 1024, 3584, 8192)
T_HIGH = (1, 4, 8)
LAYOUTS = ((32, 4, 32), (32, 4, 32), (32, 4, 32), (16, 3, 5), (8, 5, 7), (32, 3, 33), (32, 8, 16))


@pytest.fixture(scope="module")
def ph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    return ph


def test_thousand_streams_match_oracle(ph, oracle_mod):
    rng = np.random.default_rng(0xC0DEC)
    lengths = case_lengths(rng)
    mismatches = []
    for index, n in enumerate(lengths):
        syms, width = case_symbols(rng, index, n)
        lay = ph.LayoutConfig(*LAYOUTS[index % len(LAYOUTS)])
        book = ph.book_for(syms, width)
        st = ph.encode(syms, book, lay, with_gap=True)
        ref = oracle_mod.oracle_decode(st).symbols
        if not np.array_equal(ref, syms):
            mismatches.append((index, "oracle"))
            continue
        cap = CAPS[index % len(CAPS)]
        cfg = ph.TunerConfig(t_high=T_HIGH[index % len(T_HIGH)])
        outs = {
            "gap": ph.gap_decoder.decode(st, capacity=cap),
            "sync": ph.sync_decoder.decode(st, capacity=cap),
            "gap_tuned": ph.gap_decoder.decode(st, tuner_config=cfg),
            "sync_tuned": ph.sync_decoder.decode(st, tuner_config=cfg),
        }
        if index % 7 == 0:
            outs["sync_staged"] = ph.sync_decoder.decode(st, stats=ph.DecodeStats())
        for k, v in outs.items():
            if not np.array_equal(v, ref):
                mismatches.append((index, k, n))
    assert mismatches == []


def test_sync_points_sound(ph, oracle_mod):
    """Every validated sync point is an oracle codeword start (criterion 5)."""
    rng = np.random.default_rng(5)
    for index in range(60):
        syms, width = case_symbols(rng, index, int(rng.integers(1000, 60_000)))
        st = ph.encode(syms, ph.book_for(syms, width), ph.DEFAULT_LAYOUT)
        state = ph.sync_decoder.synchronize(st)
        orc = oracle_mod.oracle_decode(st)
        ref = oracle_mod.synchronize(st)
        assert np.array_equal(state.entry_bits, ref.entry_bits)
        assert np.array_equal(state.iterations, ref.iterations)
        starts = np.append(orc.starts, st.total_bits)
        assert np.isin(state.entry_bits, starts).all()


@pytest.mark.parametrize("cap,warps", [("256", "4"), ("512", "8"), ("1024", "32"), ("", "1")])
def test_fused_staging_rounds_and_bypass(ph, oracle_mod, monkeypatch, cap, warps):
    """Small staging capacities force the fused kernel into the reference's
    round/straddler/bypass rule; the output must not change."""
    if cap:
        monkeypatch.setenv("BH_FUSED_CAP", cap)
    monkeypatch.setenv("BH_FUSED_WARPS", warps)
    rng = np.random.default_rng(int(cap or 0) + int(warps))
    for sharp, n in ((0.999, 300_000), (0.9, 200_000), (0.3, 100_000)):
        syms, _ = case_symbols(rng, 0, n)
        from streams import synth_codes
        syms = synth_codes(n, sharp, int(rng.integers(1 << 30)))
        st = ph.encode(syms, ph.book_for(syms, 16), ph.DEFAULT_LAYOUT, with_gap=True)
        assert np.array_equal(ph.gap_decoder.decode(st), syms)
        assert np.array_equal(ph.sync_decoder.decode(st), syms)


def test_fused_matches_staged_on_layouts(ph):
    rng = np.random.default_rng(77)
    for lay in ((32, 4, 32), (16, 3, 5), (8, 5, 7), (32, 1, 32), (32, 8, 16), (8, 1, 32), (32, 2, 3)):
        for _ in range(3):
            syms, width = case_symbols(rng, int(rng.integers(0, 100)), int(rng.integers(1, 80_000)))
            st = ph.encode(syms, ph.book_for(syms, width), ph.LayoutConfig(*lay), with_gap=True)
            assert np.array_equal(ph.gap_decoder.decode(st), syms), lay
            assert np.array_equal(ph.sync_decoder.decode(st), syms), lay


@pytest.mark.parametrize("wide", ["", "0", "1"])
@pytest.mark.parametrize("sigma,eps", [(0.2, 1e-3), (0.6, 0.0), (3.0, 0.0), (8.0, 0.0), (22.0, 0.0), (8.0, 2e-3)])
def test_table_layouts_on_cusz_fields(ph, monkeypatch, wide, sigma, eps):
    """Both decode-table layouts (narrow 8-bit replicated / wide 12-bit) and
    the automatic choice decode cuSZ-shaped fields bit-exactly -- short and
    long codes, seed-dependent seams (sigma 22), codes past 12 bits (eps)."""
    from paper_2201_09118_b200.synth import gaussian_codes
    if wide:
        monkeypatch.setenv("BH_FUSED_WIDE", wide)
    codes = gaussian_codes(1_500_000, 1024, sigma, eps, seed=int(sigma * 10) + 3)
    st = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
    assert np.array_equal(ph.gap_decoder.decode(st), codes)
    assert np.array_equal(ph.sync_decoder.decode(st), codes)
