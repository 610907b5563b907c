"""The paper's online tuner on the fused fast path (tuner.py:117-191, PAPER
Alg. 2 / Table I): with a TunerConfig the fused kernel classifies every tile
by its compression ratio, stages it with that class's capacity (classes whose
capacity is below a tile's output take the reference's straddler/bypass
rounds), and histograms the reference sequences into exactly tuner.plan's
classes.  Output never depends on the tuning (test_tuner.py:165-178)."""

import ctypes as C

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


def fused_tuned(ph, st, variant, cfg):
    """bh_decode_async on the fused path with the tuner; returns (output, class histogram)."""
    import torch
    from paper_2201_09118_b200 import _lib
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200._pipeline import make_tune
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty
    lib = _lib.load()
    ds = device_stream(st)
    tune = make_tune(tuner_config=cfg, max_len=st.codebook.max_len, min_len=st.codebook.min_len)
    var = _lib.VARIANT_GAP if variant == "gap" else _lib.VARIANT_SYNC
    wsb = lib.bh_workspace_bytes(ds.ref, var, C.byref(tune))
    ws = torch.zeros(wsb, dtype=torch.uint8, device=ds.device)
    out = empty(st.symbol_count, np.uint16, ds.device)
    rep = DeviceReport(ds.device).init()
    check(lib.bh_decode_async(ds.ref, var, C.byref(tune), out.data_ptr(), ws.data_ptr(), wsb, rep.ptr,
                              stream_handle()), "decode")
    check(rep.read().status, "decode")
    freq = np.zeros(cfg.t_high + 1, np.uint64)
    rc = lib.bh_tuner_class_freq(ds.ref, C.byref(tune), ws.data_ptr(), freq.ctypes.data, freq.size,
                                 stream_handle())
    return out[: st.symbol_count].cpu().numpy().view(np.uint16), (freq if rc == 0 else None)


@pytest.mark.parametrize("sigma,n", [(0.6, 2_000_000), (3.0, 1_000_000), (8.0, 1_500_000), (22.0, 700_000)])
@pytest.mark.parametrize("cfg", [dict(t_high=8), dict(t_high=1), dict(t_high=4, capacity_table={1: 1, 2: 7}),
                                 dict(t_high=16, capacity_table={17: 64})])
def test_fused_tuner_classes_match_plan(ph, sigma, n, cfg):
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(n, 1024, sigma, seed=int(10 * sigma))
    st = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
    tc = ph.TunerConfig(**cfg)
    s = ph.gap_decoder.entries_from_gap(st)
    ph.gap_decoder.count_pass(st, s)
    plan = ph.tuner.plan(st, ph.tuner.sequence_counts(st, s.counts), tc)
    for variant in ("gap", "sync"):
        out, freq = fused_tuned(ph, st, variant, tc)
        assert np.array_equal(out, codes), (variant, cfg)
        assert freq is not None
        assert np.array_equal(freq.astype(np.int64), plan.class_freq), (variant, freq, plan.class_freq)
    # the public API with a tuner takes the same path
    assert np.array_equal(ph.gap_decoder.decode(st, tuner_config=tc), codes)
    assert np.array_equal(ph.sync_decoder.decode(st, tuner_config=tc), codes)


def test_tiny_class_capacities_force_rounds_bit_exact(ph):
    """Capacities of a few symbols per class: every tile takes the reference
    rounds (straddlers, bypass) on the fused path; still bit-exact."""
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(300_000, 1024, 3.0, seed=5)
    st = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
    for caps in ({c: 1 for c in range(1, 10)}, {c: 37 for c in range(1, 10)}, {c: 700 for c in range(1, 10)}):
        tc = ph.TunerConfig(t_high=8, capacity_table=caps)
        for variant in ("gap", "sync"):
            out, _ = fused_tuned(ph, st, variant, tc)
            assert np.array_equal(out, codes), (variant, caps)
