"""Python API contract on the GPU: phase-named timings that add up to the call
(reference tests/test_container_cli.py:253-266), and concurrent callers
(reference decoders are safe for concurrent use; staging.py:48-62)."""

import threading
import time

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


@pytest.fixture(scope="module")
def field(ph):
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(12_000_000, 1024, 3.0, seed=2)
    return codes, ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)


@pytest.mark.parametrize("variant,tuned", [("gap", False), ("gap", True), ("sync", False), ("sync", True)])
@pytest.mark.parametrize("stats", [False, True])
def test_report_accounting(ph, field, variant, tuned, stats):
    codes, st = field
    dec = ph.gap_decoder if variant == "gap" else ph.sync_decoder
    dec.decode(st)  # warm: device mirror and tables built
    timings = {}
    kw = {"tuner_config": ph.TunerConfig()} if tuned else {}
    if stats:
        kw["stats"] = ph.DecodeStats()
    t0 = time.perf_counter()
    out = dec.decode(st, timings=timings, **kw)
    total = time.perf_counter() - t0
    assert np.array_equal(out, codes)
    want = (["entries_from_gap", "count_pass"] if variant == "gap" else
            ["intra_sync", "inter_sync", "output_index"]) + (["tune"] if tuned else []) + ["decode_write"]
    assert list(timings) == want
    assert all(v >= 0 for v in timings.values())
    assert sum(timings.values()) == pytest.approx(total, rel=0.05)
    # the device phases are real: the count / sync phase took device time
    key = "count_pass" if variant == "gap" else "intra_sync"
    assert timings[key] > 0


def test_concurrent_callers_on_their_own_streams(ph):
    """Four host threads, each on its own CUDA stream, decode different fields
    at the same time through the Python API: every result bit-exact (the
    workspace is per (device, stream), the device mirror is ordered by an
    event)."""
    import torch
    from paper_2201_09118_b200.synth import gaussian_codes
    fields = []
    for i in range(4):
        c = gaussian_codes(1_500_000 + 1000 * i, 1024, (0.6, 3.0, 8.0, 22.0)[i], seed=40 + i)
        fields.append((c, ph.encode(c, ph.book_for(c, 16), ph.DEFAULT_LAYOUT, with_gap=True)))
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                codes, st = fields[i]
                for _ in range(5):
                    for dec in (ph.gap_decoder, ph.sync_decoder):
                        if not np.array_equal(dec.decode(st), codes):
                            errors.append((i, dec.__name__))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((i, repr(e)))

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert errors == []
