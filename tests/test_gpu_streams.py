"""GPU: the C ABI is stream-ordered with no hidden synchronisation and
thread-safe per (workspace, stream) pair (include/b200huff.h).
Two decodes of different fields are kept in flight on two CUDA streams --
each with its own workspace, report and output, host copies in between like
bench.py's e2e leg -- and every result must be bit-exact."""

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


@pytest.mark.parametrize("variant", ["gap", "sync"])
def test_two_streams_in_flight(ph, variant):
    import torch
    from paper_2201_09118_b200 import _lib
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200._pipeline import make_tune
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty
    from paper_2201_09118_b200.synth import gaussian_codes
    lib = _lib.load()
    var = _lib.VARIANT_GAP if variant == "gap" else _lib.VARIANT_SYNC
    ctxs = []
    for sigma, n, seed in ((0.6, 2_000_000, 3), (8.0, 1_200_000, 4)):
        codes = gaussian_codes(n, 1024, sigma, seed=seed)
        book = ph.book_for(codes, 16)
        stream = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
        ds = device_stream(stream)
        tune = make_tune(max_len=book.max_len, min_len=book.min_len)
        wsb = lib.bh_workspace_bytes(C.byref(ds.c), var, C.byref(tune))
        cs = torch.cuda.Stream()
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=ds.device)
        lib.bh_workspace_reset(ws.data_ptr(), ws.numel(), stream_handle(cs))
        out = empty(n, np.uint16, ds.device)
        host = torch.empty(n, dtype=torch.int16).pin_memory()
        ctxs.append(dict(codes=codes, ds=ds, tune=tune, wsb=wsb, st=cs, ws=ws, out=out, host=host,
                         rep=DeviceReport(ds.device).init()))
    torch.cuda.synchronize()
    for _ in range(3):
        for c in ctxs:  # no synchronisation between the calls
            with torch.cuda.stream(c["st"]):
                c["out"].zero_()
                check(lib.bh_decode_async(C.byref(c["ds"].c), var, C.byref(c["tune"]), c["out"].data_ptr(),
                                          c["ws"].data_ptr(), c["wsb"], c["rep"].ptr, stream_handle(c["st"])),
                      "decode")
                c["host"].copy_(c["out"], non_blocking=True)
    torch.cuda.synchronize()
    for c in ctxs:
        check(c["rep"].read().status, "decode")
        assert np.array_equal(c["host"].numpy().view(np.uint16), c["codes"])


def test_host_threads_decode_concurrently(ph):
    """Four host threads, each with its own stream/workspace/report, call the
    library at the same time (ctypes drops the GIL inside the calls); the
    launch-configuration caches are shared and must stay consistent."""
    import threading

    import torch
    from paper_2201_09118_b200 import _lib
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200._pipeline import make_tune
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty
    from paper_2201_09118_b200.synth import gaussian_codes
    lib = _lib.load()
    fields = []
    for k, sigma in enumerate((0.6, 3.0, 8.0, 22.0)):
        codes = gaussian_codes(600_000, 1024, sigma, seed=40 + k)
        st = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
        fields.append((codes, st, device_stream(st)))
    torch.cuda.synchronize()
    errors = []

    def worker(k):
        try:
            codes, st, ds = fields[k]
            var = _lib.VARIANT_GAP if k % 2 == 0 else _lib.VARIANT_SYNC
            tune = make_tune(max_len=st.codebook.max_len, min_len=st.codebook.min_len)
            cs = torch.cuda.Stream()
            wsb = lib.bh_workspace_bytes(C.byref(ds.c), var, C.byref(tune))
            ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=ds.device)
            out = empty(len(codes), np.uint16, ds.device)
            with torch.cuda.stream(cs):
                lib.bh_workspace_reset(ws.data_ptr(), ws.numel(), stream_handle(cs))
                rep = DeviceReport(ds.device).init()
                for _ in range(5):
                    check(lib.bh_decode_async(C.byref(ds.c), var, C.byref(tune), out.data_ptr(), ws.data_ptr(),
                                              wsb, rep.ptr, stream_handle(cs)), "decode")
            cs.synchronize()
            check(rep.read().status, "decode")
            if not np.array_equal(out.cpu().numpy().view(np.uint16), codes):
                errors.append((k, "mismatch"))
        except Exception as e:  # noqa: BLE001 -- reported below
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert errors == []
