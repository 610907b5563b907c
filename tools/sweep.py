"""SURVEY.md §8(d) sweeps on one B200 (python tools/sweep.py > profiles/.../sweeps.md):

* HACC-shaped field: stream layout units_per_subseq x subseqs_per_seq
  ({2,4,8} x {16,32,64}), both decoders (subseqs_per_seq 64 runs the
  reference-structured pipeline: the fused kernel maps one warp lane per
  subsequence);
* staging capacity 1024..8192 step 512 (BH_FUSED_CAP) against the tuned one,
  Hurricane and HACC, gap decoder;
* the cuSZ-style coarse baseline over chunk sizes 2^8..2^14 (HACC).

Every point is checked bit-exact against the generated codes before timing.
"""
import ctypes as C
import os
import statistics
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_09118_b200 as ph  # noqa: E402
from bench import Decoder, FLUSH_BYTES, time_steps  # noqa: E402
from paper_2201_09118_b200 import _lib  # noqa: E402
from paper_2201_09118_b200.synth import FIELDS, field_codes  # noqa: E402

flush_buf = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")


def flush():
    flush_buf.zero_()


def timed(dec, n, steps=20):
    dec()
    torch.cuda.synchronize()
    _lib.check(dec.status().status, "sweep")
    got = dec.out[:n].cpu().numpy().view(np.uint16)
    ts = time_steps(dec, steps, 3, flush)
    return got, statistics.mean(ts)


def gbs(n, ms):
    return 2 * n / (ms / 1e3) / 1e9


def layout_sweep():
    spec = FIELDS["hacc"]
    codes = field_codes(spec)
    book = ph.book_for(codes, 16)
    print("## HACC-shaped field (281 M codes): stream layout sweep\n")
    print("| units/subseq | subseqs/seq | CR | gap GB/s | sync GB/s |")
    print("|---|---|---|---|---|")
    for ups in (2, 4, 8):
        for sps in (16, 32, 64):
            lay = ph.LayoutConfig(32, ups, sps)
            st = ph.encode(codes, book, lay, with_gap=True)
            row = []
            for var in ("gap", "sync"):
                dec = Decoder(st, var)
                got, ms = timed(dec, len(codes), 10)
                assert np.array_equal(got, codes), (ups, sps, var)
                row.append(f"{gbs(len(codes), ms):.0f}")
                del dec
            print(f"| {ups} | {sps} | {16 * len(codes) / st.total_bits:.2f} | {row[0]} | {row[1]} |", flush=True)
            del st
            torch.cuda.empty_cache()


def capacity_sweep():
    print("\n## Staging capacity (symbols per warp; BH_FUSED_CAP) vs the tuned capacity, gap decoder\n")
    print("| field | capacity | GB/s |")
    print("|---|---|---|")
    for name in ("hurricane", "hacc"):
        spec = FIELDS[name]
        codes = field_codes(spec)
        book = ph.book_for(codes, 16)
        st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
        caps = [""] + [str(c) for c in range(1024, 8193, 512)]
        for cap in caps:
            if cap:
                os.environ["BH_FUSED_CAP"] = cap
            else:
                os.environ.pop("BH_FUSED_CAP", None)
            dec = Decoder(st, "gap")
            try:
                got, ms = timed(dec, len(codes), 10)
            except RuntimeError as e:  # capacity leaves too little shared memory for one warp
                print(f"| {spec.name} | {cap} | (does not fit: {e}) |")
                continue
            assert np.array_equal(got, codes), (name, cap)
            print(f"| {spec.name} | {cap or 'tuned'} | {gbs(len(codes), ms):.0f} |", flush=True)
            del dec
        os.environ.pop("BH_FUSED_CAP", None)


def coarse_sweep():
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty, h2d
    from paper_2201_09118_b200.encoder import encode_device
    print("\n## cuSZ-style coarse-grained baseline (K8) over chunk sizes, HACC-shaped field\n")
    print("| chunk (symbols) | GB/s |")
    print("|---|---|")
    spec = FIELDS["hacc"]
    codes = field_codes(spec)
    book = ph.book_for(codes, 16)
    st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    lib = _lib.load()
    ds = device_stream(st)
    sd = h2d(codes, ds.device)
    out = empty(len(codes), np.uint16, ds.device)
    for k in range(8, 15):
        chunk = 1 << k
        _, _, _, offs = encode_device(sd, len(codes), book, ph.DEFAULT_LAYOUT, False, chunk)
        rep = DeviceReport(ds.device).init()

        def fn():
            check(lib.bh_coarse_decode(ds.ref, offs.data_ptr(), chunk, out.data_ptr(), rep.ptr,
                                       stream_handle()), "coarse")
        fn()
        torch.cuda.synchronize()
        check(rep.read().status, "coarse")
        assert np.array_equal(out[: len(codes)].cpu().numpy().view(np.uint16), codes)
        ms = statistics.mean(time_steps(fn, 5, 2, flush))
        print(f"| {chunk} | {gbs(len(codes), ms):.1f} |", flush=True)


if __name__ == "__main__":
    print("# Round-1 sweeps (B200, one GPU; CUDA events per decode, L2 flushed between decodes)\n")
    which = sys.argv[1:] or ["layout", "capacity", "coarse"]
    if "layout" in which:
        layout_sweep()
    if "capacity" in which:
        capacity_sweep()
    if "coarse" in which:
        coarse_sweep()
