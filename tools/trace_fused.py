"""Per-warp timeline of the fused decode kernel (debug instantiation).

    python tools/trace_fused.py [--config hurricane] [--variant gap]

Records globaltimer stamps at the pipeline's phase boundaries for every warp
(bh_debug_fused_trace) and prints where a CTA's time goes.
"""
import argparse
import os
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import Piece, load_synth  # noqa: E402

SLOTS = 64


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hurricane")
    ap.add_argument("--variant", default="gap")
    ap.add_argument("--noflush", action="store_true")
    args = ap.parse_args()
    import paper_2201_09118_b200 as ph
    synth = load_synth()
    spec = synth.FIELDS[args.config]
    codes = synth.field_codes(spec)
    stream = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
    piece = Piece(stream, args.variant)
    piece.table_build(torch.cuda.current_stream().cuda_stream)

    class Dec:  # one fused decode per call (tables already built)
        lib = piece.lib
        out = piece.out

        def __call__(self):
            piece.decode(torch.cuda.current_stream().cuda_stream)
    dec = Dec()
    lib = dec.lib
    lib.bh_debug_fused_trace.argtypes = [C.c_void_p]
    lib.bh_debug_fused_shape.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                         C.c_void_p, C.c_void_p]
    W, sm = C.c_uint32(), C.c_uint32()
    lib.bh_debug_fused_shape(C.byref(piece.c), C.byref(piece.tune), C.byref(W), C.byref(sm), None, None)
    W = W.value
    nmax = 148 * 8 * W
    tr = torch.zeros(nmax * SLOTS, dtype=torch.int64, device="cuda")
    lib.bh_debug_fused_trace(C.c_void_p(tr.data_ptr()))
    for _ in range(5):
        dec()
    torch.cuda.synchronize()
    tr.zero_()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    if not args.noflush:
        flush.zero_()
    torch.cuda.synchronize()
    dec()
    torch.cuda.synchronize()
    lib.bh_debug_fused_trace(None)
    ok = np.array_equal(dec.out[: len(codes)].cpu().numpy().view(np.uint16), codes)
    t = tr.cpu().numpy().reshape(-1, SLOTS).astype(np.int64)
    used = t[:, 0] > 0
    t = t[used]
    ncta = len(t) // W
    t0 = t[:, 0].min()
    rel = np.where(t > 0, t - t0, -1)
    print(f"{spec.name} {args.variant}: bit-exact {ok}; {ncta} CTAs x {W} warps; smem {sm.value}")
    end = rel[:, SLOTS - 1]
    print(f"kernel span (first start .. last finish) {end.max() / 1e3:.2f} us")

    def q(x):
        x = x[x >= 0]
        return f"med {np.median(x) / 1e3:6.2f} p90 {np.percentile(x, 90) / 1e3:6.2f} max {x.max() / 1e3:6.2f}" if len(x) else "-"

    if os.environ.get("BH_FUSED_V", "2") != "1":
        print("start            ", q(rel[:, 0]))
        print("count tables in  ", q(rel[:, 1]))
        print("count loop done  ", q(rel[:, 9]))
        print("count phase done ", q(rel[:, 2]))
        print("scan+publish     ", q(rel[:, 3]))
        w0 = rel.reshape(ncta, W, SLOTS)[:, 0, :]
        print("warp0 look-back  ", q(w0[:, 3] - w0[:, 2]), " done at", q(w0[:, 3]))
        print("warp0 agg publish", q(w0[:, 5]), " (look-back proper", q(w0[:, 3] - w0[:, 5]), ")")
        raw0 = t.reshape(ncta, W, SLOTS)[:, 0, :]
        print("first poll done  ", q(w0[:, 6]), " last round ready", q(w0[:, 7]), " polls", q(raw0[:, 8] * 1000.0))
        first_flush = rel[:, 4]
        if (first_flush > 0).any():
            print("first flush start", q(first_flush))
        print("decode phase done", q(rel[:, SLOTS - 2]))
        print("finish           ", q(rel[:, SLOTS - 1]))
        cta_end = rel[:, SLOTS - 1].reshape(ncta, W).max(1)
        print("CTA end          ", q(cta_end))
        np.save("gpurun_out/trace_%s_%s.npy" % (args.config, args.variant), rel)
        return
    print("start            ", q(rel[:, 0]))
    print("barrier init     ", q(rel[:, SLOTS - 5]))
    print("bulk tables in   ", q(rel[:, SLOTS - 4]))
    print("replicated       ", q(rel[:, SLOTS - 3]))
    print("tables+words in  ", q(rel[:, 1]))
    print("prologue count   ", q(rel[:, 2]))
    print("prologue publish ", q(rel[:, 3]))
    for k in range(11):
        b = 4 + 5 * k
        if b + 4 >= SLOTS - 2 or (rel[:, b] < 0).all():
            break
        prev = rel[:, 3] if k == 0 else rel[:, b - 1]
        m = rel[:, b + 4] >= 0
        d = lambda i, j: np.where(m, rel[:, j] - rel[:, i], -1)
        print(f"iter {k}: count {q(np.where(m, rel[:, b] - prev, -1))} | decode {q(d(b, b + 1))} | publish {q(d(b + 1, b + 2))}"
              f" | wait {q(d(b + 2, b + 3))} | flush {q(d(b + 3, b + 4))} | done at {q(rel[:, b + 4])}")
    print("loop end         ", q(rel[:, SLOTS - 2]))
    print("finish           ", q(rel[:, SLOTS - 1]))
    # CTA end spread
    cta_end = rel[:, SLOTS - 1].reshape(ncta, W).max(1)
    cta_beg = rel[:, 0].reshape(ncta, W).min(1)
    print("CTA begin        ", q(cta_beg), "\nCTA end          ", q(cta_end))
    np.save("gpurun_out/trace_%s_%s.npy" % (args.config, args.variant), rel)


if __name__ == "__main__":
    main()
