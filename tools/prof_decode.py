"""Run a few steps of one bench workload (for ncu / compute-sanitizer runs):
K1 table build + fused decode per iteration, optionally the K8 coarse decoder.

    ncu --set full -k regex:k_fused -s 2 -c 1 -o gpurun_out/x python tools/prof_decode.py --config hacc
    ncu --set full -k regex:k_table_canon -s 2 -c 1 -o gpurun_out/k1 python tools/prof_decode.py
    ncu --set full -k regex:k_coarse -s 1 -c 1 -o gpurun_out/k8 python tools/prof_decode.py --coarse 256
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hacc")
    ap.add_argument("--variant", default="gap")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--coarse", type=int, default=0, help="also run K8 with this chunk size")
    args = ap.parse_args()
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200._lib import check, stream_handle
    from bench import Piece, load_synth
    synth = load_synth()
    codes = synth.field_codes(synth.FIELDS[args.config])
    sd = torch.from_numpy(codes.view(np.int16)).cuda()
    book = ph.book_for_device(sd, codes.size, 16)
    stream = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    p = Piece(stream, args.variant)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(args.iters):
        p.table_build(st)
        p.decode(st)
    torch.cuda.synchronize()
    check(p.rep.read().status, "decode")
    ok = torch.equal(p.out[: codes.size], sd)
    print(f"{args.config} {args.variant}: {'bit-exact' if ok else 'MISMATCH'}")
    if args.coarse:
        from bench import coarse_baseline  # noqa: F401
        from paper_2201_09118_b200.device import DeviceReport, device_stream, empty
        from paper_2201_09118_b200.encoder import encode_device
        from paper_2201_09118_b200 import _lib
        ds = device_stream(stream)
        _, _, _, offs = encode_device(sd, codes.size, book, ph.DEFAULT_LAYOUT, False, args.coarse)
        out = empty(codes.size, np.uint16, ds.device)
        rep = DeviceReport(ds.device).init()
        for _ in range(2):
            check(_lib.load().bh_coarse_decode(ds.ref, offs.data_ptr(), args.coarse, out.data_ptr(), rep.ptr,
                                               stream_handle()), "coarse")
        torch.cuda.synchronize()
        print("coarse", "bit-exact" if torch.equal(out[: codes.size], sd) else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
