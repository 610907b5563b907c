"""Run a few decodes of one bench workload (for ncu / compute-sanitizer runs).

    ncu --set full -k regex:k_fused -s 2 -c 1 -o gpurun_out/x python tools/prof_decode.py
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import Decoder, build_field  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hurricane")
    ap.add_argument("--variant", default="gap")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--fused", type=int, default=1)
    args = ap.parse_args()
    spec, codes, book, stream = build_field(args.config, 0)
    dec = Decoder(stream, args.variant, fused=bool(args.fused))
    for _ in range(args.iters):
        dec()
    torch.cuda.synchronize()
    r = dec.status()
    ok = np.array_equal(dec.out[: len(codes)].cpu().numpy().view(np.uint16), codes)
    print(f"{spec.name} {args.variant}: status {r.status} bit-exact {ok}")


if __name__ == "__main__":
    main()
