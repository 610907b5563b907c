"""Randomized soak of the fused decoders on cuSZ-shaped fields (GPU).

    python tools/fuzz.py [--minutes 8] [--seed 1]

Every case draws a field (size, bins, sigma, uniform floor), a stream layout
and the library's tuning knobs (lane window, table layout, warps, staging
capacity), encodes it and checks that both decoders, the tuner-partitioned
decoder and a sequence-aligned chunked decode return the generated codes
bit-exactly.  Prints one line per case and a summary; exits 1 on a mismatch.
"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

LAYOUTS = ((32, 4, 32), (32, 4, 32), (32, 4, 32), (16, 3, 5), (8, 5, 7), (32, 3, 33), (32, 8, 16), (32, 2, 64),
           (16, 8, 16), (32, 1, 32))
KNOBS = ("BH_FUSED_SPL", "BH_FUSED_WIDE", "BH_FUSED_WARPS", "BH_FUSED_CAP", "BH_FUSED_MODE", "BH_FUSED_SMEM_TILES",
         "BH_FUSED_GRID")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=8.0)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200.synth import gaussian_codes
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + 60 * args.minutes
    cases = fails = 0
    while time.time() < t_end:
        for k in KNOBS:
            os.environ.pop(k, None)
        n = int(rng.choice([1, 7, 1000, 65_537, 400_000, 2_000_000, 6_000_000]))
        bins = int(rng.choice([2, 16, 256, 1024, 4096]))
        sigma = float(rng.choice([0.05, 0.3, 0.6, 2.0, 8.0, 22.0, 60.0]))
        eps = float(rng.choice([0.0, 0.0, 1e-4, 1e-2]))
        lay = LAYOUTS[int(rng.integers(len(LAYOUTS)))]
        knobs = {}
        if rng.random() < 0.5:
            knobs["BH_FUSED_SPL"] = str(int(rng.choice([1, 2, 4])))
        if rng.random() < 0.3:
            knobs["BH_FUSED_WIDE"] = str(int(rng.integers(2)))
        if rng.random() < 0.3:
            knobs["BH_FUSED_WARPS"] = str(int(rng.choice([1, 3, 8, 16, 24])))
        if rng.random() < 0.2:
            knobs["BH_FUSED_CAP"] = str(int(rng.choice([64, 300, 1024, 4096])))
        if rng.random() < 0.3:
            knobs["BH_FUSED_MODE"] = str(int(rng.integers(1, 3)))
        if rng.random() < 0.15:
            knobs["BH_FUSED_SMEM_TILES"] = str(int(rng.choice([0, 4, 64])))
        if rng.random() < 0.15:
            knobs["BH_FUSED_GRID"] = str(int(rng.choice([1, 2, 7, 40])))
        os.environ.update(knobs)
        codes = gaussian_codes(n, bins, sigma, eps, seed=int(rng.integers(1 << 31)))
        import torch
        book = ph.book_for_device(torch.from_numpy(codes.view(np.int16)).cuda(), n, 16)
        if rng.random() < 0.2 and book.entries != ph.book_for(codes, 16).entries:
            print(f"case {cases + 1}: device book differs from the host build_lengths", flush=True)
            fails += 1
        st = ph.encode(codes, book, ph.LayoutConfig(*lay), with_gap=True)
        th = int(rng.integers(1, 9))
        outs = {
            "gap": ph.gap_decoder.decode(st),
            "sync": ph.sync_decoder.decode(st),
            "gap_tuned": ph.gap_decoder.decode(st, tuner_config=ph.TunerConfig(t_high=th)),
            "sync_tuned": ph.sync_decoder.decode(st, tuner_config=ph.TunerConfig(t_high=th)),
        }
        from paper_2201_09118_b200 import _lib as _l
        from paper_2201_09118_b200.device import device_stream
        shardable = bool(_l.load().bh_fused_supported(device_stream(st).ref, _l.VARIANT_GAP))
        if shardable and (lay[0] * lay[1] * lay[2]) % 128 == 0 and st.num_seqs > 2 and rng.random() < 0.5:
            from paper_2201_09118_b200 import shard
            world = int(rng.integers(2, 5))
            v = "gap" if rng.random() < 0.5 else "sync"
            parts = []
            for r in range(world):
                parts += [(o0, t.cpu().numpy().view(np.uint16)) for _, o0, t in shard.decode_shard([st], r, world, v)]
            outs[f"shard{world}_{v}"] = np.concatenate([p for _, p in sorted(parts, key=lambda x: x[0])])
        bad = [k for k, v in outs.items() if not np.array_equal(v, codes)]
        cases += 1
        fails += bool(bad)
        print(f"case {cases:4d} n={n:8d} bins={bins:4d} sigma={sigma:5.2f} eps={eps:g} layout={lay} "
              f"max_len={book.max_len:2d} knobs={knobs} -> {'MISMATCH ' + ','.join(bad) if bad else 'ok'}",
              flush=True)
    print(f"fuzz: {cases} cases, {fails} mismatching", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
