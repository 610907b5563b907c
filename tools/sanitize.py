"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2201_09118_b200 as ph  # noqa: E402
from paper_2201_09118_b200.synth import gaussian_codes  # noqa: E402

for sigma, n in ((0.6, 300_000), (8.0, 200_000), (22.0, 150_000)):
    codes = gaussian_codes(n, 1024, sigma, seed=5)
    st = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
    for name, mod in (("gap", ph.gap_decoder), ("sync", ph.sync_decoder)):
        out = mod.decode(st)
        assert np.array_equal(out, codes), (sigma, name)
        print(f"sigma {sigma} {name}: ok", flush=True)
