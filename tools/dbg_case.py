"""Debug one golden case on the GPU: fused decoders vs the oracle (counts, status)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402

import paper_2201_09118_b200 as ph  # noqa: E402
from golden_cases import case  # noqa: E402
from test_gpu_parity import as_stream  # noqa: E402

name = sys.argv[1]
c = case(name)
st = as_stream(ph, c)
print(name, "tb", st.total_bits, "n", st.symbol_count, "nsub", st.num_subseqs, "layout", st.layout, "gap", None if st.gap is None else st.gap[:8])
for var in ("gap", "sync"):
    mod = ph.gap_decoder if var == "gap" else ph.sync_decoder
    try:
        out = mod.decode(st)
        print(var, "no raise; out", out[:10], "ok" if np.array_equal(out, c.symbols) else "differs")
    except Exception as e:  # noqa: BLE001
        print(var, "raised", type(e).__name__, e)
