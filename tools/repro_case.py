import os, sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2201_09118_b200 as ph
from golden_cases import case
from test_gpu_parity import as_stream
c = case(sys.argv[1])
st = as_stream(ph, c)
for w in sys.argv[2:]:
    os.environ["BH_FUSED_WARPS"] = w
    for name, fn in (("gap", ph.gap_decoder.decode), ("sync", ph.sync_decoder.decode)):
        try:
            out = fn(st)
            print("W", w, name, np.array_equal(out, c.symbols))
        except Exception as e:
            print("W", w, name, "ERR", e)
