import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2201_09118_b200 as ph
from streams import case_lengths, case_symbols
rng = np.random.default_rng(0xC0DEC)
lengths = case_lengths(rng)
for index, n in enumerate(lengths):
    syms, width = case_symbols(rng, index, n)
    if index == 997: break
lay = ph.LayoutConfig(16, 3, 5)
st = ph.encode(syms, ph.book_for(syms, width), lay, with_gap=True)
try:
    out = ph.gap_decoder.decode(st)
    print("equal", np.array_equal(out, syms))
except Exception as e:
    print("error", e)
