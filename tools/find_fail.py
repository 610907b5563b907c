import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2201_09118_b200 as ph
from streams import case_lengths, case_symbols
from oracle import oracle
LAYOUTS = ((32, 4, 32), (32, 4, 32), (32, 4, 32), (16, 3, 5), (8, 5, 7), (32, 3, 33), (32, 8, 16))
rng = np.random.default_rng(0xC0DEC)
lengths = case_lengths(rng)
for index, n in enumerate(lengths):
    syms, width = case_symbols(rng, index, n)
    lay = ph.LayoutConfig(*LAYOUTS[index % len(LAYOUTS)])
    st = ph.encode(syms, ph.book_for(syms, width), lay, with_gap=True)
    for name, fn in (("gap", lambda: ph.gap_decoder.decode(st)), ("sync", lambda: ph.sync_decoder.decode(st))):
        try:
            out = fn()
            ok = np.array_equal(out, syms)
        except Exception as e:
            ok = False; out = repr(e)
        if not ok:
            print("FAIL", index, n, width, lay, name, st.num_seqs, st.total_bits, out if isinstance(out, str) else '')
            break
    else:
        continue
    if index > 400: break
print("done")
