"""K1 phase timeline (CTA 0, thread 0 globaltimer stamps) from a build with
-DBH_K1_STAMPS (BH_LIB=... pointing at it): histogram, scan, ranks, l12,
c15, fill."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2201_09118_b200 as ph  # noqa: E402
from paper_2201_09118_b200 import _lib  # noqa: E402
from bench import load_synth  # noqa: E402

synth = load_synth()
lib = _lib.load()
names = ["launch->hist", "hist", "scan", "ranks", "l12", "(cwin start)", "cwin+wlut3+fill"]
for name in ("hurricane", "hacc", "nyx4096"):
    codes = synth.field_codes(synth.FIELDS[name], n=2_000_000)
    book = ph.book_for(codes, 16)
    lens = torch.from_numpy(book.length_bytes()).cuda()
    mc = max(len(book.entries), 1)
    table = torch.empty(lib.bh_table_bytes(mc), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        _lib.check(lib.bh_table_build(lens.data_ptr(), lens.numel(), table.data_ptr(), mc, st))
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 8)()
    lib.bh_debug_k1_stamps(buf)
    s = list(buf)
    print(name, f"entry->init {(s[0] - s[7]) / 1e3:.2f}us ", "  ".join(f"{names[k]} {(s[k] - s[k - 1]) / 1e3:.2f}us" for k in range(1, 7)),
          f"total {(s[6] - s[7]) / 1e3:.2f}us")
