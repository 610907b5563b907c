"""K1 (bh_table_build) alone: CUDA-event time per build, back to back and
after an L2 flush, for the bench configs' books."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_09118_b200 as ph  # noqa: E402
from paper_2201_09118_b200 import _lib  # noqa: E402
from bench import load_synth  # noqa: E402

synth = load_synth()
lib = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in ("hurricane", "hacc", "nyx4096", "qmcpack"):
    codes = synth.field_codes(synth.FIELDS[name], n=2_000_000)
    book = ph.book_for(codes, 16)
    lens = torch.from_numpy(book.length_bytes()).cuda()
    mc = max(len(book.entries), 1)
    table = torch.empty(lib.bh_table_bytes(mc), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def build():
        _lib.check(lib.bh_table_build(lens.data_ptr(), lens.numel(), table.data_ptr(), mc, st))
    for _ in range(5):
        build()
    torch.cuda.synchronize()
    res = {}
    for mode in ("back-to-back", "after L2 flush"):
        ts = []
        for _ in range(50):
            if mode != "back-to-back":
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            build()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[mode] = statistics.median(ts)
    # an empty event pair for reference
    ts = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"{name:10s} alphabet {lens.numel():5d} max_len {book.max_len:2d}: K1 "
          + ", ".join(f"{k} {v:.1f} us" for k, v in res.items()) + f"; empty event pair {statistics.median(ts):.1f} us")
