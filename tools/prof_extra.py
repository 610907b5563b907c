"""Small drivers for ncu captures of the non-decode kernels: the device book
builder (k_histogram, k_build_lengths) on the HACC field and the dequantize
scan (k_dequant) on 281 M codes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_09118_b200 as ph  # noqa: E402
from paper_2201_09118_b200 import quant  # noqa: E402
from bench import load_synth  # noqa: E402

synth = load_synth()
codes = synth.field_codes(synth.FIELDS["hacc"])
sd = torch.from_numpy(codes.view(np.int16)).cuda()
for _ in range(2):
    book = ph.book_for_device(sd, codes.size, 16)
q = (sd.to(torch.int32) - 512 + 32768).to(torch.int16)
for _ in range(2):
    st = {}
    out = quant.dequantize_device(q, codes.size, [], [], quant.QuantConfig(2.0 ** -12), stats=st)
torch.cuda.synchronize()
print("book max_len", book.max_len, "dequant path", st["path"])
