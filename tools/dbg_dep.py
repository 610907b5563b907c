"""Debug: fraction of sync tiles whose exit depends on the seed (BH_X_DEPSTAT build)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from bench import Decoder, build_field  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "hacc"
spec, codes, book, stream = build_field(cfg, 0)
dec = Decoder(stream, "sync")
dec()
torch.cuda.synchronize()
raw = dec.rep.buf.cpu().numpy().view(np.uint64)
# DevReport: pad[0..3] are the last four u64 words
p3 = int(raw[15])
print(cfg, "tiles>0:", p3 >> 32, "dependent:", p3 & 0xffffffff, "maxlen", book.max_len)
