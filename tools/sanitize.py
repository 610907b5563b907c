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

# round-2 paths: device book, tuner on the fused path, sharded chunks, dequantize, ingest
import torch  # noqa: E402
from paper_2201_09118_b200 import ingest, quant, shard  # noqa: E402

codes = gaussian_codes(300_000, 1024, 8.0, seed=9)
book = ph.book_for_device(torch.from_numpy(codes.view(np.int16)).cuda(), codes.size, 16)
assert book.entries == ph.book_for(codes, 16).entries
st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
for mod in (ph.gap_decoder, ph.sync_decoder):
    assert np.array_equal(mod.decode(st, tuner_config=ph.TunerConfig(t_high=4)), codes)
for v in ("gap", "sync"):
    parts = sorted((o0, t.cpu().numpy().view(np.uint16)) for r in range(3)
                   for _, o0, t in shard.decode_shard([st], r, 3, v))
    assert np.array_equal(np.concatenate([p for _, p in parts]), codes)
q = (codes.astype(np.int64) - 512 + 32768).astype(np.uint16)
out = quant.dequantize(quant.QuantResult(q, np.array([5, 7000]), np.array([1.0, -2.0])), quant.QuantConfig(2.0 ** -8))
assert out.shape == codes.shape
ph.write_container(st, "/tmp/_san.huf2")
assert np.array_equal(ingest.decode_container("/tmp/_san.huf2", device_out=False), codes)
print("round-2 paths: ok", flush=True)
