"""GPU: sequence-aligned chunks of one stream (the sharded multi-GPU decode,
SURVEY.md §8e) decode independently and concatenate to the whole stream's
output, for both decoders -- bit-exact against the generated symbols."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    return ph


@pytest.mark.parametrize("sigma,n", [(0.6, 3_000_000), (8.0, 2_000_000), (22.0, 1_500_000)])
@pytest.mark.parametrize("variant", ["gap", "sync"])
@pytest.mark.parametrize("nchunks", [1, 3, 7])
def test_chunked_decode_matches_whole_stream(ph, sigma, n, variant, nchunks):
    import torch
    from paper_2201_09118_b200 import _lib, shard
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200._pipeline import make_tune
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty
    from paper_2201_09118_b200.synth import gaussian_codes
    lib = _lib.load()
    codes = gaussian_codes(n, 1024, sigma, seed=11)
    book = ph.book_for(codes, 16)
    stream = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    st = ph.gap_decoder.entries_from_gap(stream)
    ph.gap_decoder.count_pass(stream, st)
    lay = stream.layout
    chunks = shard.chunk_stream(stream.total_bits, lay.subseq_bits, lay.subseqs_per_seq, stream.gap,
                                st.counts, nchunks)
    ds = device_stream(stream)
    var = _lib.VARIANT_GAP if variant == "gap" else _lib.VARIANT_SYNC
    got = np.empty(n, np.uint16)
    for ch in chunks:
        c = _lib.Stream(ds.c.words_dev + 4 * ch.word0, ch.total_bits, ch.n, lay.subseq_bits,
                        lay.subseqs_per_seq, book.symbol_width, ds.max_codes, ds.c.gap_dev + ch.sub0,
                        ds.c.table_dev, ch.first_entry, 0)
        tune = make_tune(max_len=book.max_len, min_len=book.min_len)
        wsb = lib.bh_workspace_bytes(C.byref(c), var, C.byref(tune))
        ws = torch.zeros(wsb, dtype=torch.uint8, device=ds.device)
        out = empty(max(ch.n, 1), np.uint16, ds.device)
        rep = DeviceReport(ds.device).init()
        check(lib.bh_decode_async(C.byref(c), var, C.byref(tune), out.data_ptr(), ws.data_ptr(), wsb, rep.ptr,
                                  stream_handle()), "chunk")
        check(rep.read().status, "chunk")
        got[ch.out0:ch.out0 + ch.n] = out[:ch.n].cpu().numpy().view(np.uint16)
    assert np.array_equal(got, codes)


@pytest.mark.parametrize("variant", ["gap", "sync"])
def test_decode_shard_single_symbol_book(variant):
    """A single-symbol book is incomplete (Kraft 1/2): the self-sync fused
    kernel declines it and a chunk has no staged fallback, so decode_shard
    enters such pieces through their gap bytes -- same symbols."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200 import shard
    codes = np.full(300_000, 7, np.uint16)
    st = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
    for world in (1, 3):
        parts = sorted((o0, t.cpu().numpy().view(np.uint16)) for r in range(world)
                       for _, o0, t in shard.decode_shard([st], r, world, variant))
        assert np.array_equal(np.concatenate([p for _, p in parts]), codes)


def test_decode_shard_refuses_layouts_the_fused_path_does_not_take():
    """Chunks decode on the fused kernel only: a layout whose 32-lane tile
    would exceed 16384 bits (subsequences of 1024 bits) is refused with a
    clear error instead of a failed launch; whole-stream decodes of it still
    work (staged pipeline)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200 import _lib, shard
    from paper_2201_09118_b200.device import device_stream
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(200_000, 1024, 3.0, seed=4)
    st = ph.encode(codes, ph.book_for(codes, 16), ph.LayoutConfig(32, 32, 8), with_gap=True)
    assert _lib.load().bh_fused_supported(device_stream(st).ref, _lib.VARIANT_GAP) == 0
    with pytest.raises(ValueError, match="fused decoder"):
        shard.decode_shard([st], 0, 2, "gap")
    assert np.array_equal(ph.gap_decoder.decode(st), codes)
