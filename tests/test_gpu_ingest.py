"""Container -> device ingest: HUF2 files written by the
real reference (tests/golden/containers) and large files written here, read
straight into device memory through pinned double-buffered staging and
decoded; per-rank shard ingest reads only its span of the file and decodes
it with an unknown count (BH_STREAM_COUNT_IS_CAPACITY)."""

from pathlib import Path

import numpy as np
import pytest

from golden_cases import case

pytestmark = pytest.mark.gpu
CONTAINERS = Path(__file__).resolve().parent / "golden" / "containers"


@pytest.fixture(scope="module")
def ph():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    return ph


@pytest.mark.parametrize("path", sorted(CONTAINERS.glob("*.huf2")), ids=lambda p: p.stem)
def test_reference_containers(ph, path):
    from paper_2201_09118_b200 import ingest
    want = case(path.stem).symbols
    st = ingest.load_container_device(path, chunk_bytes=4096)  # many staging rounds
    assert np.array_equal(np.asarray(st.units), ph.read_container(path).units)
    variants = ["sync"] + (["gap"] if st.gap is not None else [])
    for v in variants:
        got = ingest.decode_container(path, v, device_out=False)
        assert np.array_equal(got, want), (path.stem, v)


@pytest.mark.parametrize("unit_bits,ups", [(32, 4), (16, 8), (8, 16)])
def test_large_file_and_shards(ph, tmp_path, unit_bits, ups):
    import torch
    from paper_2201_09118_b200 import ingest
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(6_000_000, 1024, 8.0, seed=unit_bits)
    st = ph.encode(codes, ph.book_for(codes, 16), ph.LayoutConfig(unit_bits, ups, 32), with_gap=True)
    path = tmp_path / "f.huf2"
    ph.write_container(st, path)
    for v in ("gap", "sync"):
        got = ingest.decode_container(path, v)
        assert torch.equal(got, torch.from_numpy(codes.view(np.int16)).cuda()), (unit_bits, v)
    for world in (1, 3, 8):
        parts = [ingest.ingest_shard(path, r, world, "gap") for r in range(world)]
        cat = np.concatenate([p[0].cpu().numpy().view(np.uint16) for p in parts])
        assert np.array_equal(cat, codes), (unit_bits, world)
    # a wrong header count surfaces like the reference (BadGap for gap, Truncated for sync)
    bad = ph.EncodedStream(layout=st.layout, units=st.units, total_bits=st.total_bits,
                           symbol_count=st.symbol_count + 1, codebook=st.codebook, gap=st.gap)
    ph.write_container(bad, path)
    with pytest.raises(ph.BadGap):
        ingest.ingest_shard(path, 0, 1, "gap")
    with pytest.raises(ph.BadGap):
        ingest.decode_container(path, "gap")


def test_shards_with_more_ranks_than_sequences(ph, tmp_path):
    from paper_2201_09118_b200 import ingest
    from paper_2201_09118_b200.synth import gaussian_codes
    codes = gaussian_codes(3000, 1024, 8.0, seed=5)
    st = ph.encode(codes, ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
    path = tmp_path / "small.huf2"
    ph.write_container(st, path)
    world = st.num_seqs + 3
    parts = [ingest.ingest_shard(path, r, world, v)[0] for v in ("gap",) for r in range(world)]
    cat = np.concatenate([p.cpu().numpy().view(np.uint16) for p in parts])
    assert np.array_equal(cat, codes)
