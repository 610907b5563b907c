"""K1 parity: the one-launch canonical table build (bh_table_build, csrc/table.cu
k_table_canon) against the general builder (bh_table_build_explicit: ranked
left-justified codes plus per-entry binary search, k_fill_luts) on the same
canonical books.  A canonical book given as explicit (code, length) pairs
must yield byte-identical decode tables (codebook.py:86-112, :209-233)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200 import _lib
    return torch, ph, _lib


def layout(max_codes: int) -> dict:
    """Byte offsets of csrc/common.cuh TableLayout."""
    a16 = lambda x: (x + 15) & ~15  # noqa: E731
    L = {"lut": 64}
    L["cnt"] = L["lut"] + 4 * 2048
    L["dlut8"] = a16(L["cnt"] + 2 * 2048)
    L["clut8"] = L["dlut8"] + 4 * 256
    L["wlut8"] = a16(L["clut8"] + 256)
    L["lut12"] = a16(L["wlut8"] + 16 * 256)
    L["clut12"] = L["lut12"] + 4 * 4096
    L["wlut12"] = a16(L["clut12"] + 2 * 4096)
    L["wlut3"] = a16(L["wlut12"] + 16 * 4096)
    L["cwin"] = a16(L["wlut3"] + 8 * 8192)
    L["len12"] = a16(L["cwin"] + 65536)
    L["lim"] = a16(L["len12"] + 4096)
    L["base"] = L["lim"] + 8 * 33
    L["lj"] = a16(L["base"] + 8 * 33)
    L["ljsym"] = a16(L["lj"] + 4 * max_codes)
    L["ljlen"] = a16(L["ljsym"] + 2 * max_codes)
    L["total"] = a16(L["ljlen"] + max_codes)
    return L


def books(ph):
    rng = np.random.default_rng(11)
    out = [ph.canonize({0: 1}, 16), ph.canonize({0: 1, 1: 1}, 16),
           ph.canonize({0: 1, 1: 3, 2: 3}, 8)]  # incomplete (Kraft < 1)
    lens = {i: i + 1 for i in range(31)}
    lens[31] = 31
    out.append(ph.canonize(lens, 16))  # 31-bit codes
    for bins, sigma in ((1024, 0.6), (1024, 8.0), (1024, 22.0), (4096, 0.2), (256, 3.0)):
        codes = np.clip(np.rint(rng.normal(0, sigma, 200_000)) + bins // 2, 0, bins - 1).astype(np.uint16)
        m = rng.random(codes.size) < 1e-3
        codes[m] = rng.integers(0, bins, int(m.sum()))
        out.append(ph.book_for(codes, 16))
    for alphabet in (3000, 9000):  # alphabets beyond one 1024-symbol block / beyond 4096
        w = 1.0 / np.arange(1, alphabet + 1)
        syms = rng.choice(alphabet, size=300_000, p=w / w.sum()).astype(np.uint16)
        out.append(ph.book_for(syms, 16))
    return out


def test_canonical_tables_match_general_builder(env):
    torch, ph, _lib = env
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    for book in books(ph):
        max_codes = max(len(book.entries), 1)
        L = layout(max_codes)
        assert lib.bh_table_bytes(max_codes) == L["total"]
        lens = book.length_bytes()
        codes, clens = book.encode_arrays()
        alphabet = len(lens)
        ld = torch.from_numpy(lens.copy()).cuda()
        cd = torch.from_numpy(codes[:alphabet].astype(np.uint32).view(np.int32).copy()).cuda()
        cl = torch.from_numpy(clens[:alphabet].copy()).cuda()
        fast = torch.zeros(L["total"], dtype=torch.uint8, device="cuda")
        gen = torch.zeros(L["total"], dtype=torch.uint8, device="cuda")
        _lib.check(lib.bh_table_build(ld.data_ptr(), alphabet, fast.data_ptr(), max_codes, st))
        _lib.check(lib.bh_table_build_explicit(cd.data_ptr(), cl.data_ptr(), alphabet, gen.data_ptr(),
                                               max_codes, st))
        f, g = fast.cpu().numpy(), gen.cpu().numpy()
        hf, hg = f[:64].view(np.uint32), g[:64].view(np.uint32)
        assert hf[0] == 0 and hg[0] == 1          # kind: canonical / explicit
        assert np.array_equal(hf[1:7], hg[1:7]), (hf[:7], hg[:7])  # max_len ncodes lut_bits alphabet status complete
        ncodes = int(hf[2])
        assert ncodes == len(book.entries)
        for name in ("lut", "cnt", "dlut8", "clut8", "wlut8", "lut12", "clut12", "wlut12", "wlut3", "cwin",
                     "len12"):
            nxt = {"lut": "cnt", "cnt": "dlut8", "dlut8": "clut8", "clut8": "wlut8", "wlut8": "lut12",
                   "lut12": "clut12", "clut12": "wlut12", "wlut12": "wlut3", "wlut3": "cwin",
                   "cwin": "len12", "len12": "lim"}[name]
            assert np.array_equal(f[L[name]:L[nxt]], g[L[name]:L[nxt]]), (name, book.max_len, ncodes)
        for name, w in (("lj", 4), ("ljsym", 2), ("ljlen", 1)):
            assert np.array_equal(f[L[name]:L[name] + w * ncodes], g[L[name]:L[name] + w * ncodes]), name
        # canonical limits (codebook.py:218-224 first_code recurrence, left-justified)
        lim = f[L["lim"]:L["lim"] + 8 * 33].view(np.uint64)
        counts = np.bincount(lens[lens > 0], minlength=33)
        code = 0
        for ln in range(1, 33):
            assert int(lim[ln]) == (code + int(counts[ln])) << (32 - ln)
            code = (code + int(counts[ln])) << 1


def _host_lengths(book):
    """codeword length at the front of a 32-bit window (0: none), by the
    canonical codes"""
    import bisect
    left = sorted(((code << (32 - ln)), ln, sym) for sym, (code, ln) in book.entries.items())
    keys = [k for k, _, _ in left]

    def at(w):
        i = bisect.bisect_right(keys, w) - 1
        if i < 0:
            return 0, 0
        k, ln, sym = left[i]
        return (ln, sym) if (w ^ k) >> (32 - ln) == 0 else (0, 0)
    return at


def test_count_and_three_codeword_table_semantics(env):
    """cwin (16-bit count table of the long-code path): for a book with every
    code >= 4 bits, entry v = (whole codewords of the zero-filled 16-bit
    window v) | (their end) << 3; all zero for books with shorter codes.
    wlut3 (13-bit three-codeword decode table): up to three whole codewords
    of 12 bits or less inside the 13-bit window, x = s0 | s1 << 16,
    y = s2 | len0 << 16 | end << 24 | 2n << 28 (0 when the first code is
    longer than 12 bits or ends past the window).  Both against a host walk
    of the canonical codes."""
    torch, ph, _lib = env
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(3)
    for sigma, want_built in ((8.0, True), (22.0, True), (0.6, False)):
        codes = np.clip(np.rint(rng.normal(0, sigma, 300_000)) + 512, 0, 1023).astype(np.uint16)
        book = ph.book_for(codes, 16)
        assert (book.min_len >= 4) == want_built
        mc = len(book.entries)
        L = layout(mc)
        lens = book.length_bytes()
        tab = torch.zeros(L["total"], dtype=torch.uint8, device="cuda")
        _lib.check(lib.bh_table_build(torch.from_numpy(lens.copy()).cuda().data_ptr(), len(lens), tab.data_ptr(), mc, st))
        t = tab.cpu().numpy()
        cwin = t[L["cwin"]:L["cwin"] + 65536]
        at = _host_lengths(book)
        if not want_built:
            assert not cwin.any()
        else:
            for v in list(range(0, 65536, 193)) + [0, 65535, 12345]:
                w0 = v << 16
                pos = n = 0
                while pos < 16:
                    ln, _ = at((w0 << pos) & 0xffffffff)
                    if ln == 0 or pos + ln > 16:
                        break
                    pos += ln
                    n += 1
                assert cwin[v] == (n | (pos << 3)), (sigma, v, cwin[v], n, pos)
            w3 = t[L["wlut3"]:L["wlut3"] + 8 * 8192].view(np.uint32).reshape(-1, 2)
            for v in list(range(0, 8192, 37)) + [0, 8191]:
                w0 = v << 19
                pos = n = l0 = 0
                syms = []
                while n < 3 and pos < 13:
                    ln, sym = at((w0 << pos) & 0xffffffff)
                    if ln == 0 or ln > 12 or pos + ln > 13:
                        break
                    l0 = l0 or ln
                    syms.append(sym)
                    pos += ln
                    n += 1
                syms += [0] * (3 - len(syms))
                want_x = syms[0] | (syms[1] << 16)
                want_y = (syms[2] | (l0 << 16) | (pos << 24) | ((2 * n) << 28)) if n else 0
                assert (int(w3[v, 0]), int(w3[v, 1])) == (want_x, want_y), (sigma, v)
