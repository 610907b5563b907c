#!/usr/bin/env python
"""Huffman decode benchmark (BASELINE.json metric: decoded GB/s per B200 and at
2/4/8 GPUs, against the reference CPU decoder).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config hacc|hurricane|nyx|...|multifield] [--variant gap|sync]

Workload.  N = 1: the HACC-shaped field (BASELINE config 4, 280,953,867
uint16 quantization codes, 1024 bins, sigma 8 -- the largest single-GPU
config), gap-array decoder.  N > 1: the multi-field batch
(config 5: CESM / RTM / QMCPACK-shaped fields) split over the ranks
(strong scaling, no collective on the data path).  Synthetic codes from
``paper_2201_09118_b200/synth.py`` (the §8d generator).

One step = one complete decode through the C ABI with the input resident in
HBM: K1 (bh_table_build from the codebook's length bytes) + the fused decoder
(bh_decode_async), both inside the step's CUDA events.  A 256 MiB buffer is
rewritten between steps (outside the events), and the payload / output are
larger than the 126 MB L2 anyway.

Extra keys: ``roofline`` (the fused decode kernel: algorithmic bytes per launch
over its own CUDA-event duration, vs MEASURED_PEAKS.json), ``e2e`` (same
metric through the C ABI from pinned host buffers, H2D of payload + gap +
lengths and D2H of the output inside the timed region), ``cpu_baseline``
(the reference parhuff decoder on this host's cores, bounded sample),
``clocks`` (nvidia-smi during the timed region), ``variants_gbs_per_gpu``
(gap, self-sync, the in-run cuSZ-style coarse decoder K8) and
``gpu_launches``.

``--impl reference`` times the unmodified reference decoder (parhuff from
baseline/_ref, its own encoder and codebook builder for the input -- nothing
of this repository's library is loaded) on a bounded sample of the same
workload, and prints the same config.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N processes (one GPU each).
"""

from __future__ import annotations

import argparse
import ctypes as C
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Huffman decode GB/s (decoded bytes)"
FLUSH_BYTES = 256 << 20
MULTI_FIELDS = ("cesm", "rtm", "qmcpack")
LAYOUT = (32, 4, 32)  # DEFAULT_LAYOUT: 32-bit units, 4 per subsequence, 32 subsequences per sequence


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, help="hacc (N=1 default), multifield (N>1 default), hurricane, ...")
    ap.add_argument("--variant", default="gap", choices=["gap", "sync"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e/variants (profiling runs)")
    a = ap.parse_args()
    if a.config is None:
        a.config = "multifield" if a.gpus > 1 else "hacc"
    if a.warmup < 3:
        ap.error("--warmup must be >= 3")
    return a


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 outside torchrun: one process per GPU via torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_synth():
    """The §8d generator module by file path (no package import: the
    reference arm must not load this repository's library)."""
    if "bh_synth" in sys.modules:
        return sys.modules["bh_synth"]
    spec = importlib.util.spec_from_file_location("bh_synth", ROOT / "paper_2201_09118_b200" / "synth.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules["bh_synth"] = mod  # dataclasses resolve their module through sys.modules
    spec.loader.exec_module(mod)
    return mod


def config_dict(args, world: int) -> dict:
    """The workload description -- identical in both arms (generator level only)."""
    synth = load_synth()
    dec = "gap-array" if args.variant == "gap" else "self-sync"
    common = {"variant": args.variant, "layout": "32-bit units, 4 per subsequence, 32 per sequence",
              "data": "synthetic cuSZ-style quant codes: clip(rint(N(0, sigma)) + bins/2) (SURVEY 8d)",
              "l2": "256 MiB buffer rewritten between steps (outside the per-step events); payload and "
                    "output exceed the 126 MB L2"}
    if args.config == "multifield":
        specs = [synth.FIELDS[k] for k in MULTI_FIELDS]
        return {"workload": "multi-field batch (" + ", ".join(f"{s.name} {s.n} codes sigma {s.sigma}" for s in specs)
                            + f"), 1024 bins, {dec} decoder",
                "fields": [s.name for s in specs], "n_symbols": sum(s.n for s in specs),
                "parallelism": f"batch cut at sequence boundaries into {world} equal spans (one per GPU), "
                               "no collective", **common}
    s = synth.FIELDS[args.config]
    par = "one field per GPU, no collective" if world > 1 else "1 GPU"
    return {"workload": f"{s.name} ({s.n} uint16 quant codes, {s.bins} bins, sigma {s.sigma}"
                        + (f", uniform floor {s.eps}" if s.eps else "") + f"), {dec} decoder",
            "field": s.name, "n_symbols": s.n, "bins": s.bins, "sigma": s.sigma, "parallelism": par, **common}


def alg_bytes(total_bits: int, n: int, nsub: int, variant: str) -> int:
    """payload words + decoded output (+ gap bytes for the gap variant)."""
    return 4 * (-(-total_bits // 32)) + 2 * n + (nsub if variant == "gap" else 0)


# --------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# --------------------------------------------------------------------------

_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
            0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
            0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.03)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [r for r in rows if not (r[2] & 0x1)] or rows
        reasons = sorted({name for r in loaded for bit, name in _REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


# --------------------------------------------------------------------------
# B200 arm: device-resident decode (K1 + fused decoder per step)
# --------------------------------------------------------------------------

class Piece:
    """One bh_decode_async call on a (chunk of a) stream, with its own
    workspace, report and K1 table build from device length bytes."""

    def __init__(self, field_stream, variant: str, chunk=None, ctas: int = 0):
        import torch
        from paper_2201_09118_b200 import _lib
        from paper_2201_09118_b200._pipeline import make_tune
        from paper_2201_09118_b200.device import DeviceReport, device_stream, empty
        self.lib = lib = _lib.load()
        ds = device_stream(field_stream)
        book = field_stream.codebook
        lay = field_stream.layout
        self.ds = ds
        self.variant = variant
        self.var = _lib.VARIANT_GAP if variant == "gap" else _lib.VARIANT_SYNC
        lens = book.length_bytes()
        self.lens_d = torch.from_numpy(lens.copy()).to(ds.device)
        self.alphabet = len(lens)
        self.max_codes = ds.max_codes
        self.table = torch.empty(lib.bh_table_bytes(self.max_codes), dtype=torch.uint8, device=ds.device)
        if chunk is None:
            self.c = _lib.Stream(ds.c.words_dev, field_stream.total_bits, field_stream.symbol_count,
                                 lay.subseq_bits, lay.subseqs_per_seq, book.symbol_width, self.max_codes,
                                 ds.c.gap_dev, self.table.data_ptr(), 0, 0)
            self.n, self.tb, self.nsub, self.out0 = field_stream.symbol_count, field_stream.total_bits, \
                field_stream.num_subseqs, 0
        else:
            self.c = _lib.Stream(ds.c.words_dev + 4 * chunk.word0, chunk.total_bits, chunk.n, lay.subseq_bits,
                                 lay.subseqs_per_seq, book.symbol_width, self.max_codes,
                                 ds.c.gap_dev + chunk.sub0, self.table.data_ptr(), chunk.first_entry, 0)
            self.n, self.tb, self.nsub, self.out0 = chunk.n, chunk.total_bits, chunk.nsub, chunk.out0
        self.tune = make_tune(max_len=book.max_len, min_len=book.min_len)
        self.tune.ctas = int(ctas)
        self.out = empty(self.n, np.uint16, ds.device)
        self.wsb = lib.bh_workspace_bytes(C.byref(self.c), self.var, C.byref(self.tune))
        self.ws = torch.zeros(max(self.wsb, 256), dtype=torch.uint8, device=ds.device)
        self.rep = DeviceReport(ds.device).init()

    def table_build(self, st: int):
        from paper_2201_09118_b200._lib import check
        check(self.lib.bh_table_build(self.lens_d.data_ptr(), self.alphabet, self.table.data_ptr(),
                                      self.max_codes, st), "table")

    def decode(self, st: int):
        from paper_2201_09118_b200._lib import check
        check(self.lib.bh_decode_async(C.byref(self.c), self.var, C.byref(self.tune), self.out.data_ptr(),
                                       self.ws.data_ptr(), self.wsb, self.rep.ptr, st), "decode")

    def alg_bytes(self) -> int:
        return alg_bytes(self.tb, self.n, self.nsub, self.variant)


def run_steps(pieces, steps: int, warmup: int, flush, split: bool = True):
    """Per step: [e0] K1 of every piece [e1] decode of every piece [e2] on
    one stream per piece (several pieces run concurrently), L2 flush between
    steps outside the events.  Returns per-step (step_ms, decode_ms) where
    decode_ms brackets the decode kernels alone.  split=False records no e1:
    each piece's decode then follows its K1 directly on its stream (launched
    with programmatic stream serialisation, its CTAs start while K1 drains),
    which is the step as a caller runs it; decode_ms is then 0."""
    import torch
    main = torch.cuda.current_stream()
    streams = [main] + [torch.cuda.Stream() for _ in pieces[1:]]

    def step(e0=None, e1=None, e2=None):
        if e0 is not None:
            e0.record(main)
        for p, s in zip(pieces, streams):
            if s is not main:
                s.wait_stream(main)
            p.table_build(s.cuda_stream)
        if e1 is not None and split:
            for s in streams[1:]:
                main.wait_stream(s)
            e1.record(main)
            for s in streams[1:]:
                s.wait_stream(main)
        for p, s in zip(pieces, streams):
            p.decode(s.cuda_stream)
        for s in streams[1:]:
            main.wait_stream(s)
        if e2 is not None:
            e2.record(main)

    for _ in range(warmup):
        step()
        flush()
    torch.cuda.synchronize()
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(steps)]
    for e in ev:
        step(*e)
        flush()
    torch.cuda.synchronize()
    return [(a.elapsed_time(c), b.elapsed_time(c) if split else 0.0) for a, b, c in ev]


def count_launches(fn) -> int:
    """Kernels of this library launched by one call (untimed pass)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    n = 0
    for e in prof.events():
        name = e.name or ""
        if e.device_type == torch.autograd.DeviceType.CUDA and ("bh::" in name or name.startswith("k_")):
            n += 1
    return n


def e2e_measure(items, variant: str, steps: int, flush):
    """The public C-ABI call sequence from pinned host buffers, every step
    inside the timed region: H2D of each piece's payload words, gap bytes and
    length bytes, K1 table build, decode, D2H of the decoded symbols.  Two
    calls are in flight, each with its own device buffers, workspace, report
    and CUDA stream (the ABI is stream-ordered with no hidden
    synchronisation), so one call's H2D and decode overlap the previous
    call's D2H on the other copy engine.  Each step starts with an L2 flush on
    its stream.  items: [(field_stream, chunk or None)].  Returns (ms per step
    -- median of three timed regions --, outputs of the last step, H2D bytes,
    D2H bytes, per-region ms)."""
    import torch
    from paper_2201_09118_b200 import _lib
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200._pipeline import make_tune
    from paper_2201_09118_b200.device import DeviceReport, empty
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    var = _lib.VARIANT_GAP if variant == "gap" else _lib.VARIANT_SYNC

    class HostPiece:
        def __init__(self, fs, ch):
            lay = fs.layout
            if ch is None:
                w0, tb, s0, ns, n, fe = 0, fs.total_bits, 0, fs.num_subseqs, fs.symbol_count, 0
            else:
                w0, tb, s0, ns, n, fe = ch.word0, ch.total_bits, ch.sub0, ch.nsub, ch.n, ch.first_entry
            self.nwords = -(-tb // 32)
            units = fs.units.view(np.int32)
            self.units_h = torch.from_numpy(units[w0:w0 + self.nwords].copy()).pin_memory()
            self.gap_h = torch.from_numpy(fs.gap[s0:s0 + ns].copy()).pin_memory()
            lens = fs.codebook.length_bytes()
            self.lens_h = torch.from_numpy(lens.copy()).pin_memory()
            self.max_codes = max(len(fs.codebook.entries), 1)
            self.args = (tb, n, lay.subseq_bits, lay.subseqs_per_seq, fs.codebook.symbol_width, fe)
            self.n = n
            self.tune = make_tune(max_len=fs.codebook.max_len, min_len=fs.codebook.min_len)

    hp = [HostPiece(fs, ch) for fs, ch in items]

    class Ctx:
        def __init__(self):
            self.st = torch.cuda.Stream(device=dev)
            self.bufs = []
            for h in hp:
                words = torch.zeros(h.nwords + _lib.WORD_PAD, dtype=torch.int32, device=dev)
                gap_d = torch.empty(max(len(h.gap_h), 1), dtype=torch.uint8, device=dev)
                lens_d = torch.empty(len(h.lens_h), dtype=torch.uint8, device=dev)
                table = torch.empty(lib.bh_table_bytes(h.max_codes), dtype=torch.uint8, device=dev)
                out_d = empty(h.n, np.uint16, dev)
                out_h = torch.empty(max(h.n, 1), dtype=torch.int16).pin_memory()
                tb, n, sb, sps, sw, fe = h.args
                cs = _lib.Stream(words.data_ptr(), tb, n, sb, sps, sw, h.max_codes, gap_d.data_ptr(),
                                 table.data_ptr(), fe, 0)
                wsb = lib.bh_workspace_bytes(C.byref(cs), var, C.byref(h.tune))
                ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
                lib.bh_workspace_reset(ws.data_ptr(), ws.numel(), stream_handle(self.st))
                rep = DeviceReport(dev).init()
                self.bufs.append((h, words, gap_d, lens_d, table, out_d, out_h, cs, wsb, ws, rep))

        def step(self):
            with torch.cuda.stream(self.st):
                st = stream_handle(self.st)
                flush()
                for h, words, gap_d, lens_d, table, out_d, out_h, cs, wsb, ws, rep in self.bufs:
                    words[:h.nwords].copy_(h.units_h, non_blocking=True)
                    gap_d[:len(h.gap_h)].copy_(h.gap_h, non_blocking=True)
                    lens_d.copy_(h.lens_h, non_blocking=True)
                    check(lib.bh_table_build(lens_d.data_ptr(), len(h.lens_h), table.data_ptr(), h.max_codes, st),
                          "table")
                    check(lib.bh_decode_async(C.byref(cs), var, C.byref(h.tune), out_d.data_ptr(), ws.data_ptr(),
                                              wsb, rep.ptr, st), "decode")
                    out_h[:h.n].copy_(out_d[:h.n], non_blocking=True)

    ctx = [Ctx(), Ctx()]
    torch.cuda.synchronize()
    for i in range(4):  # warm-up
        ctx[i % 2].step()
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    runs = []
    for _ in range(3):  # three timed regions of `steps` calls; the median is reported
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        for c in ctx:
            c.st.wait_event(a)
        for i in range(steps):
            ctx[i % 2].step()
        for c in ctx:
            main.wait_stream(c.st)
        b.record(main)
        torch.cuda.synchronize()
        runs.append(a.elapsed_time(b) / steps)
    last = ctx[(steps - 1) % 2]
    outs = []
    for h, *_, out_h, cs, wsb, ws, rep in last.bufs:
        check(rep.read().status, "e2e decode")
        outs.append(out_h[:h.n].numpy().view(np.uint16))
    bi = sum(4 * h.nwords + len(h.gap_h) + len(h.lens_h) for h in hp)
    bo = sum(2 * h.n for h in hp)
    return statistics.median(runs), outs, bi, bo, runs


def coarse_baseline(ph, codes, book, stream, flush):
    """cuSZ-style coarse-grained decoder (K8): best chunk of the SURVEY §8d
    sweep 2^8 .. 2^14 symbols per thread."""
    import torch
    from paper_2201_09118_b200 import _lib
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty, h2d
    from paper_2201_09118_b200.encoder import encode_device
    lib = _lib.load()
    ds = device_stream(stream)
    sd = h2d(codes, ds.device)
    want = torch.from_numpy(codes.view(np.int16)).to(ds.device)
    best, sweep = None, {}
    for lg in range(8, 15):
        chunk = 1 << lg
        _, _, _, offs = encode_device(sd, len(codes), book, ph.DEFAULT_LAYOUT, False, chunk)
        out = empty(len(codes), np.uint16, ds.device)
        rep = DeviceReport(ds.device).init()

        def fn():
            check(lib.bh_coarse_decode(ds.ref, offs.data_ptr(), chunk, out.data_ptr(), rep.ptr,
                                       stream_handle()), "coarse")
        fn()
        torch.cuda.synchronize()
        check(rep.read().status, "coarse")
        assert torch.equal(out[: len(codes)], want), f"coarse decode mismatch (chunk {chunk})"
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            flush()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        v = 2 * len(codes) / (statistics.median(ts) / 1e3) / 1e9
        sweep[chunk] = round(v, 2)
        if best is None or v > best["value"]:
            best = {"value": v, "chunk": chunk,
                    "alg_bytes": 4 * (-(-stream.total_bits // 32)) + 8 * (-(-len(codes) // chunk)) + 2 * len(codes)}
        del offs, out
    best["sweep_gbs"] = sweep
    return best


# --------------------------------------------------------------------------
# CPU reference (baseline/_ref parhuff: its own codebook builder and encoder)
# --------------------------------------------------------------------------

def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    ref = ROOT / "baseline" / "_ref"
    if ref.exists() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import parhuff  # noqa: F401
    return parhuff


def ref_book(parhuff, codes):
    """parhuff.canonize(parhuff.build_lengths(histogram)) of the full field."""
    counts = np.bincount(codes.astype(np.int64))
    nz = np.nonzero(counts)[0]
    return parhuff.canonize(parhuff.build_lengths({int(s): int(counts[s]) for s in nz}), symbol_width=16)


def ref_sample(parhuff, codes, book, n):
    return parhuff.encode(codes[:n], book, parhuff.LayoutConfig(*LAYOUT), with_gap=True)


class RefWorkload:
    """Bounded samples of the workload's fields, encoded by the reference
    itself, decoded by the stock parhuff decoder on all host cores."""

    def __init__(self, parhuff, fields, variant: str, per_call_s: float):
        from parhuff import gap_decoder, sync_decoder
        self.dec = gap_decoder if variant == "gap" else sync_decoder
        self.cores = len(os.sched_getaffinity(0))
        self.items = []
        total_n = sum(len(c) for _, c in fields)
        probe = []
        for name, codes in fields:
            book = ref_book(parhuff, codes)
            probe.append((name, codes, book))
        # JIT warm-up and rate probe on a small sample of the first field
        tiny = ref_sample(parhuff, probe[0][1], probe[0][2], 20_000)
        self.dec.decode(tiny, workers=self.cores)
        t0 = time.perf_counter()
        self.dec.decode(tiny, workers=self.cores)
        rate = 20_000 / max(time.perf_counter() - t0, 1e-6)
        budget = int(max(100_000, rate * per_call_s))
        for name, codes, book in probe:
            n = int(min(len(codes), max(20_000, budget * len(codes) // total_n)))
            self.items.append((name, n, codes, ref_sample(parhuff, codes, book, n)))
        self.n = sum(n for _, n, _, _ in self.items)

    def __call__(self):
        return [self.dec.decode(s, workers=self.cores) for _, _, _, s in self.items]

    def check(self, outs):
        for (name, n, codes, _), o in zip(self.items, outs):
            assert np.array_equal(o, codes[:n]), f"reference decode mismatch on {name}"

    def sample(self) -> str:
        parts = ", ".join(f"first {n} of {len(c)} symbols of {name}" for name, n, c, _ in self.items)
        return f"parhuff.{self.dec.__name__.split('.')[-1]}.decode(workers={self.cores}) on {parts}"


def workload_fields(args):
    synth = load_synth()
    keys = MULTI_FIELDS if args.config == "multifield" else (args.config,)
    return [(synth.FIELDS[k].name, synth.field_codes(synth.FIELDS[k])) for k in keys]


def cpu_baseline_leg(args, fields, budget_s=20.0, reps=3):
    """cpu_baseline of the B200 arm: the reference (else the C oracle port)
    on a bounded sample of the same workload, median of `reps` calls."""
    try:
        parhuff = import_reference()
        w = RefWorkload(parhuff, fields, args.variant, budget_s / reps)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            outs = w()
            times.append(time.perf_counter() - t0)
        w.check(outs)
        v = 2 * w.n / statistics.median(times) / 1e9
        return {"value": v, "unit": "GB/s", "cores": w.cores, "kind": "reference",
                "sample": w.sample() + f", median of {reps}"}
    except Exception as e:  # reference unavailable: the C oracle port (test infrastructure)
        from oracle import oracle
        import paper_2201_09118_b200 as ph
        name, codes = fields[0]
        n = min(len(codes), 5_000_000)
        st = ph.encode(codes[:n], ph.book_for(codes, 16), ph.DEFAULT_LAYOUT, with_gap=True)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            oracle.gap_decode(st) if args.variant == "gap" else oracle.sync_decode(st)
            times.append(time.perf_counter() - t0)
        return {"value": 2 * n / statistics.median(times) / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
                "sample": f"C oracle port ({type(e).__name__}: reference unavailable), first {n} symbols of {name}"}


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    parhuff = import_reference()
    fields = workload_fields(args)
    per_step = max(0.2, 120.0 / max(args.steps + args.warmup, 1))
    w = RefWorkload(parhuff, fields, args.variant, per_step)
    for _ in range(args.warmup):
        w()
    times, outs = [], None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        outs = w()
        times.append(time.perf_counter() - t0)
    w.check(outs)
    total = sum(times)
    value = 2 * w.n * args.steps / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.config == "multifield" else "weak",
        "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": config_dict(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": w.cores, "kind": "reference",
                         "sample": w.sample() + " per step"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# main (B200 arm)
# --------------------------------------------------------------------------

def build_workload(args, rank: int, world: int):
    """Encode the workload's fields on the GPU; returns (fields, items) where
    items = [(field index, chunk or None)] is this rank's share."""
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200 import shard
    import torch
    fields = []
    for name, codes in workload_fields(args):
        # the encode side on the device: histogram -> build_lengths -> canonize -> pack + gap
        book = ph.book_for_device(torch.from_numpy(codes.view(np.int16)).cuda(), codes.size, 16)
        st = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
        fields.append((name, codes, book, st))
    if args.config != "multifield":
        if world > 1:  # weak scaling: every rank its own field (different seed)
            synth = load_synth()
            from dataclasses import replace
            spec = replace(synth.FIELDS[args.config], seed=synth.FIELDS[args.config].seed + rank)
            codes = synth.field_codes(spec)
            book = ph.book_for_device(torch.from_numpy(codes.view(np.int16)).cuda(), codes.size, 16)
            fields = [(spec.name, codes, book, ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True))]
        return fields, [(0, None)]
    spans = shard.balanced_pieces([f[3].num_seqs for f in fields], world)[rank]
    items = []
    for fi, q0, q1 in spans:
        st = fields[fi][3]
        if q0 == 0 and q1 == st.num_seqs:
            items.append((fi, None))
            continue
        s = ph.gap_decoder.entries_from_gap(st)
        ph.gap_decoder.count_pass(st, s)  # per-subsequence counts (encode-side metadata)
        lay = st.layout
        items.append((fi, shard.piece_chunk(st.total_bits, lay.subseq_bits, lay.subseqs_per_seq, st.gap,
                                            s.counts, q0, q1)))
    return fields, items


def main():
    args = parse()
    rank, local, world = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args)
    import torch
    # BH_BENCH_SHARED_DEVICE=1 (testing the N-rank code path on a one-GPU
    # box): every rank on cuda:0, gloo for the barriers and reductions
    shared = os.environ.get("BH_BENCH_SHARED_DEVICE") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2201_09118_b200 as ph

    fields, items = build_workload(args, rank, world)
    ctas = torch.cuda.get_device_properties(local).multi_processor_count
    tot_bits = sum((ch.total_bits if ch else fields[fi][3].total_bits) for fi, ch in items)
    pieces = []
    for fi, ch in items:
        tb = ch.total_bits if ch else fields[fi][3].total_bits
        share = max(1, round(ctas * tb / tot_bits)) if len(items) > 1 else 0  # concurrent pieces: one wave
        pieces.append(Piece(fields[fi][3], args.variant, ch, share))
    flush_buf = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    def flush():
        flush_buf.zero_()

    # correctness before timing: every piece bit-exact against its codes
    run_steps(pieces, 1, 3, flush)
    for (fi, ch), p in zip(items, pieces):
        r = p.rep.read()
        from paper_2201_09118_b200._lib import check
        check(r.status, "bench decode")
        codes = fields[fi][1]
        want = codes if ch is None else codes[ch.out0:ch.out0 + ch.n]
        assert torch.equal(p.out[:p.n], torch.from_numpy(want.view(np.int16)).cuda()), "decode mismatch"

    def one_step():
        st = torch.cuda.current_stream().cuda_stream
        for p in pieces:
            p.table_build(st)
            p.decode(st)
    launches = count_launches(one_step)

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        if world > 1:
            torch.distributed.barrier()
        # the step as a caller runs it (K1 then decode, no event between them)
        times = run_steps(pieces, args.steps, args.warmup, flush, split=False)
        if world > 1:
            torch.distributed.barrier()
        # the same steps with an event between K1 and decode: the decode
        # kernel's own duration (roofline) and K1's share
        stimes = run_steps(pieces, args.steps, args.warmup, flush, split=True)
        if world > 1:
            torch.distributed.barrier()
    for p in pieces:
        ph._lib.check(p.rep.read().status, "bench decode")
    step_ms = sum(t[0] for t in times)
    dec_ms = sum(t[1] for t in stimes)
    sstep_ms = sum(t[0] for t in stimes)
    my_alg = sum(p.alg_bytes() for p in pieces)
    my_n = sum(p.n for p in pieces)
    t = torch.tensor([step_ms, dec_ms, float(my_alg), float(my_n), sstep_ms], dtype=torch.float64, device="cuda")
    tot_alg, tot_n = float(my_alg), float(my_n)
    if world > 1:
        tmax, tsum = t.clone(), t.clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(tsum, op=torch.distributed.ReduceOp.SUM)
        step_ms, dec_ms, sstep_ms = float(tmax[0].item()), float(tmax[1].item()), float(tmax[4].item())
        tot_alg, tot_n = float(tsum[2].item()), float(tsum[3].item())
    value = 2 * tot_n * args.steps / (step_ms / 1e3) / 1e9

    peak, peak_src = measured_peak()
    dec_avg = dec_ms / args.steps
    achieved = tot_alg / world / (dec_avg / 1e3) / 1e9  # per GPU, decode kernel(s) alone
    traffic = None
    nc = ROOT / "profiles" / "ncu_summary.json"
    if nc.exists() and len(pieces) == 1:
        try:
            traffic = json.loads(nc.read_text()).get(args.config, {}).get(args.variant, {}).get(
                "dram_bytes_per_launch")
        except Exception:
            traffic = None
    st0 = fields[0][3]
    line = {
        "impl": "b200", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.config == "multifield" else "weak",
        "vs_baseline": None, "dtype": "u32 words -> u16 symbols", "data": "synthetic",
        "config": config_dict(args, world),
        "stream": {"total_bits": [f[3].total_bits for f in fields],
                   "compression_ratio": [round(16 * f[3].symbol_count / max(f[3].total_bits, 1), 3) for f in fields],
                   "max_len": [f[2].max_len for f in fields], "pieces_on_rank0": len(pieces)},
        "step": "K1 table build (bh_table_build) + fused decode (bh_decode_async), device-resident",
        "roofline": {"bound": "hbm", "kernel": f"k_fused2<{args.variant}> (fused decode)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "alg_bytes_per_launch": tot_alg / world, "avg_launch_ms": dec_avg, "peak_source": peak_src,
                     "k1_ms_per_step": (sstep_ms - dec_ms) / args.steps,
                     "split_step_ms": sstep_ms / args.steps,
                     "timing": "value: K1 + decode back to back per step (events around the step only); "
                               "avg_launch_ms and k1_ms_per_step: a second pass of the same steps with an "
                               "event between K1 and the decode",
                     "whole_step_frac": tot_alg / world / (step_ms / args.steps / 1e3) / 1e9 / peak},
        "clocks": clk.summary(),
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
    }

    if not args.no_extras:
        ksteps = max(3, min(args.steps, 20))
        if world > 1:
            torch.distributed.barrier()
        ems, outs, bi, bo, eruns = e2e_measure([(fields[fi][3], ch) for fi, ch in items], args.variant, ksteps,
                                               flush)
        for (fi, ch), o in zip(items, outs):
            codes = fields[fi][1]
            assert np.array_equal(o, codes if ch is None else codes[ch.out0:ch.out0 + ch.n]), "e2e mismatch"
        te = torch.tensor([ems, float(bi), float(bo)], dtype=torch.float64, device="cuda")
        if world > 1:  # whole job: every rank's share, slowest rank's time
            tm, ts = te.clone(), te.clone()
            torch.distributed.all_reduce(tm, op=torch.distributed.ReduceOp.MAX)
            torch.distributed.all_reduce(ts, op=torch.distributed.ReduceOp.SUM)
            ems, bi, bo = float(tm[0].item()), float(ts[1].item()), float(ts[2].item())
        line["e2e"] = {"value": 2 * tot_n / (ems / 1e3) / 1e9, "unit": "GB/s",
                       "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(bo), "steps": ksteps,
                       "ms_per_step": ems, "in_flight": 2, "regions": 3, "ms_per_step_regions": eruns,
                       "call": "bh_table_build + bh_decode_async from pinned host buffers"}
        if len(items) == 1 and items[0][1] is None:
            # the other decoder and the in-run coarse-grained cuSZ-style baseline
            variants = {args.variant: 2 * my_n * args.steps / (step_ms / 1e3) / 1e9}
            other = "sync" if args.variant == "gap" else "gap"
            op = Piece(fields[0][3], other)
            ot = run_steps([op], 20, 3, flush)
            variants[other] = 2 * op.n / (statistics.mean(t[0] for t in ot) / 1e3) / 1e9
            variants[other + "_decode_kernel"] = 2 * op.n / (statistics.mean(t[1] for t in ot) / 1e3) / 1e9
            variants["coarse_cusz"] = coarse_baseline(ph, fields[0][1], fields[0][2], fields[0][3], flush)
            line["variants_gbs_per_gpu"] = variants
            line["speedup_vs_coarse"] = {k: v / variants["coarse_cusz"]["value"]
                                         for k, v in variants.items() if k != "coarse_cusz"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_leg(args, [(f[0], f[1]) for f in fields])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
