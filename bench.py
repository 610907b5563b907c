#!/usr/bin/env python
"""Huffman decode benchmark (BASELINE.json metric: decoded GB/s per B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config hurricane] [--variant gap|sync]

One step = one full decode of the configured field (synthetic cuSZ-style
quantization codes) through ``bh_decode_async`` with the input
already resident in HBM and the output preallocated.  Each step is bracketed by
CUDA events on the decode stream; a 256 MiB buffer is rewritten between steps
(outside the events) so every step starts with a cold L2.  With N GPUs
(torchrun) every rank decodes its own field (different seed) -- weak scaling,
no collective on the data path; the reported time is the max over ranks.

Extra keys: ``roofline`` (dominant kernel, algorithmic bytes per launch over
its CUDA-event duration vs MEASURED_PEAKS.json), ``e2e`` (same metric through
the public C-ABI call with pinned host buffers, H2D + table build + decode +
D2H inside the timed region), ``cpu_baseline`` (the reference package on this
host's cores), ``clocks`` (nvidia-smi during the timed region), ``variants``
(gap / sync / cuSZ-style coarse baseline).

``--impl reference`` times the unmodified reference decoder (parhuff from
baseline/_ref) on the host's cores on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time
import warnings
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
warnings.filterwarnings("ignore", message=".*Profiler clears events.*")
sys.path.insert(0, str(ROOT))

METRIC = "Huffman decode GB/s (decoded bytes)"
FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="hurricane")
    ap.add_argument("--variant", default="gap", choices=["gap", "sync"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e/variants (profiling runs)")
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--graph", type=int, default=1, help="replay the decode as a captured CUDA graph")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------
# workload
# --------------------------------------------------------------------------

def build_field(config: str, rank: int):
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200.synth import FIELDS, field_codes
    spec = FIELDS[config]
    spec = replace(spec, seed=spec.seed + rank)
    codes = field_codes(spec)
    book = ph.book_for(codes, 16)
    stream = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
    return spec, codes, book, stream


def alg_bytes(stream, variant: str) -> int:
    """payload words + decoded output (+ gap bytes for the gap variant)."""
    b = 4 * (-(-stream.total_bits // 32)) + 2 * stream.symbol_count
    if variant == "gap":
        b += stream.num_subseqs
    return b


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
        self.out = ""
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
# device-resident timing
# --------------------------------------------------------------------------

class Decoder:
    """Preallocated bh_decode_async call for one stream."""

    def __init__(self, stream, variant: str, fused: bool = True, tuner=None):
        import torch
        from paper_2201_09118_b200 import _lib
        from paper_2201_09118_b200._pipeline import make_tune
        from paper_2201_09118_b200.device import DeviceReport, device_stream, empty
        self.torch = torch
        self.lib = _lib.load()
        self.ds = device_stream(stream)
        self.variant = _lib.VARIANT_GAP if variant == "gap" else _lib.VARIANT_SYNC
        self.tune = make_tune(3584, tuner, False, fused, max_len=stream.codebook.max_len)
        self.out = empty(stream.symbol_count, np.uint16, self.ds.device)
        self.wsb = self.lib.bh_workspace_bytes(self.ds.ref, self.variant, C.byref(self.tune))
        self.ws = torch.empty(max(self.wsb, 256), dtype=torch.uint8, device=self.ds.device)
        from paper_2201_09118_b200._lib import stream_handle
        self.lib.bh_workspace_reset(self.ws.data_ptr(), self.ws.numel(), stream_handle())
        self.rep = DeviceReport(self.ds.device).init()

    def __call__(self):
        from paper_2201_09118_b200._lib import check, stream_handle
        check(self.lib.bh_decode_async(self.ds.ref, self.variant, C.byref(self.tune), self.out.data_ptr(),
                                       self.ws.data_ptr(), self.wsb, self.rep.ptr, stream_handle()), "decode")

    def status(self):
        return self.rep.read()


def time_steps(fn, steps: int, warmup: int, flush, events=True):
    """Per-step CUDA-event times (ms) with an L2 flush between steps."""
    import torch
    for _ in range(warmup):
        fn()
        flush()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
        flush()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def count_launches(fn) -> int:
    """Kernels launched by one call that come from our library (untimed pass)."""
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


def e2e_measure(stream, book, variant: str, steps: int, flush):
    """Public C-ABI calls with pinned host buffers: H2D of payload+gap+lengths,
    table build, decode, D2H of the decoded symbols, every step inside the
    timed region.  Two calls are in flight, each with its own device buffers,
    workspace, report and CUDA stream (the ABI is stream-ordered with no
    hidden synchronisation), so one call's H2D and decode overlap the
    previous call's D2H on the other copy engine.  Each step starts with an
    L2 flush on its stream (inside the timed region).  Returns the time per
    step (ms) of the median of three timed regions, the last output, the
    bytes moved and the three per-region times."""
    import torch
    from paper_2201_09118_b200 import _lib
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200._pipeline import make_tune
    from paper_2201_09118_b200.device import DeviceReport, empty
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    nwords = -(-stream.total_bits // 32)
    units_h = torch.from_numpy(stream.units.view(np.int32).copy()).pin_memory()
    gap_h = torch.from_numpy(stream.gap.copy()).pin_memory()
    lens = book.length_bytes()
    lens_h = torch.from_numpy(lens.copy()).pin_memory()
    max_codes = len(book.entries)
    lay = stream.layout
    var = _lib.VARIANT_GAP if variant == "gap" else _lib.VARIANT_SYNC
    tune = make_tune(max_len=stream.codebook.max_len)

    class Ctx:
        def __init__(self):
            self.st = torch.cuda.Stream(device=dev)
            self.out_h = torch.empty(stream.symbol_count, dtype=torch.int16).pin_memory()
            self.words = torch.zeros(nwords + _lib.WORD_PAD, dtype=torch.int32, device=dev)
            self.gap_d = torch.empty(len(stream.gap), dtype=torch.uint8, device=dev)
            self.lens_d = torch.empty(len(lens), dtype=torch.uint8, device=dev)
            self.table = torch.empty(lib.bh_table_bytes(max_codes), dtype=torch.uint8, device=dev)
            self.out_d = empty(stream.symbol_count, np.uint16, dev)
            self.cs = _lib.Stream(self.words.data_ptr(), stream.total_bits, stream.symbol_count,
                                  lay.subseq_bits, lay.subseqs_per_seq, 16, max_codes,
                                  self.gap_d.data_ptr(), self.table.data_ptr())
            self.wsb = lib.bh_workspace_bytes(C.byref(self.cs), var, C.byref(tune))
            self.ws = torch.empty(max(self.wsb, 256), dtype=torch.uint8, device=dev)
            lib.bh_workspace_reset(self.ws.data_ptr(), self.ws.numel(), stream_handle(self.st))
            self.rep = DeviceReport(dev).init()

        def step(self):
            with torch.cuda.stream(self.st):
                st = stream_handle(self.st)
                flush()
                self.words[:nwords].copy_(units_h, non_blocking=True)
                self.gap_d.copy_(gap_h, non_blocking=True)
                self.lens_d.copy_(lens_h, non_blocking=True)
                check(lib.bh_table_build(self.lens_d.data_ptr(), len(lens), self.table.data_ptr(), max_codes, st),
                      "table")
                check(lib.bh_decode_async(C.byref(self.cs), var, C.byref(tune), self.out_d.data_ptr(),
                                          self.ws.data_ptr(), self.wsb, self.rep.ptr, st), "decode")
                self.out_h.copy_(self.out_d[: stream.symbol_count], non_blocking=True)

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
    ms = statistics.median(runs)
    for c in ctx:
        check(c.rep.read().status, "e2e decode")
    got = ctx[(steps - 1) % 2].out_h.numpy().view(np.uint16)
    return ms, got, 4 * nwords + len(stream.gap) + len(lens), 2 * stream.symbol_count, runs


# --------------------------------------------------------------------------
# CPU reference (baseline/_ref parhuff, else the C oracle port)
# --------------------------------------------------------------------------

def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    ref = ROOT / "baseline" / "_ref"
    if ref.exists() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import parhuff  # noqa: F401
    return parhuff


def ref_stream(parhuff, stream, book):
    lengths = {s: ln for s, (_, ln) in book.entries.items()}
    rbook = parhuff.canonize(lengths, symbol_width=16)
    lay = parhuff.LayoutConfig(stream.layout.unit_bits, stream.layout.units_per_subseq,
                               stream.layout.subseqs_per_seq)
    return parhuff.EncodedStream(layout=lay, units=stream.units, total_bits=stream.total_bits,
                                 symbol_count=stream.symbol_count, codebook=rbook, gap=stream.gap)


def sample_stream(codes, book, n):
    """First n symbols re-encoded with the same book (a bounded CPU sample)."""
    import paper_2201_09118_b200 as ph
    return ph.encode(codes[:n], book, ph.DEFAULT_LAYOUT, with_gap=True)


def cpu_reference(codes, book, variant: str, budget_s: float, reps: int = 3):
    """Time the reference CPU decoder; returns (GB/s, cores, kind, sample, times)."""
    cores = len(os.sched_getaffinity(0))
    try:
        parhuff = import_reference()
        from parhuff import gap_decoder, sync_decoder
        tiny = sample_stream(codes, book, 20_000)
        rs = ref_stream(parhuff, tiny, book)
        gap_decoder.decode(rs, workers=cores)       # numba JIT warm-up
        sync_decoder.decode(rs, workers=cores)
        t0 = time.perf_counter()
        gap_decoder.decode(rs, workers=cores) if variant == "gap" else sync_decoder.decode(rs, workers=cores)
        rate = 20_000 / max(time.perf_counter() - t0, 1e-6)
        n = int(min(len(codes), max(100_000, rate * budget_s / reps)))
        st = sample_stream(codes, book, n)
        rs = ref_stream(parhuff, st, book)
        fn = (lambda: gap_decoder.decode(rs, workers=cores)) if variant == "gap" else \
             (lambda: sync_decoder.decode(rs, workers=cores))
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            out = fn()
            times.append(time.perf_counter() - t0)
        assert np.array_equal(out, codes[:n])
        med = statistics.median(times)
        return (2 * n / med / 1e9, cores, "reference",
                f"parhuff.{variant}_decoder.decode(workers={cores}) on the first {n} symbols "
                f"({n / len(codes):.1%} of the field), median of {reps}", times, n)
    except Exception as e:  # reference not importable: fall back to the C oracle port
        from oracle import oracle
        n = min(len(codes), 5_000_000)
        st = sample_stream(codes, book, n)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            out = oracle.gap_decode(st) if variant == "gap" else oracle.sync_decode(st)
            times.append(time.perf_counter() - t0)
        med = statistics.median(times)
        return (2 * n / med / 1e9, 1, "port",
                f"C oracle port ({type(e).__name__}: reference unavailable) on {n} symbols", times, n)


def run_reference(args):
    rank, local, world = dist_env()
    if rank != 0:
        return 0
    import torch  # noqa: F401  (GPU only used to build the identical input)
    # the batch config is timed on its first (largest) field
    spec, codes, book, stream = build_field("cesm" if args.config == "multifield" else args.config, 0)
    per_step = max(0.2, 150.0 / max(args.steps + args.warmup, 1))
    cores = len(os.sched_getaffinity(0))
    parhuff = import_reference()
    from parhuff import gap_decoder, sync_decoder
    tiny = ref_stream(parhuff, sample_stream(codes, book, 20_000), book)
    gap_decoder.decode(tiny, workers=cores)
    sync_decoder.decode(tiny, workers=cores)
    t0 = time.perf_counter()
    (gap_decoder if args.variant == "gap" else sync_decoder).decode(tiny, workers=cores)
    rate = 20_000 / max(time.perf_counter() - t0, 1e-6)
    n = int(min(len(codes), max(100_000, rate * per_step)))
    rs = ref_stream(parhuff, sample_stream(codes, book, n), book)
    dec = gap_decoder if args.variant == "gap" else sync_decoder
    for _ in range(args.warmup):
        dec.decode(rs, workers=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out = dec.decode(rs, workers=cores)
        times.append(time.perf_counter() - t0)
    assert np.array_equal(out, codes[:n])
    total = sum(times)
    value = 2 * n * args.steps / total / 1e9
    sample = (f"parhuff.{args.variant}_decoder.decode(workers={cores}) on the first {n} of {len(codes)} "
              f"symbols of {spec.name} per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": {"workload": f"{spec.name} ({spec.n} uint16 quant codes, {spec.bins} bins, sigma {spec.sigma}), "
                               f"{args.variant}-array decoder" if args.variant == "gap" else
                               f"{spec.name}, self-sync decoder", "variant": args.variant, "sample_symbols": n},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# main (B200 arm)
# --------------------------------------------------------------------------

MULTI_FIELDS = ("cesm", "rtm", "qmcpack")
MULTI_CHUNKS = 24  # sequence-aligned chunks over the batch (>= 3 per GPU at 8 GPUs)


def run_multifield(args, rank, world):
    """BASELINE config 5: a CESM/RTM/QMCPACK-shaped batch cut into sequence-
    aligned chunks (shard.chunk_stream) spread over the ranks by LPT on payload
    bits -- strong scaling, no collective on the data path.  Every rank builds
    the same batch, decodes only its chunks, and the step time is the max over
    ranks of its CUDA-event time (one CUDA graph of its chunk launches)."""
    import torch
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200 import _lib, shard
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200._pipeline import make_tune
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty
    from paper_2201_09118_b200.synth import FIELDS, field_codes
    lib = _lib.load()
    var = _lib.VARIANT_GAP if args.variant == "gap" else _lib.VARIANT_SYNC
    fields = []
    for name in MULTI_FIELDS:
        spec = FIELDS[name]
        codes = field_codes(spec)
        book = ph.book_for(codes, 16)
        stream = ph.encode(codes, book, ph.DEFAULT_LAYOUT, with_gap=True)
        st = ph.gap_decoder.entries_from_gap(stream)
        ph.gap_decoder.count_pass(stream, st)        # per-subsequence counts (encode-side metadata)
        fields.append((spec, codes, book, stream, st.counts.copy()))
    total_bits = sum(f[3].total_bits for f in fields)
    chunks = []
    for fi, (spec, codes, book, stream, counts) in enumerate(fields):
        lay = stream.layout
        k = max(1, round(MULTI_CHUNKS * stream.total_bits / total_bits))
        for ch in shard.chunk_stream(stream.total_bits, lay.subseq_bits, lay.subseqs_per_seq, stream.gap,
                                     counts, k):
            chunks.append((fi, ch))
    assign = shard.lpt_assign([ch.total_bits for _, ch in chunks], world)
    mine = [chunks[i] for i in assign[rank]]
    decs = []
    wsb = 256
    for fi, ch in mine:
        spec, codes, book, stream, _ = fields[fi]
        ds = device_stream(stream)
        lay = stream.layout
        c = _lib.Stream(ds.c.words_dev + 4 * ch.word0, ch.total_bits, ch.n, lay.subseq_bits,
                        lay.subseqs_per_seq, book.symbol_width, ds.max_codes, ds.c.gap_dev + ch.sub0,
                        ds.c.table_dev, ch.first_entry, 0)
        tune = make_tune(max_len=book.max_len)
        wsb = max(wsb, lib.bh_workspace_bytes(C.byref(c), var, C.byref(tune)))
        decs.append((fi, ch, c, tune, empty(ch.n, np.uint16, ds.device), DeviceReport(ds.device).init()))
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")

    def step():
        hs = stream_handle()
        for _, _, c, tune, out, rep in decs:
            check(lib.bh_decode_async(C.byref(c), var, C.byref(tune), out.data_ptr(), ws.data_ptr(), wsb,
                                      rep.ptr, hs), "chunk decode")

    step()
    torch.cuda.synchronize()
    for fi, ch, _, _, out, rep in decs:
        check(rep.read().status, "chunk decode")
        assert np.array_equal(out.cpu().numpy().view(np.uint16), fields[fi][1][ch.out0:ch.out0 + ch.n]), \
            f"chunk mismatch (field {fields[fi][0].name}, sequences {ch.q0}..{ch.q1})"
    fn = step
    if args.graph and decs:
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        fn = graph.replay
    flush_buf = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        if world > 1:
            torch.distributed.barrier()
        times = time_steps(fn, args.steps, args.warmup, lambda: flush_buf.zero_())
        if world > 1:
            torch.distributed.barrier()
    my_ms = sum(times)
    my_alg = sum(4 * (-(-ch.total_bits // 32)) + 2 * ch.n + (ch.nsub if args.variant == "gap" else 0)
                 for _, ch, *_ in decs)
    t = torch.tensor([my_ms, float(my_alg)], dtype=torch.float64, device="cuda")
    tot_alg = float(my_alg)
    if world > 1:
        tmax = t.clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tsum = t.clone()
        torch.distributed.all_reduce(tsum, op=torch.distributed.ReduceOp.SUM)
        my_ms, tot_alg = float(tmax[0].item()), float(tsum[1].item())
    nsym = sum(len(f[1]) for f in fields)
    value = 2 * nsym * args.steps / (my_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    achieved = tot_alg * args.steps / (my_ms / 1e3) / 1e9 / world
    line = {
        "impl": "b200", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": my_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32 words -> u16 symbols",
        "data": "synthetic",
        "config": {"workload": "multi-field batch (" + ", ".join(f[0].name for f in fields) + f"), {nsym} uint16 "
                               f"quant codes, {len(chunks)} sequence-aligned chunks, "
                               f"{'gap-array' if args.variant == 'gap' else 'self-sync'} decoder",
                   "variant": args.variant, "n_symbols": nsym, "chunks": len(chunks),
                   "chunks_per_rank": [len(a) for a in assign],
                   "l2": "256 MiB buffer rewritten between steps (outside the per-step events)",
                   "parallelism": f"{len(chunks)} chunks over {world} GPU(s) by LPT on payload bits, no collective",
                   "cuda_graph": bool(args.graph)},
        "roofline": {"bound": "hbm", "kernel": "fused_" + args.variant + " (all chunk launches of a step)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "alg_bytes_per_step": tot_alg, "peak_source": peak_src},
        "clocks": clk.summary(),
        "gpu_launches": len(decs) * args.steps, "gpu_launches_per_step": len(decs),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, local, world = dist_env()
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
    if args.config == "multifield":
        return run_multifield(args, rank, world)
    import paper_2201_09118_b200 as ph
    from paper_2201_09118_b200 import _lib

    spec, codes, book, stream = build_field(args.config, rank)
    n = stream.symbol_count
    dec = Decoder(stream, args.variant, fused=bool(args.fused))
    flush_buf = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    def flush():
        flush_buf.zero_()

    # correctness before timing (bit-exact against the generated field)
    dec()
    r = dec.status()
    _lib.check(r.status, "bench decode")
    assert np.array_equal(dec.out[:n].cpu().numpy().view(np.uint16), codes), "decode mismatch"

    launches = count_launches(dec)
    step_fn = dec
    if args.graph:
        # the fused decode is one kernel with its epoch kept on the device, so
        # the whole call is capturable: replay removes host launch overhead
        for _ in range(3):
            dec()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            dec()
        torch.cuda.synchronize()
        step_fn = graph.replay
        step_fn()
        torch.cuda.synchronize()
        assert np.array_equal(dec.out[:n].cpu().numpy().view(np.uint16), codes), "graph decode mismatch"
        launches = count_launches(step_fn)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    if not args.graph:
        _lib.profile_enable(True)
    with ClockSampler(local) as clk:
        if world > 1:
            torch.distributed.barrier()
        times = time_steps(step_fn, args.steps, args.warmup, flush)
        if world > 1:
            torch.distributed.barrier()
    if args.graph:
        # one kernel per replay: the per-step events bracket exactly that launch
        prof = {("fused_" + args.variant) if args.fused else "decode": (sum(times), len(times))}
    else:
        prof = _lib.profile_read()
        _lib.profile_enable(False)
    r = dec.status()
    _lib.check(r.status, "bench decode")
    total_ms = sum(times)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(t.item())
    value = world * 2 * n * args.steps / (total_ms / 1e3) / 1e9

    peak, peak_src = measured_peak()
    # dominant phase: largest summed time (warm-up phases included in the sum
    # only via the timed steps since profiling starts right before them)
    dom, (dom_ms, dom_cnt) = max(prof.items(), key=lambda kv: kv[1][0]) if prof else ("decode", (total_ms, args.steps))
    dom_avg = dom_ms / max(dom_cnt, 1)
    ab = alg_bytes(stream, args.variant)
    achieved = ab / (dom_avg / 1e3) / 1e9
    traffic = None
    nc = ROOT / "profiles" / "ncu_summary.json"
    if nc.exists():
        try:
            d = json.loads(nc.read_text())
            traffic = d.get(args.config, {}).get(args.variant, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "impl": "b200", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 words -> u16 symbols",
        "data": "synthetic",
        "config": {
            "workload": f"{spec.name} ({n} uint16 quant codes, {spec.bins} bins, sigma {spec.sigma}), "
                        f"{'gap-array' if args.variant == 'gap' else 'self-sync'} decoder",
            "variant": args.variant, "n_symbols": n, "total_bits": stream.total_bits,
            "compression_ratio": round(16 * n / stream.total_bits, 3), "layout": "32-bit units, 4/subseq, 32/seq",
            "l2": "256 MiB buffer rewritten between steps (outside the per-step events)",
            "parallelism": f"{world} field(s), one per GPU, no collective",
            "fused": bool(args.fused),
            "cuda_graph": bool(args.graph),
        },
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "alg_bytes_per_launch": ab,
                     "avg_launch_ms": dom_avg, "peak_source": peak_src,
                     "phases_ms_per_step": {k: v[0] / max(v[1], 1) for k, v in prof.items()},
                     "whole_decode_frac": (ab / (total_ms / args.steps / 1e3) / 1e9) / peak},
        "clocks": clk.summary(),
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
    }

    if not args.no_extras:
        # e2e through the public C-ABI call with host buffers
        ksteps = max(3, min(args.steps, 50))
        if world > 1:
            torch.distributed.barrier()
        ems, got, bi, bo, eruns = e2e_measure(stream, book, args.variant, ksteps, flush)
        assert np.array_equal(got, codes), "e2e decode mismatch"
        if world > 1:  # whole job: every rank's field, slowest rank's time
            te = torch.tensor([ems], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
            ems = float(te.item())
        line["e2e"] = {"value": world * 2 * n / (ems / 1e3) / 1e9, "unit": "GB/s",
                       "h2d_bytes_per_step": world * bi, "d2h_bytes_per_step": world * bo, "steps": ksteps,
                       "ms_per_step": ems, "in_flight": 2, "regions": 3,
                       "ms_per_step_regions": eruns}
        # other variants and the in-run coarse-grained cuSZ-style baseline
        variants = {args.variant: value / world}
        other = "sync" if args.variant == "gap" else "gap"
        od = Decoder(stream, other, fused=bool(args.fused))
        ot = time_steps(od, max(3, min(args.steps, 100)), 3, flush)
        variants[other] = 2 * n / (statistics.mean(ot) / 1e3) / 1e9
        variants["coarse_cusz"] = coarse_baseline(ph, codes, book, stream, flush)
        line["variants_gbs_per_gpu"] = variants
        line["speedup_vs_coarse"] = {k: v / variants["coarse_cusz"]["value"]
                                     for k, v in variants.items() if k != "coarse_cusz"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            v, cores, kind, sample, ts, ns = cpu_reference(codes, book, args.variant, budget_s=20.0)
            line["cpu_baseline"] = {"value": v, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def coarse_baseline(ph, codes, book, stream, flush):
    """cuSZ-style coarse-grained decoder (K8): best chunk of a small sweep."""
    import torch
    from paper_2201_09118_b200 import _lib
    from paper_2201_09118_b200._lib import check, stream_handle
    from paper_2201_09118_b200.device import DeviceReport, device_stream, empty, h2d
    from paper_2201_09118_b200.encoder import encode_device
    lib = _lib.load()
    ds = device_stream(stream)
    sd = h2d(codes, ds.device)
    best = None
    for chunk in (256, 1024, 4096):
        _, _, _, offs = encode_device(sd, len(codes), book, ph.DEFAULT_LAYOUT, False, chunk)
        out = empty(len(codes), np.uint16, ds.device)
        rep = DeviceReport(ds.device).init()

        def fn():
            check(lib.bh_coarse_decode(ds.ref, offs.data_ptr(), chunk, out.data_ptr(), rep.ptr,
                                       stream_handle()), "coarse")
        fn()
        torch.cuda.synchronize()
        check(rep.read().status, "coarse")
        assert np.array_equal(out[: len(codes)].cpu().numpy().view(np.uint16), codes)
        ts = time_steps(fn, 10, 2, flush)
        v = 2 * len(codes) / (statistics.mean(ts) / 1e3) / 1e9
        if best is None or v > best["value"]:
            best = {"value": v, "chunk": chunk,
                    "alg_bytes": 4 * (-(-stream.total_bits // 32)) + 8 * (-(-len(codes) // chunk)) + 2 * len(codes)}
    return best


if __name__ == "__main__":
    sys.exit(main())
