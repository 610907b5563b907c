"""SURVEY.md §8(d) sweeps on one B200 (python tools/sweep.py [table1 layout coarse] > profiles/.../sweeps.md):

* table1 -- the paper's Table I analog: per config, the
  fused decoder's staging capacity chosen online from the stream header
  (symbols per warp, `cap`) against a brute-force sweep of capacities
  (BH_FUSED_CAP, 0.5x .. 3x of the expected symbols per tile), plus the
  paper's class tuner (TunerConfig(t_high=8)) on the same kernel;
* layout -- HACC-shaped field: units_per_subseq x subseqs_per_seq
  ({2,4,8} x {16,32,64}), both decoders;
* coarse -- the cuSZ-style coarse baseline over chunk sizes 2^8..2^14 (HACC).

Every point is checked bit-exact against the generated codes before timing.
Times are CUDA events around the decode kernel alone (tables prebuilt), L2
flushed between decodes.
"""
import ctypes as C
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_09118_b200 as ph  # noqa: E402
from bench import FLUSH_BYTES, Piece, load_synth, run_steps  # noqa: E402

flush_buf = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
synth = load_synth()


def flush():
    flush_buf.zero_()


def field(name, layout=ph.DEFAULT_LAYOUT):
    codes = synth.field_codes(synth.FIELDS[name])
    sd = torch.from_numpy(codes.view(np.int16)).cuda()
    book = ph.book_for_device(sd, codes.size, 16)
    return codes, sd, ph.encode(codes, book, layout, with_gap=True)


def timed(piece, sd, steps=10, tuner=None):
    if tuner is not None:
        from paper_2201_09118_b200._pipeline import make_tune
        t = make_tune(tuner_config=tuner, max_len=piece.tune.max_len, min_len=piece.tune.min_len)
        piece.tune = t
    ts = run_steps([piece], steps, 3, flush)
    ph._lib.check(piece.rep.read().status, "sweep")
    assert torch.equal(piece.out[: piece.n], sd), "sweep decode mismatch"
    return statistics.median(t[1] for t in ts)


def gbs(n, ms):
    return 2 * n / (ms / 1e3) / 1e9


def shape(piece):
    lib = piece.lib
    lib.bh_debug_fused_shape.argtypes = [C.c_void_p, C.c_void_p] + [C.POINTER(C.c_uint32)] * 4
    w, sm, cap, spl = (C.c_uint32() for _ in range(4))
    lib.bh_debug_fused_shape(C.byref(piece.c), C.byref(piece.tune), C.byref(w), C.byref(sm), C.byref(cap),
                             C.byref(spl))
    return w.value, sm.value, cap.value, spl.value


def table1(configs=("hurricane", "nyx", "cesm", "rtm", "hacc", "qmcpack")):
    print("## Table I analog: staging capacity chosen online vs brute force (gap decoder)\n")
    print("`cap` = staging symbols per warp (one tile of 32 lanes x spl subsequences); warps per CTA follow "
          "from the shared memory left.  `online` = the header-CR rule of `fused_cfg` "
          "(csrc/fused.cu), `tuner` = the same launch with the paper's class tuner "
          "(TunerConfig(t_high=8): per-tile class capacity, tuner.py:98-106).\n")
    print("| config | CR | spl | symbols/tile | online cap (warps) | online GB/s | tuner GB/s | best brute-force cap "
          "(warps) | best GB/s | online / best |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for name in configs:
        codes, sd, st = field(name)
        p = Piece(st, "gap")
        p.table_build(torch.cuda.current_stream().cuda_stream)
        w0, _, cap0, spl = shape(p)
        per_tile = 32 * spl * st.layout.subseq_bits * codes.size / st.total_bits
        t_online = timed(p, sd)
        t_tuner = timed(Piece(st, "gap"), sd, tuner=ph.TunerConfig(t_high=8))
        best = (t_online, cap0, w0)
        rows = []
        for f in (0.5, 0.75, 0.9, 1.0, 1.05, 1.25, 1.5, 2.0, 3.0):
            cap = int(per_tile * f) // 8 * 8
            if cap < 64:
                continue
            os.environ["BH_FUSED_CAP"] = str(cap)
            try:
                q = Piece(st, "gap")
                q.table_build(torch.cuda.current_stream().cuda_stream)
                w, _, _, _ = shape(q)
                t = timed(q, sd)
            except Exception as e:  # the capacity leaves no room for a warp
                rows.append(f"cap {cap}: {type(e).__name__}")
                continue
            finally:
                os.environ.pop("BH_FUSED_CAP", None)
            rows.append(f"{cap}:{gbs(codes.size, t):.0f}")
            if t < best[0]:
                best = (t, cap, w)
        print(f"| {name} | {16 * codes.size / st.total_bits:.2f} | {spl} | {per_tile:.0f} | {cap0} ({w0}) | "
              f"{gbs(codes.size, t_online):.0f} | {gbs(codes.size, t_tuner):.0f} | {best[1]} ({best[2]}) | "
              f"{gbs(codes.size, best[0]):.0f} | {best[0] and t_online and best[0] / t_online:.3f} |", flush=True)
        print(f"<!-- {name} sweep cap:GB/s {' '.join(rows)} -->", flush=True)
        del p, st, sd
        torch.cuda.empty_cache()


def layout_sweep():
    codes = synth.field_codes(synth.FIELDS["hacc"])
    sd = torch.from_numpy(codes.view(np.int16)).cuda()
    book = ph.book_for_device(sd, codes.size, 16)
    print("\n## HACC-shaped field (281 M codes): stream layout sweep\n")
    print("| units/subseq | subseqs/seq | CR | gap GB/s | sync GB/s |")
    print("|---|---|---|---|---|")
    for ups in (2, 4, 8):
        for sps in (16, 32, 64):
            st = ph.encode(codes, book, ph.LayoutConfig(32, ups, sps), with_gap=True)
            row = []
            for var in ("gap", "sync"):
                p = Piece(st, var)
                p.table_build(torch.cuda.current_stream().cuda_stream)
                row.append(f"{gbs(codes.size, timed(p, sd, 5)):.0f}")
                del p
            print(f"| {ups} | {sps} | {16 * codes.size / st.total_bits:.2f} | {row[0]} | {row[1]} |", flush=True)
            del st
            torch.cuda.empty_cache()


def coarse_sweep():
    from bench import coarse_baseline
    codes, sd, st = field("hacc")
    r = coarse_baseline(ph, codes, st.codebook, st, flush)
    print("\n## cuSZ-style coarse-grained baseline (K8) over chunk sizes, HACC-shaped field\n")
    print("| chunk (symbols) | GB/s |")
    print("|---|---|")
    for k, v in r["sweep_gbs"].items():
        print(f"| {k} | {v} |")


if __name__ == "__main__":
    print("# Sweeps (B200, one GPU; CUDA events per decode, L2 flushed between decodes)\n")
    which = sys.argv[1:] or ["table1", "layout", "coarse"]
    if "table1" in which:
        table1()
    if "layout" in which:
        layout_sweep()
    if "coarse" in which:
        coarse_sweep()
