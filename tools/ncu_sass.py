"""SASS listing with per-instruction stall reasons and shared-memory wavefronts
from an ncu report: python tools/ncu_sass.py REPORT [min_exec] [addr_lo addr_hi]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_exec = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 64
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows[2:] if len(r) == len(h))
for r in rows[2:]:
    if len(r) != len(h):
        continue
    a = int(r[0], 16)
    ex = int(r[ix["Instructions Executed"]] or 0)
    if ex < min_exec or not (lo <= (a & 0xffffff) < hi):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:2]
    wf, wfi = r[ix["L1 Wavefronts Shared"]], r[ix["L1 Wavefronts Shared Ideal"]]
    sh = f" wf {wf}/{wfi}" if wf not in ("0", "") else ""
    th = r[ix["Avg. Threads Executed"]]
    print(f"{a & 0xffffff:06x} {ex:8d} t{float(th):4.1f} st {100 * s / tot:4.1f}% "
          f"{' '.join(f'{k}:{v}' for v, k in top if v):28s} {r[1].strip()[:60]}{sh}")
