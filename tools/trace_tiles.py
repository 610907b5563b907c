"""Per-tile breakdown of a trace_fused.py timeline (gpurun_out/trace_<cfg>_<variant>.npy):
words wait / count per count-phase tile, words wait / decode / flush per decode-phase tile."""
import sys

import numpy as np

rel = np.load(sys.argv[1])


def q(x):
    x = x[x >= 0]
    return f"med {np.median(x) / 1e3:5.2f} p90 {np.percentile(x, 90) / 1e3:5.2f} n {len(x):5d}" if len(x) else "-"


def d(i, j):
    m = (rel[:, i] > 0) & (rel[:, j] > 0)
    return np.where(m, rel[:, j] - rel[:, i], -1)


print(f"prologue: start {q(rel[:, 0])} | syncthreads {q(rel[:, 56])} | count tables {q(rel[:, 1])}")
for k in range(8):
    a, b = 10 + 2 * k, 11 + 2 * k
    prev = 1 if k == 0 else 9 + 2 * k
    if (rel[:, a] <= 0).all():
        break
    print(f"count tile {k}: wait {q(d(prev, a))} | count {q(d(a, b))}")
for k in range(8):
    a, b, c = 30 + 3 * k, 31 + 3 * k, 32 + 3 * k
    prev = 3 if k == 0 else 29 + 3 * k
    if (rel[:, a] <= 0).all():
        break
    print(f"decode tile {k}: wait {q(d(prev, a))} | decode {q(d(a, b))} | flush {q(d(b, c))}")
