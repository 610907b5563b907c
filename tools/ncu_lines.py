"""Per-source-line instruction / stall totals from an ncu report (cuda,sass view)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
import os
extra = ["--kernel-name", os.environ["NCU_KERNEL"], "--launch-count", "1"] if os.environ.get("NCU_KERNEL") else []
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + extra,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = defaultdict(lambda: [0, 0, ""])
fname = ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    try:
        n = int(r[hdr["Instructions Executed"]] or 0)
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        continue
    k = (fname, int(r[0]))
    agg[k][0] += n
    agg[k][1] += s
    agg[k][2] = r[1][:80]
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {tot}  stall samples {ts}")
key = 1 if os.environ.get("NCU_SORT") == "stall" else 0
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    print(f"{k[0]}:{k[1]:<5} {100 * v[0] / tot:5.1f}% instr {100 * v[1] / ts:5.1f}% stall  {v[2].strip()}")
