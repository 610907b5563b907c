"""Instruction / stall totals per fused.cu function (line ranges found by
regex in the source) from an ncu report: where the warp instructions go."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

rep = sys.argv[1]
src = (Path(__file__).resolve().parent.parent / "paper_2201_09118_b200" / "csrc" / "fused.cu").read_text().splitlines()
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"^(?:template <[^>]*>\s*)?(?:__global__|__device__|struct)\b.*?(\w+)\s*(?:\(|\{)", l)
    if m:
        starts.append((i, m.group(1)))
def func(line):
    name = "?"
    for s, n in starts:
        if s <= line:
            name = n
        else:
            break
    return name
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0])
fname, hdr = "", None
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        fname, hdr = r[1].split("/")[-1], None
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
    k = func(int(r[0])) if fname == "fused.cu" else fname
    agg[k][0] += n
    agg[k][1] += s
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot}  stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if v[0] / tot > 0.002:
        print(f"{k:<24} {100 * v[0] / tot:5.1f}% instr {100 * v[1] / ts:5.1f}% stall")
