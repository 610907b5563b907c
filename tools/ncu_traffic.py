"""Write profiles/ncu_summary.json: per-launch DRAM traffic of the fused
kernels from `ncu --set full` captures (bench.py reads it for roofline.traffic).

usage: python tools/ncu_traffic.py CONFIG VARIANT REPORT [CONFIG VARIANT REPORT ...]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent.parent / "profiles" / "ncu_summary.json"
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = lambda n: float(vals[hdr.index(n)].replace(",", "")) * UNIT.get(units[hdr.index(n)], 1)
    return {"dram_read_bytes": get("dram__bytes_read.sum"), "dram_write_bytes": get("dram__bytes_write.sum"),
            "duration_us": float(vals[hdr.index("gpu__time_duration.sum")].replace(",", "")) *
            {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(units[hdr.index("gpu__time_duration.sum")], 1.0),
            "kernel": vals[hdr.index("Kernel Name")]}


d = json.loads(OUT.read_text()) if OUT.exists() else {}
a = sys.argv[1:]
for cfg, var, rep in zip(a[0::3], a[1::3], a[2::3]):
    m = metrics(rep)
    m["dram_bytes_per_launch"] = m["dram_read_bytes"] + m["dram_write_bytes"]
    m["report"] = Path(rep).name
    m["note"] = ("ncu replays with caches flushed before the kernel; decoded output still resident in the "
                 "126 MB L2 at kernel end is written back after it, so dram writes undercount the output")
    d.setdefault(cfg, {})[var] = m
OUT.write_text(json.dumps(d, indent=1) + "\n")
print(json.dumps(d, indent=1))
