"""Debug: seam-walk statistics of the fused self-sync decoder on a BASELINE
config (needs a library built with -DBH_SEAM_STATS, passed as BH_LIB).
usage: BH_LIB=build/ab/stats.so python tools/seam_stats.py hacc qmcpack ..."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

for cfg in sys.argv[1:]:
    import argparse
    ns = argparse.Namespace(config=cfg, variant="sync", gpus=1, steps=1, warmup=0, impl="b200",
                            no_cpu_baseline=True, no_extras=True)
    fields, items = bench.build_workload(ns, 0, 1)
    st = fields[0][3]
    p = bench.Piece(st, "sync")
    s = torch.cuda.current_stream().cuda_stream
    p.table_build(s)
    p.decode(s)
    torch.cuda.synchronize()
    r = p.rep.read()
    print(f"{cfg}: status {r.status} walk failures {r.repair_needed} serial re-syncs {r.stale_seams} "
          f"dependent first tiles {r.seam_passes} (bits {st.total_bits})", flush=True)
