#!/bin/bash
# Per config and decoder: warp instructions per decoded symbol, IPC, issue
# utilisation, thread efficiency and DRAM bytes of the fused kernel (one ncu
# launch each, the 7th k_fused launch of a short bench run).
# usage: tools/ipc_table.sh [configs...]   (default: every BASELINE config, gap and sync)
O=gpurun_out/ipc; mkdir -p $O
CFGS="$*"
[ -z "$CFGS" ] && CFGS="hurricane nyx256 nyx nyx4096 hacc cesm rtm qmcpack hurricane:sync nyx:sync hacc:sync cesm:sync rtm:sync qmcpack:sync"
M=smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
printf "%-10s %-4s %11s %9s %10s %6s %6s %6s %9s %9s %9s %6s\n" config var symbols time_us warp_inst inst/sym IPC issue% thr_eff dram_rd_MB dram_wr_MB conf%
for c in $CFGS; do
  v=gap; cfg=$c
  case $c in *:sync) v=sync; cfg=${c%:sync};; esac
  f=$O/${cfg}_$v.csv
  ncu --metrics $M --clock-control none -k regex:k_fused -s 6 -c 1 --csv \
    python bench.py --config $cfg --variant $v --steps 3 --warmup 3 --no-extras --no-cpu-baseline > $f 2>/dev/null
  python - $f $cfg $v <<'PY'
import csv, json, sys
from paper_2201_09118_b200 import synth
lines = open(sys.argv[1]).read().splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[i:]))
h = rows[0]
m = {}
for r in rows[1:]:
    if len(r) == len(h):
        d = dict(zip(h, r))
        v = float(d["Metric Value"].replace(",", ""))
        u = d.get("Metric Unit", "")
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
        v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        m[d["Metric Name"]] = v
n = synth.FIELDS[sys.argv[2]].n
inst = m["smsp__inst_executed.sum"]
t_us = m["gpu__time_duration.sum"]
conf = 100 * m["l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"] / max(1.0, m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"])
print(f"{sys.argv[2]:<10} {sys.argv[3]:<4} {n:>11} {t_us:9.1f} {inst/1e6:9.1f}M {inst/n:6.2f} "
      f"{m['sm__inst_executed.avg.per_cycle_active']:6.2f} {m['smsp__issue_active.avg.pct_of_peak_sustained_active']:6.1f} "
      f"{m['smsp__thread_inst_executed_per_inst_executed.ratio']:9.2f} {m['dram__bytes_read.sum']/1e6:9.1f} "
      f"{m['dram__bytes_write.sum']/1e6:9.1f} {conf:6.1f}")
PY
done
