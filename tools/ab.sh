#!/bin/bash
# A/B the library builds under build/ab/*.so (make EXTRA=... LIB=... BUILD=...):
# compact bench lines + ncu instruction count / IPC of the fused kernel.
# usage: tools/ab.sh "configs..." lib1.so lib2.so ...
O=gpurun_out/ab; mkdir -p $O
CFGS="$1"; shift
for L in "$@"; do
  n=$(basename $L .so)
  echo "== $n"
  BH_LIB=$PWD/$L bash tools/quick.sh $CFGS
  BH_LIB=$PWD/$L ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,smsp__thread_inst_executed_per_inst_executed.ratio,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum \
     --clock-control none -k regex:k_fused -s 6 -c 1 --csv python bench.py --config ${NCU_CFG:-hacc} --steps 3 --warmup 3 --no-extras --no-cpu-baseline > $O/ncu_$n.csv 2>/dev/null
  python - $O/ncu_$n.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
h, rows = rows[i], rows[i:]
for r in rows[1:]:
    d = dict(zip(h, r)); print(f"   ncu {d['Metric Name']:<60} {d['Metric Value']}")
PY
done
