#!/bin/bash
# quick GPU check: gpu tests + compact bench lines for the given configs
# usage: tools/quick.sh [tests] [configs...]
O=gpurun_out/quick; mkdir -p $O
if [ "$1" = "tests" ]; then shift; python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log; fi
for c in "$@"; do
  v=gap; cfg=$c
  case $c in *:sync) v=sync; cfg=${c%:sync};; esac
  python bench.py --no-cpu-baseline --no-extras --config $cfg --variant $v > $O/b_${cfg}_$v.json 2> $O/b_${cfg}_$v.err
  python - "$O/b_${cfg}_$v.json" "$cfg" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:>10} {sys.argv[3]:>4} {d['value']:9.1f} GB/s  {d['ms_per_step']*1e3:8.1f} us  frac {d['roofline']['frac']:.3f}  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
done
