#!/bin/bash
# One optimisation iteration on the GPU box: parity suite, compact bench lines,
# per-warp trace of the Hurricane gap decode.  usage: tools/iter.sh [configs...]
O=gpurun_out/iter; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1; tail -2 $O/tests.log
if [ $# -eq 0 ]; then set -- hurricane hurricane:sync nyx hacc; fi
bash tools/quick.sh "$@"
python tools/trace_fused.py > $O/trace_gap.txt 2>&1; head -12 $O/trace_gap.txt
