#!/bin/bash
# One GPU call: bench lines (gap default, sync), ncu launch list of the bench
# command, full ncu captures of the fused gap/sync kernels (Hurricane), and
# the per-config quick lines.  Outputs in gpurun_out/prof/.
set -x
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --variant sync --no-cpu-baseline > $O/bench_sync.json 2> $O/bench_sync.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/launches_bench.log 2>&1
for v in gap sync; do
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -f -o $O/fused_$v \
      python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline --variant $v > $O/ncu_$v.log 2>&1
done
bash tools/quick.sh 1m hurricane hurricane:sync nyx nyx256 nyx4096 hacc hacc:sync qmcpack cesm rtm > $O/quick.txt 2>&1
python bench.py --config multifield --steps 20 --warmup 3 > $O/bench_multifield.json 2> $O/bench_multifield.err
ls -la $O
