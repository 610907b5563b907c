#!/bin/bash
# Final-state evidence in one GPU call: GPU tests, bench lines (default HACC
# gap, sync, reference arm, multifield), the launch list of the bench command,
# ncu --set full of the fused decoders (HACC/QMCPACK gap and sync), every
# config's quick line and ipc table, K1's ncu, a 5-minute fuzz soak.
# (compute-sanitizer is closed on the GPU pool.)
# Outputs in gpurun_out/final/.
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1; tail -2 $O/tests.log
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
python bench.py --variant sync --no-cpu-baseline > $O/bench_sync.json 2> $O/bench_sync.err
python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --config multifield --steps 20 --warmup 3 > $O/bench_multifield.json 2> $O/bench_multifield.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/launches_bench.log 2>&1
for cv in hacc:gap hacc:sync qmcpack:gap qmcpack:sync; do
  c=${cv%:*}; v=${cv#*:}
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 4 -c 1 -f -o $O/${c}_$v \
      python bench.py --config $c --steps 3 --warmup 3 --no-extras --no-cpu-baseline --variant $v > $O/ncu_${c}_$v.log 2>&1
done
bash tools/quick.sh 1m hurricane hurricane:sync nyx nyx:sync nyx256 nyx4096 hacc hacc:sync qmcpack qmcpack:sync cesm cesm:sync rtm rtm:sync > $O/quick.txt 2>&1
bash tools/ipc_table.sh > $O/ipc_table.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_table_canon -s 4 -c 1 -f -o $O/k1 \
    python bench.py --config hacc --steps 3 --warmup 3 --no-extras --no-cpu-baseline > $O/ncu_k1.log 2>&1
timeout 420 python tools/fuzz.py --minutes 5 > $O/fuzz.txt 2>&1; tail -1 $O/fuzz.txt
ls $O
