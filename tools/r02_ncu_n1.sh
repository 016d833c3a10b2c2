#!/bin/bash
# N=1 bench (C3 default) evidence: the plain run, then the ncu launch list of
# the timed region (gpu__time_duration, clock control off), then ncu --set
# full of our kernels in the timed region (dram bytes per launch -> traffic).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_ncu_n1}
mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err
BENCH_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file $O/launches_n1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
BENCH_PROFILE_RANGE=1 timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"consume_update|encode_kernel|absmax" -c 6 -f -o $O/n1_kernels python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done >> $O/ncu_full.log
