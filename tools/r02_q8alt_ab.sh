#!/bin/bash
# quant8 alternating chunk direction (PIPESGD_Q8_ALTERNATE=1 variant) vs default, alternating repeats.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_q8alt_ab
mkdir -p $O
for np in 4 2; do
  for rep in 1 2; do
    for v in default q8alt; do
      if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
      PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29644 \
        tools/ring_sweep.py --sizes 4194307,16777216,61100840,268435456 --codecs quant8 --iters 10 --warmup 3 --check \
        2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/sweep.jsonl
    done
  done
done
