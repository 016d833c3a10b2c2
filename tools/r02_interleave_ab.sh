#!/bin/bash
# Direct reduce-scatter job order: block-major (default) vs destination-fastest, large sizes, alternating repeats.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_interleave_ab
mkdir -p $O
for rep in 1 2 3; do
  for v in default interleave; do
    if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
    PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 \
      tools/ring_sweep.py --sizes 4194304,16777216,67108864,268435456 --codecs none --iters 20 --warmup 5 \
      2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/sweep.jsonl
  done
done
