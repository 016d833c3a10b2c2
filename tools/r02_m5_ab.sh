#!/bin/bash
# quant8 ring at 5 CTAs per SM (96 registers, small spills; 740 CTAs) vs 4 (128 registers; 592 CTAs).
cd "$(dirname "$0")/.."
O=gpurun_out/r02_m5_ab
mkdir -p $O
for np in 4 2; do
  for rep in 1 2; do
    for v in default m5; do
      if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; G=592; else L=$PWD/variants/lib_$v.so; G=740; fi
      PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29645 \
        tools/ring_sweep.py --sizes 4194307,16777216,61100840,268435456 --codecs quant8,trunc16 --ctas $G --iters 10 \
        --warmup 3 --check 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/sweep.jsonl
    done
  done
done
