#!/bin/bash
# quant8 ring: 2 groups per lane with 3 / 2 CTAs per SM vs the default (1 group, 4 CTAs per SM), p = 4 and 2.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_q8u_ab
mkdir -p $O
for np in 4 2; do
  for v in default q8u2_m3 q8u2_m2 m3; do
    if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
    PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29642 \
      tools/ring_sweep.py --sizes 16777216,61100840,268435456 --codecs quant8,trunc16 --iters 10 --warmup 3 --check \
      > $O/p${np}_$v.log 2>&1
    grep '^{' $O/p${np}_$v.log > $O/p${np}_$v.jsonl
  done
done
