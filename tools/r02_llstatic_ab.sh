#!/bin/bash
# LL static chunk stride (default now) vs the phase counter, and larger LL slots with static striding.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_llstatic_ab}
mkdir -p $O
S=65536,262144,648010,1048576,1572864,2097152,3145728,4194304,8388608
for np in 4 2; do
  for v in default lldyn llreg4s llreg8s; do
    if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
    PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29638 \
      tools/ring_sweep.py --sizes $S --codecs none,trunc16,quant8 --iters 30 --warmup 5 --check \
      $([ $v = default ] && echo --nccl) > $O/p${np}_$v.log 2>&1
    grep '^{' $O/p${np}_$v.log > $O/p${np}_$v.jsonl
  done
done
