#!/bin/bash
# Flag-protocol batch (groups per lane) and LL threshold A/B, p = 2 and 4, mid and large sizes.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_batch_ab}
mkdir -p $O
S=648010,1048576,2097152,4194304,8388608,16777216,25557032,67108864,268435456
for np in 4 2; do
  for v in default b512 b256 llhop1 b256_llhop1; do
    if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
    PIPESGD_LIB=$L timeout 400 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29632 \
      tools/ring_sweep.py --sizes $S --codecs none,trunc16,quant8 --iters 20 --warmup 5 --check \
      $([ $v = default ] && echo --nccl) > $O/p${np}_$v.log 2>&1
    grep '^{' $O/p${np}_$v.log > $O/p${np}_$v.jsonl
  done
done
