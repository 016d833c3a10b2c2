#!/bin/bash
# Flag-protocol minimum chunk A/B (1024 default vs 512 / 256 elements) at mid sizes.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_minchunk}
mkdir -p $O
for np in 4 2; do
  for v in default minchunk512 minchunk256; do
    if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
    echo "{\"lag\": \"$v\"}" >> $O/sweep.jsonl
    PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29701 \
      tools/ring_sweep.py --sizes 2097152,4194304,4710538,8388608,16777216,25557032,61100840 \
      --codecs none,trunc16,quant8 --ctas 592 --iters 20 --warmup 5 --check $([ $v = default ] && echo --nccl) \
      2>&1 | grep '^{' >> $O/sweep.jsonl
  done
done
