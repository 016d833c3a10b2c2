#!/bin/bash
# LL threshold A/B with the short LL chunks: hop budget 512 KiB (default) vs 1 / 2 MiB x (p-1).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_llhop}
mkdir -p $O
for np in 4 2; do
  for v in default llhop1 llhop2; do
    if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
    echo "{\"lag\": \"$v\"}" >> $O/sweep.jsonl
    PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29631 \
      tools/ring_sweep.py --sizes 262144,648010,1048576,2097152,4194304,8388608 --codecs none,trunc16,quant8 \
      --ctas 592 --iters 20 --warmup 5 --check $([ $v = default ] && echo --nccl) 2>&1 | grep '^{' >> $O/sweep.jsonl
  done
done
