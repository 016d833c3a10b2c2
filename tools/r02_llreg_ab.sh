#!/bin/bash
# LL for larger blocks (short LL chunks + the smaller LL code): default vs 4 MiB / 8 MiB LL regions.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_llreg_ab}
mkdir -p $O
for np in 4 2; do
  S=648010,1048576,1572864,2097152,3145728,4194304,8388608
  for v in default llhop1 llreg4 llreg8; do
    if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
    PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29635 \
      tools/ring_sweep.py --sizes $S --codecs none,trunc16,quant8 --iters 30 --warmup 5 --check \
      $([ $v = default ] && echo --nccl) > $O/p${np}_$v.log 2>&1
    grep '^{' $O/p${np}_$v.log > $O/p${np}_$v.jsonl
  done
done
