#!/bin/bash
# p = 4 codec none mid sizes: direct reduce-scatter scheduling variants (+ timelines at 12 MiB).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_direct_ab}
mkdir -p $O
S=1048576,1572864,2097152,3145728,4194304,8388608,16777216,67108864
for v in default flagstatic interleave flagstatic_interleave; do
  if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
  PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29639 \
    tools/ring_sweep.py --sizes $S --codecs none,trunc16 --iters 30 --warmup 5 --check \
    $([ $v = default ] && echo --nccl) > $O/p4_$v.log 2>&1
  grep '^{' $O/p4_$v.log > $O/p4_$v.jsonl
  PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 \
    tools/ring_timeline.py --numel 3145728 --codec none > $O/timeline_$v.log 2>&1
done
