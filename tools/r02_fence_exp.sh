#!/bin/bash
# Is the per-chunk system-scope release what makes mid-size flag-protocol calls slow? (timing only)
cd "$(dirname "$0")/.."
O=gpurun_out/r02_fence_exp
mkdir -p $O
S=1048576,2097152,4194304,8388608,16777216,67108864
for np in 4 2; do
  for v in default nofence; do
    if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
    PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29633 \
      tools/ring_sweep.py --sizes $S --codecs none,trunc16 --iters 20 --warmup 5 > $O/p${np}_$v.log 2>&1
    grep '^{' $O/p${np}_$v.log > $O/p${np}_$v.jsonl
  done
done
PIPESGD_LIB=$PWD/variants/lib_nofence.so timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29634 tools/ring_timeline.py --numel 2097152 --codec none > $O/timeline_nofence.log 2>&1
