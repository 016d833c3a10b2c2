#!/bin/bash
# codec none at p = 4 (and 2): direct reduce-scatter vs the ring's p-1 hops vs NCCL.
cd "$(dirname "$0")/.."
S="256,4096,65536,262144,524288,1048576,2097152,4194304,6389258,16777216,67108864"
for np in 4 2; do
  for d in 1 0; do
    [ $np -eq 2 ] && [ $d -eq 0 ] && continue
    echo "== p=$np direct=$d"
    PIPESGD_DIRECT=$d timeout 600 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29513 \
      tools/ring_sweep.py --sizes $S --codecs none --iters 20 --warmup 5 --check $([ $d -eq 1 ] && echo --nccl) 2>&1 | grep '^{'
  done
done
