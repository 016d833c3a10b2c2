#!/bin/bash
# Every codec at p = 2 and 4 over the BASELINE gradient sizes and a few C5
# points, NCCL beside it (quick A/B of kernel changes).
cd "$(dirname "$0")/.."
S=${SIZES:-"256,262144,648010,1048576,4194304,4710538,16777216,25557032,61100840,268435456"}
for np in ${PS:-4 2}; do
  echo "== p=$np"
  timeout 900 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29513 \
    tools/ring_sweep.py --sizes $S --iters 20 --warmup 5 --check --nccl 2>&1 | grep '^{'
done
