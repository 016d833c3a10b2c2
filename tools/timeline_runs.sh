#!/bin/bash
cd "$(dirname "$0")/.."
NP=${NP:-2}
for args in ${RUNS:-"--numel 16777216 --codec quant8" "--numel 16777216 --codec trunc16" "--numel 67108864 --codec quant8"}; do
  echo "== $args"
  timeout 120 torchrun --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29544 tools/ring_timeline.py $args 2>&1 | grep -v -E "^W1|OMP|\*\*\*|NCCL version"
done
