#!/bin/bash
cd "$(dirname "$0")/.."
NP=${NP:-2}
for L in 0 1; do
for args in ${RUNS:-"--numel 65536 --codec none" "--numel 4194304 --codec trunc16"}; do
  echo "== launch=$L $args"
  PIPESGD_LAUNCH=$L timeout 120 torchrun --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29544 tools/ring_timeline.py $args 2>&1 | grep -v -E "^W1|OMP|\*\*\*|NCCL version"
done
done
