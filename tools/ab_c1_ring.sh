#!/bin/bash
# C1 (comm-bound) Pipe-SGD at N=4 vs the ring's CTA budget and the comm stream priority
cd "$(dirname "$0")/.."
Q="--no-cpu-baseline --no-allreduce-sweep --model c1 --codec none --global-batch 100 --steps 300 --warmup 30"
for c in 128 256 592; do
  for pr in 0 -1; do
    echo "== ctas=$c prio=$pr"
    PIPESGD_COMM_PRIORITY=$pr timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 4 --ctas $c $Q 2>/dev/null | grep '^{'
  done
done
