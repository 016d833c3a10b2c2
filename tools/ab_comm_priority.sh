#!/bin/bash
# engine iters/s and in-step ring time vs the comm stream's priority
cd "$(dirname "$0")/.."
Q="--no-cpu-baseline --no-allreduce-sweep"
for n in 1 2 4; do
  for pr in 0 -1 -5; do
    echo "== n=$n prio=$pr"
    if [ $n -eq 1 ]; then PIPESGD_COMM_PRIORITY=$pr timeout 300 python bench.py $Q 2>/dev/null | grep '^{'
    else PIPESGD_COMM_PRIORITY=$pr timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $n $Q 2>/dev/null | grep '^{'; fi
  done
done
