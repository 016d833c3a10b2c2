#!/bin/bash
# engine iters/s vs the ring's CTA budget inside the pipeline
cd "$(dirname "$0")/.."
Q="--no-cpu-baseline --no-allreduce-sweep"
for n in 2 4; do
  for c in ${CTAS_LIST:-32 64 128 256}; do
    echo "== n=$n ctas=$c"
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $n --ctas $c --steps 100 --warmup 10 $Q 2>/dev/null | grep '^{'
  done
done
