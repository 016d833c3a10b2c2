#!/bin/bash
# Pipe-SGD comm CTA budget for C2 / C3 (and C1 at 128), N=4.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_engine_ctas2}
mkdir -p $O
run() {  # model mode ctas steps
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29651 bench.py --gpus 4 --model $1 --mode $2 --ctas $3 --steps $4 --warmup 10 \
    --no-allreduce-sweep > $O/$1_$2_c$3.json 2> $O/$1_$2_c$3.err
}
run c1 pipe_sgd 128 200
run c1 pipe_sgd 64 200
for c in 64 128 256; do run c2 pipe_sgd $c 60; done
run c2 d_sync 256 60
for c in 64 128 256; do run c3 pipe_sgd $c 30; done
run c3 d_sync 256 30
