#!/bin/bash
# Full-GPU ring budget (592 CTAs) for the large-gradient configs, N=4.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_engine_ctas3}
mkdir -p $O
run() {  # model mode ctas steps
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29661 bench.py --gpus 4 --model $1 --mode $2 --ctas $3 --steps $4 --warmup 10 \
    --no-allreduce-sweep > $O/$1_$2_c$3.json 2> $O/$1_$2_c$3.err
}
for c in 592 384 256; do run c3 pipe_sgd $c 30; run c3 d_sync $c 30; done
for c in 592 256; do run c4 pipe_sgd $c 20; run c4 d_sync $c 20; done
