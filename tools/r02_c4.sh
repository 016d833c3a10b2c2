#!/bin/bash
# C4 ResNet-50 (codec none): N = 1 and N = 4, Pipe-SGD (engine policy) vs D-Sync.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_c4
mkdir -p $O
timeout 600 python bench.py --model c4 --no-cpu-baseline --no-allreduce-sweep --steps 10 > $O/c4_n1_pipe.json 2> $O/c4_n1_pipe.err
for m in pipe_sgd d_sync; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29745 \
    bench.py --gpus 4 --model c4 --mode $m --no-allreduce-sweep --steps 10 > $O/c4_n4_$m.json 2> $O/c4_n4_$m.err
done
