#!/bin/bash
# 4-GPU part of the driver view (N=2, N=4, both arms) + the e2e copy-scheduling A/B at N=4.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_driver4}
mkdir -p $O
for np in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
    --master-port 29681 bench.py --impl reference --gpus $np > $O/bench_ref_n$np.json 2> $O/bench_ref_n$np.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
    --master-port 29682 bench.py --gpus $np > $O/bench_n$np.json 2> $O/bench_n$np.err
done
for v in 0 1; do
  BENCH_COPY_AFTER_RING=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29683 bench.py --gpus 4 --no-allreduce-sweep \
    > $O/bench_n4_copy$v.json 2> $O/bench_n4_copy$v.err
done
