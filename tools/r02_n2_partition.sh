#!/bin/bash
# C3 N = 2: green-context partition size for the pipelined ring (24 / 32 / 48 SMs) and D-Sync beside it.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_n2_partition
mkdir -p $O
run2() { name=$1; shift
  timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29743 bench.py --gpus 2 --no-allreduce-sweep --steps 20 "$@" > $O/$name.json 2> $O/$name.err
}
run2 sms48 --comm-sms 48 --ctas 192
run2 sms32 --comm-sms 32 --ctas 128
run2 sms24 --comm-sms 24 --ctas 96
run2 sms64 --comm-sms 64 --ctas 256
run2 dsync --mode d_sync
