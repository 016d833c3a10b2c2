#!/bin/bash
# The pipelined ring on a green-context SM partition (--comm-sms) at C3, N=4 (sms 0 = no partition).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_green}
mkdir -p $O
run() {  # sms ctas graphs
  timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29721 bench.py --gpus 4 --comm-sms $1 --ctas $2 --graphs $3 --no-allreduce-sweep --steps 20 \
    > $O/c3_sms$1_c$2_g$3.json 2> $O/c3_sms$1_c$2_g$3.err
}
run 16 64 0
run 16 64 1
run 32 128 1

