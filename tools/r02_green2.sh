#!/bin/bash
# Green-context comm partition sweep, N=4: C3 (24 / 32 / 48 SMs), C2 (16 / 32), C1 (16).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_green2}
mkdir -p $O
run() {  # model sms ctas steps
  timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29731 bench.py --gpus 4 --model $1 --comm-sms $2 --ctas $3 --no-allreduce-sweep --steps $4 \
    > $O/$1_sms$2_c$3.json 2> $O/$1_sms$2_c$3.err
}
run c3 24 96 20
run c3 32 128 20
run c3 48 192 20
run c2 16 64 60
run c2 32 128 60
run c1 16 64 200
run c1 8 32 200
