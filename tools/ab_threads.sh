#!/bin/bash
cd "$(dirname "$0")/.."
T128=$PWD/paper_1811_03619_b200/libpipesgd_t128.so
tr() { timeout 300 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 "$@" 2>&1 | grep '^{'; }
echo "== sweep 512t ctas 32"; tr tools/ring_sweep.py --sizes 4194304,67108864 --codecs none,trunc16,quant8 --ctas 32 --iters 10
echo "== sweep 128t ctas 128"; PIPESGD_LIB=$T128 tr tools/ring_sweep.py --sizes 4194304,67108864 --codecs none,trunc16,quant8 --ctas 128 --iters 10
echo "== sweep 512t ctas 148"; tr tools/ring_sweep.py --sizes 4194304,67108864 --codecs none,trunc16,quant8 --ctas 148 --iters 10
echo "== sweep 128t ctas 592"; PIPESGD_LIB=$T128 tr tools/ring_sweep.py --sizes 4194304,67108864 --codecs none,trunc16,quant8 --ctas 592 --iters 10
for cfg in "512 32" "128 128" "128 256" "128 592"; do
  set -- $cfg
  LIB=""; [ "$1" = 128 ] && LIB=$T128
  echo "== bench c2 ${1}t ctas $2"; PIPESGD_LIB=$LIB tr bench.py --gpus 2 --steps 50 --warmup 10 --ctas $2 --no-allreduce-sweep
  echo "== bench c3 ${1}t ctas $2"; PIPESGD_LIB=$LIB tr bench.py --gpus 2 --model c3 --codec quant8 --global-batch 256 --steps 10 --warmup 3 --ctas $2 --no-allreduce-sweep
done
