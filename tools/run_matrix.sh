#!/bin/bash
# BASELINE.json configs on 1/2/4 GPUs of one box: one bench.py JSON line each.
#   C2 small CNN trunc16 width 2 (the bench line), C3 AlexNet quant8 width 2,
#   C4 ResNet-50 width 2 vs synchronous width 1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/matrix
NG=$(nvidia-smi -L | wc -l)
run() {  # name ngpu args...
  local name=$1 n=$2; shift 2
  if [ "$n" -gt "$NG" ]; then return; fi
  if [ "$n" -eq 1 ]; then
    timeout 600 python bench.py --gpus 1 "$@" > gpurun_out/matrix/$name.json 2> gpurun_out/matrix/$name.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29555 bench.py --gpus $n "$@" > gpurun_out/matrix/$name.json 2> gpurun_out/matrix/$name.err
  fi
  echo "$name exit $?"
}
for n in 1 2 4; do
  run c2_n$n $n --steps 50 --warmup 10 --no-cpu-baseline ${EXTRA}
done
for n in 1 2 4; do
  run c3_q8_n$n $n --model c3 --codec quant8 --global-batch 256 --steps 10 --warmup 3 --no-cpu-baseline --no-allreduce-sweep
  run c4_pipe_n$n $n --model c4 --codec none --global-batch 256 --steps 10 --warmup 3 --no-cpu-baseline --no-allreduce-sweep
  run c4_sync_n$n $n --model c4 --codec none --mode d_sync --global-batch 256 --steps 10 --warmup 3 --no-cpu-baseline --no-allreduce-sweep
done
