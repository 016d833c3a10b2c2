#!/bin/bash
# BASELINE.json configs on 1/2/4 GPUs of one box: one bench.py JSON line each.
#   C1 MLP (width 2, none), C2 small CNN trunc16 (the bench line) with the
#   paper's three schemes, C3 AlexNet quant8 three schemes, C4 ResNet-50
#   width 2 vs width 1.
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
Q="--no-cpu-baseline --no-allreduce-sweep"
for n in 1 2 4; do
  run c1_pipe_n$n $n --model c1 --codec none --global-batch 100 --steps 300 --warmup 30 $Q
  run c1_sync_n$n $n --model c1 --codec none --mode d_sync --global-batch 100 --steps 300 --warmup 30 $Q
  run c2_pipe_n$n $n --steps 100 --warmup 10 $Q
  run c2_pipe_eager_n$n $n --graphs 0 --steps 100 --warmup 10 $Q
  run c2_sync_n$n $n --mode d_sync --steps 100 --warmup 10 $Q
  run c2_sync_eager_n$n $n --mode d_sync --graphs 0 --steps 100 --warmup 10 $Q
  run c2_ps_n$n $n --mode ps_sync --steps 100 --warmup 10 $Q
  run c3_pipe_n$n $n --model c3 --codec quant8 --global-batch 256 --steps 20 --warmup 5 $Q
  run c3_sync_n$n $n --model c3 --codec quant8 --mode d_sync --global-batch 256 --steps 20 --warmup 5 $Q
  run c3_sync_eager_n$n $n --model c3 --codec quant8 --mode d_sync --graphs 0 --global-batch 256 --steps 20 --warmup 5 $Q
  run c3_ps_n$n $n --model c3 --codec quant8 --mode ps_sync --global-batch 256 --steps 20 --warmup 5 $Q
  run c4_pipe_n$n $n --model c4 --codec none --global-batch 256 --steps 10 --warmup 3 $Q
  run c3_pipe_eager_n$n $n --model c3 --codec quant8 --graphs 0 --global-batch 256 --steps 20 --warmup 5 $Q
  run c4_sync_n$n $n --model c4 --codec none --mode d_sync --global-batch 256 --steps 10 --warmup 3 $Q
done
