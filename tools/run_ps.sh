#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/matrix
NG=$(nvidia-smi -L | wc -l)
Q="--no-cpu-baseline --no-allreduce-sweep"
for n in 1 2 4; do
  [ $n -gt $NG ] && continue
  for cfg in "c2_ps --mode ps_sync --steps 100 --warmup 10" "c3_ps --model c3 --codec quant8 --mode ps_sync --global-batch 256 --steps 20 --warmup 5"; do
    set -- $cfg; name=${1}_n$n; shift
    if [ $n -eq 1 ]; then timeout 600 python bench.py --gpus 1 "$@" $Q > gpurun_out/matrix/$name.json 2> gpurun_out/matrix/$name.err
    else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $n "$@" $Q > gpurun_out/matrix/$name.json 2> gpurun_out/matrix/$name.err; fi
    echo "$name exit $?"
  done
done
