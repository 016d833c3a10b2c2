#!/bin/bash
cd "$(dirname "$0")/.."
for g in 0 1; do
  for m in c2 c1; do
    GB=512; [ $m = c1 ] && GB=100
    timeout 300 python bench.py --model $m --global-batch $GB --steps 200 --warmup 20 --graphs $g --no-cpu-baseline > gpurun_out/g_${m}_n1_g$g.json 2> gpurun_out/g_${m}_n1_g$g.err
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --model $m --global-batch $GB --steps 200 --warmup 20 --graphs $g --no-allreduce-sweep > gpurun_out/g_${m}_n2_g$g.json 2> gpurun_out/g_${m}_n2_g$g.err
    echo "$m g=$g done"
  done
done
