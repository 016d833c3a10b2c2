#!/bin/bash
# Engine comm CTA budget A/B: C1 (comm-heavy MLP) Pipe-SGD vs D-Sync, N=4, ring budgets
# 16 / 32 / 64 / 256 CTAs; then the LL threshold A/B.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_engine_ctas}
mkdir -p $O
for ctas in 16 32 64 256; do
  for mode in pipe_sgd d_sync; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29641 bench.py --gpus 4 --model c1 --mode $mode --ctas $ctas --steps 200 --warmup 10 \
      --no-allreduce-sweep > $O/c1_${mode}_c$ctas.json 2> $O/c1_${mode}_c$ctas.err
  done
done
bash tools/r02_llhop_ab.sh
