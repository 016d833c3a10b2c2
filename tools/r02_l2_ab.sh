#!/bin/bash
# L2 eviction-policy A/B for the ring's pass-A loads: does the evict_last
# pinning slow the CNN compute overlapping the ring (Pipe-SGD e2e at C3, N=4)?
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_l2}
mkdir -p $O
for v in default l2keep0 l2keep2; do
  if [ $v = default ]; then L=$PWD/paper_1811_03619_b200/libpipesgd.so; else L=$PWD/variants/lib_$v.so; fi
  PIPESGD_LIB=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29595 bench.py --gpus 4 --no-allreduce-sweep > $O/bench_pipe_$v.json 2> $O/bench_pipe_$v.err
  echo "{\"lag\": \"$v\"}" >> $O/sweep.jsonl
  PIPESGD_LIB=$L timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596 tools/ring_sweep.py \
    --sizes 16777216,61100840,268435456 --codecs quant8 --ctas 592 --iters 10 --warmup 3 --check 2>&1 | grep '^{' >> $O/sweep.jsonl
done
