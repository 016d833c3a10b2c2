#!/bin/bash
# quant8 LL protocol at large blocks (A/B): the LL-region variant library with
# the quant8 LL limit raised vs the same library at the default limit.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_q8ll}
mkdir -p $O
LIB=$PWD/variants/lib_ll128.so
for np in 4 2; do
  for q8ll in 0 134217728; do
    echo "{\"lag\": \"q8ll=$q8ll\"}" >> $O/sweep.jsonl
    PIPESGD_LIB=$LIB PIPESGD_Q8_LL_BYTES=$q8ll timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 \
      --master-port 29561 tools/ring_sweep.py --sizes 4194304,16777216,61100840,268435456 --codecs quant8 --ctas 592 \
      --iters 10 --warmup 3 --check 2>&1 | grep '^{' >> $O/sweep.jsonl
  done
done
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 tools/ring_sweep.py \
  --sizes 1024,4194304,61100840 --codecs quant8,trunc16,none --ctas 592 --iters 10 --warmup 3 --check --nccl \
  --clocks --eq5 --cpu-ref-max 4194304 > $O/eq5_sweep.log 2>&1
grep '^{' $O/eq5_sweep.log > $O/eq5_sweep.jsonl
