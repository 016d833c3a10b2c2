#!/bin/bash
# LL chunk size A/B (PIPESGD_LL_CHUNK: elements per LL chunk, 0 = the
# flag-protocol chunk) at small and mid sizes, p = 4 and 2, NCCL beside it.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_llchunk}
mkdir -p $O
for np in 4 2; do
  for ch in 0 256 128 64; do
    echo "{\"lag\": \"llchunk=$ch\"}" >> $O/sweep.jsonl
    PIPESGD_LL_CHUNK=$ch timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29611 \
      tools/ring_sweep.py --sizes 256,1024,4096,16384,65536,262144,648010,1048576 --codecs none,trunc16,quant8 \
      --ctas 592 --iters 20 --warmup 5 --check $([ $ch = 0 ] && echo --nccl) 2>&1 | grep '^{' >> $O/sweep.jsonl
  done
done
