#!/bin/bash
# Large buckets: largest warp chunk 64 KiB (default) vs 128 / 256 KiB (fewer releases per byte).
cd "$(dirname "$0")/.."
O=gpurun_out/r02_maxchunk_ab
mkdir -p $O
for np in 4 2; do
  for mc in 65536 131072 262144; do
    PIPESGD_MAX_CHUNK_BYTES=$mc timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29637 \
      tools/ring_sweep.py --sizes 16777216,67108864,268435456 --codecs none,trunc16,quant8 --iters 10 --warmup 3 --check \
      > $O/p${np}_mc$mc.log 2>&1
    grep '^{' $O/p${np}_mc$mc.log > $O/p${np}_mc$mc.jsonl
  done
done
