#!/bin/bash
# LL chunk (elements per warp) re-measured with the round's LL code: 128 (default) / 256 / 512, C1-size and mid LL sizes.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_llchunk2_ab
mkdir -p $O
for np in 4 2; do
  for ch in 128 256 512; do
    for rep in 1 2; do
      PIPESGD_LL_CHUNK=$ch timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29643 \
        tools/ring_sweep.py --sizes 16384,262144,648010,1048576,2097152 --codecs none,trunc16 --iters 40 --warmup 5 \
        2>/dev/null | grep '^{' | sed "s/^{/{\"llchunk\": $ch, \"rep\": $rep, /" >> $O/sweep.jsonl
    done
  done
done
