#!/bin/bash
# ring time vs chunks per warp (PIPESGD_CHUNKS_PER_WARP) at the standalone CTA budget
cd "$(dirname "$0")/.."
for np in ${NPS:-2 4}; do
  for cpw in ${CPW:-1 2 4 8}; do
    echo "== p=$np cpw=$cpw"
    PIPESGD_CHUNKS_PER_WARP=$cpw timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29512 tools/ring_sweep.py --sizes ${SIZES:-4194304,16777216,67108864,268435456} --codecs ${CODECS:-none,trunc16,quant8} --iters 10 2>&1 | grep '^{'
  done
done
