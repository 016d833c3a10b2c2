#!/bin/bash
# Quick ring-vs-NCCL check at the current HEAD (no Eq. 5 / CPU columns): p = 2, 4.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_quick_c5}
mkdir -p $O
S=256,4096,65536,262144,648010,1048576,2097152,4194304,8388608,16777216,25557032,67108864
for np in 2 4; do
  timeout 600 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29515 tools/ring_sweep.py \
    --sizes $S --iters 30 --warmup 5 --nccl --codecs ${CODECS:-none,trunc16,quant8} > $O/p$np.log 2>&1
  grep '^{' $O/p$np.log > $O/p$np.jsonl
done
