#!/bin/bash
# ring timelines at the C2 gradient size on 2 GPUs (plain and engine-fused forms)
cd "$(dirname "$0")/.."
for ctas in ${CTAS:-128 0}; do
  for c in ${CODECS:-trunc16 none}; do
    for f in ${FUSED:-0 1}; do
      echo "== ctas=$ctas codec=$c fused=$f"
      timeout 120 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 tools/ring_timeline.py --numel ${NUMEL:-4710538} --codec $c --ctas $ctas --fused $f --reps 6 2>&1 | grep -v -E "^W1|OMP|\*\*\*|NCCL version"
    done
  done
done
