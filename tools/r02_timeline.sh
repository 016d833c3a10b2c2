#!/bin/bash
# Per-warp ring timelines (tools/ring_timeline.py) at the C3 gradient size:
# p = 2 and 4, every codec, plain and engine-fused, engine and full CTA budgets.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_timeline}
mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
for np in ${PS:-4 2}; do
  [ $np -gt $NG ] && continue
  for ctas in ${CTAS:-256 592}; do
    timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29544 tools/ring_timeline.py \
      --numel ${NUMEL:-61100840} --codec ${CODECS:-quant8,trunc16,none} --ctas $ctas --fused ${FUSED:-0,1} --reps 4 \
      2>&1 | grep '^{' >> $O/timeline.jsonl
  done
done
