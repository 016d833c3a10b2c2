#!/bin/bash
# Small/mid-size ring latency at p = 4: timelines at 4 KiB / 16 KiB / 1 MiB / 2.6 MB (C1),
# codecs none and trunc16.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_small}
mkdir -p $O
for n in 1024 4096 262144 648010; do
  timeout 120 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601 tools/ring_timeline.py \
    --numel $n --codec none,trunc16,quant8 --ctas 592 --fused 0 --reps 4 2>&1 | grep '^{' >> $O/timeline_small.jsonl
done
