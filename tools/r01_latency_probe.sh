#!/bin/bash
# codec-kernel variants (1 GPU) + ring timelines at the C2 gradient size (2 GPUs)
cd "$(dirname "$0")/.."
for L in variants/lib_*.so; do PIPESGD_LIB=$PWD/$L timeout 120 python tools/kernel_micro.py; done > gpurun_out/cu_variants.jsonl 2>gpurun_out/cu_variants.err
echo "micro $?"
for ctas in 128 0; do
  for c in trunc16 none quant8; do
    echo "== ctas=$ctas codec=$c"
    timeout 120 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 tools/ring_timeline.py --numel 4710538 --codec $c --ctas $ctas --reps 6 2>&1 | grep -v -E "^W1|OMP|\*\*\*|NCCL version"
  done
done > gpurun_out/timeline_c2.log 2>&1
echo "timeline $?"
