#!/bin/bash
# N = 1 C3: comm-stream priority vs the live HBM fraction of the encode kernels and iterations/s.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_prio_n1
mkdir -p $O
for pr in 0 -5 0 -5; do
  PIPESGD_COMM_PRIORITY=$pr timeout 300 python bench.py --no-cpu-baseline --no-allreduce-sweep 2>/dev/null | grep '^{' >> $O/prio_$pr.jsonl
done
