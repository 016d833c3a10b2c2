#!/bin/bash
# p = 4, 12 MiB codec none: per-warp timeline with the LL protocol (4 MiB LL slot variant) vs the flag protocol.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_ll_large_timeline
mkdir -p $O
T="timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 tools/ring_timeline.py --numel 3145728 --codec none"
PIPESGD_LIB=$PWD/variants/lib_llreg4s.so $T > $O/ll.log 2>&1
$T > $O/flag.log 2>&1
