#!/bin/bash
# p=2 small-message: codec none vs trunc16 (timeline + back-to-back, codec order swapped, LL chunk variants)
cd "$(dirname "$0")/.."
O=gpurun_out/r02_p2small
mkdir -p $O
T="timeout 300 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516"
$T tools/ring_timeline.py --numel 4096 --codec none,trunc16 > $O/timeline.log 2>&1
$T tools/ring_sweep.py --sizes 4096,262144 --codecs trunc16,none,trunc16,none --iters 50 > $O/order.log 2>&1
PIPESGD_LL_CHUNK=256 $T tools/ring_sweep.py --sizes 4096,262144 --codecs none,trunc16 --iters 50 > $O/ll256.log 2>&1
PIPESGD_LL_CHUNK=64 $T tools/ring_sweep.py --sizes 4096,262144 --codecs none,trunc16 --iters 50 > $O/ll64.log 2>&1
