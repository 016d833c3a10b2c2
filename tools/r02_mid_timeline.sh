#!/bin/bash
# p = 4 mid-size codec none: per-warp timeline of the direct reduce-scatter (flag protocol) vs the ring form.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_mid_timeline
mkdir -p $O
T="timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517"
$T tools/ring_timeline.py --numel 2097152 --codec none,trunc16 > $O/p4_2M.log 2>&1
PIPESGD_DIRECT=0 $T tools/ring_timeline.py --numel 2097152 --codec none > $O/p4_2M_ring.log 2>&1
$T tools/ring_timeline.py --numel 4194304 --codec none > $O/p4_4M.log 2>&1
PIPESGD_DIRECT=0 $T tools/ring_sweep.py --sizes 1048576,2097152,4194304,8388608 --codecs none --iters 30 > $O/p4_ring_sweep.log 2>&1
