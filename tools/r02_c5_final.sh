#!/bin/bash
# Final round-2 C5 sweep (clocks, Eq. 5 + extension, CPU reference) and the C1 / C3 N = 4 benches.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_c5_final
mkdir -p $O
timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 \
  bench.py --gpus 4 --model c1 --no-allreduce-sweep --steps 200 > $O/bench_c1_n4.json 2> $O/bench_c1_n4.err
OUT=$O CPU_MAX=${CPU_MAX:-4194304} bash tools/c5_sweep.sh > $O/c5.log 2>&1
