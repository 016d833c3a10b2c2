#!/bin/bash
cd "$(dirname "$0")/.."
tr() { timeout 300 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 "$@" 2>&1 | grep '^{'; }
for LIB in "" "$PWD/paper_1811_03619_b200/libpipesgd_q8b.so"; do
  echo "== lib=${LIB##*/}"
  PIPESGD_LIB=$LIB tr tools/ring_sweep.py --sizes 4194304,16777216,67108864 --codecs quant8,trunc16 --iters 10 --check
done
