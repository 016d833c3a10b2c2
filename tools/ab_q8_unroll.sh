#!/bin/bash
cd "$(dirname "$0")/.."
for np in ${NPS:-2 4}; do
  for L in variants/lib_q8_*.so; do
    echo "== p=$np ${L##*/}"
    PIPESGD_LIB=$PWD/$L timeout 300 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29512 tools/ring_sweep.py --sizes ${SIZES:-4194304,16777216,67108864} --codecs quant8 --iters 10 --check 2>&1 | grep '^{'
  done
done
