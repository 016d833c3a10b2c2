#!/bin/bash
# run the 2-GPU sweep at large sizes under several CTA / chunk settings (raw JSON lines)
cd "$(dirname "$0")/.."
NP=${NP:-2}
for ch in ${CHUNKS:-16384 65536}; do
 for ctas in ${CTAS:-32 64 148}; do
  echo "== ctas=$ctas chunk=$ch"
  PIPESGD_MAX_CHUNK=$ch timeout 300 torchrun --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29512 tools/ring_sweep.py --sizes ${SIZES:-16777216,67108864} --codecs none,trunc16,quant8 --ctas $ctas --iters 10 2>&1 | grep '^{'
 done
done
