#!/bin/bash
# ring sweep under several CTA / chunks-per-warp settings (raw JSON lines)
cd "$(dirname "$0")/.."
NP=${NP:-2}
for cpw in ${CPW:-1 2 4}; do
 for ctas in ${CTAS:-32 64 148}; do
  echo "== ctas=$ctas cpw=$cpw"
  PIPESGD_CHUNKS_PER_WARP=$cpw timeout 300 torchrun --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29512 tools/ring_sweep.py --sizes ${SIZES:-16777216,67108864} --codecs ${CODECS:-none,trunc16,quant8} --ctas $ctas --iters 10 2>&1 | grep '^{'
 done
done
