#!/bin/bash
# ring sweep vs minimum chunk payload (raw JSON lines)
cd "$(dirname "$0")/.."
NP=${NP:-2}
for mb in ${MINB:-4096 16384 32768}; do
 for ctas in ${CTAS:-64 148}; do
  echo "== ctas=$ctas minbytes=$mb"
  PIPESGD_MIN_CHUNK_BYTES=$mb timeout 300 torchrun --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29512 tools/ring_sweep.py --sizes ${SIZES:-1048576,4194304,16777216,67108864} --codecs ${CODECS:-none,trunc16,quant8} --ctas $ctas --iters 10 2>&1 | grep '^{'
 done
done
