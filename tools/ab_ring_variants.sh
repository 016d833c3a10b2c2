#!/bin/bash
# ring sweep + engine bench per ring variant library (2 GPUs)
cd "$(dirname "$0")/.."
for L in variants/lib_r_*.so; do
  for ctas in 128 0; do
    echo "== ${L##*/} ctas=$ctas"
    PIPESGD_LIB=$PWD/$L timeout 300 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/ring_sweep.py --sizes 4710538,16777216,67108864 --codecs none,trunc16,quant8 --ctas $ctas --iters 20 --check 2>&1 | grep '^{'
  done
  echo "== ${L##*/} bench"
  PIPESGD_LIB=$PWD/$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-cpu-baseline --no-allreduce-sweep 2>/dev/null | grep '^{'
done
