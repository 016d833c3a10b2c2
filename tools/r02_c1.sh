#!/bin/bash
# Full GPU tests, then the comm-heavy C1 MLP and the C2 CNN at N=4 (Pipe-SGD vs D-Sync).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_c1}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=30 --junitxml=$O/pytest_gpu.xml > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
for model in c1 c2; do
  for mode in pipe_sgd d_sync; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29621 bench.py --gpus 4 --model $model --mode $mode --steps 100 --warmup 10 \
      > $O/bench_n4_${model}_$mode.json 2> $O/bench_n4_${model}_$mode.err
  done
done
