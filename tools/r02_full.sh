#!/bin/bash
# Full GPU validation + NVLink counters + bench lines (pipe / d_sync, N = 2, 4).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_full}
mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=40 --junitxml=$O/pytest_gpu.xml > $O/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu.log
fi
timeout 300 python tools/nvlink_probe.py > $O/nvlink_probe.jsonl 2> $O/nvlink_probe.err
for np in 2 4; do
  [ $np -gt $NG ] && continue
  timeout 600 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29571 tools/nvlink_traffic.py \
    > $O/nvlink_traffic_p$np.log 2>&1
done
for np in 4 2; do
  [ $np -gt $NG ] && continue
  for mode in pipe_sgd d_sync; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
      --master-port 29572 bench.py --gpus $np --mode $mode > $O/bench_n${np}_$mode.json 2> $O/bench_n${np}_$mode.err
  done
done
