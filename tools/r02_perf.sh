#!/bin/bash
# Quick A/B loop: parity subset, then the ring at the C3 / 1 GiB / mid sizes,
# p = 4 and 2, engine (256) and full (592) CTA budgets, NCCL beside it.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_perf}
mkdir -p $O
if [ -z "$NO_TESTS" ]; then
  timeout 900 python -m pytest -x -q ${TESTS:-tests/test_gpu_codec.py tests/test_gpu_ring.py tests/test_gpu_fused.py tests/test_gpu_configs.py tests/test_gpu_stress.py tests/test_gpu_bounds.py} > $O/pytest.log 2>&1
  echo "pytest exit $?" >> $O/pytest.log
fi
NG=$(nvidia-smi -L | wc -l)
for lag in ${LAGS:-50}; do
for np in ${PS:-4 2}; do
  [ $np -gt $NG ] && continue
  for ctas in ${CTAS:-592 256}; do
    echo "{\"lag\": $lag}" >> $O/sweep.jsonl
    PIPESGD_QUEUE_LAG=$lag timeout 600 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29555 tools/ring_sweep.py \
      --sizes ${SIZES:-4194304,16777216,61100840,268435456} --codecs ${CODECS:-quant8,trunc16,none} --ctas $ctas \
      --iters 10 --warmup 3 --check $NCCL 2>&1 | grep '^{' >> $O/sweep.jsonl
  done
done
done
