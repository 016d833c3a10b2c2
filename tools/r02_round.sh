#!/bin/bash
# Full GPU tests, NVLink counter probe (nvidia-smi), e2e CTA-budget A/B at N=4.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_round}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=40 --junitxml=$O/pytest_gpu.xml > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 120 python tools/nvlink_smi_probe.py > $O/nvlink_smi_probe.jsonl 2>&1
for ctas in 64 128 256; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29581 bench.py --gpus 4 --ctas $ctas --no-allreduce-sweep > $O/bench_n4_ctas$ctas.json 2> $O/bench_n4_ctas$ctas.err
done
