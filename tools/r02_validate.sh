#!/bin/bash
# Round-2 validation on one box: GPU tests with test IDs and durations
# (junit XML), smoke(), bench N=1 (driver default) and N=all GPUs.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_validate}
mkdir -p $O
nvidia-smi -L > $O/gpus.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=40 --junitxml=$O/pytest_gpu.xml > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench1 exit $?" >> $O/bench_n1.err
NG=$(nvidia-smi -L | wc -l)
if [ "$NG" -gt 1 ]; then
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG > $O/bench_n$NG.json 2> $O/bench_n$NG.err; echo "bench exit $?" >> $O/bench_n$NG.err
fi
