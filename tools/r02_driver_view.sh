#!/bin/bash
# What the driver runs at round end: pytest -m gpu, smoke(), bench N=1 (both arms);
# with >1 GPU also N=2 and N=4 for both arms.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_driver}
mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=30 --junitxml=$O/pytest_gpu_${NG}gpu.xml > $O/pytest_gpu_${NG}gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu_${NG}gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
for np in 2 4; do
  [ $np -gt $NG ] && continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
    --master-port 29671 bench.py --impl reference --gpus $np > $O/bench_ref_n$np.json 2> $O/bench_ref_n$np.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
    --master-port 29672 bench.py --gpus $np > $O/bench_n$np.json 2> $O/bench_n$np.err
done
