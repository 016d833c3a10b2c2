#!/bin/bash
# One-GPU box (the driver's GPUTEST view): GPU tests incl. the per-rank ring
# with ranks sharing the GPU, then compute-sanitizer.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_gpu1}
mkdir -p $O
nvidia-smi -L > $O/gpus.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=40 --junitxml=$O/pytest_gpu.xml > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
[ -n "$NO_SANITIZE" ] || bash tools/sanitize.sh
