#!/bin/bash
# Final 4-GPU evidence: pytest -m gpu (junit), quick ring-vs-NCCL sweep, and the driver's N = 2 / 4 benches (both arms).
cd "$(dirname "$0")/.."
O=gpurun_out/r02_final_4gpu
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=30 --junitxml=$O/pytest_gpu_4gpu.xml > $O/pytest_gpu_4gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu_4gpu.log
TAG=r02_final_4gpu/quick_c5 bash tools/r02_quick_c5.sh
TAG=r02_final_4gpu bash tools/r02_driver4.sh
