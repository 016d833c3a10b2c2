#!/bin/bash
# quant8 encode sweeping down after absmax's upward sweep: parity tests, N = 1 bench x2, ncu DRAM bytes.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_encode_down
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_engine.py tests/test_gpu_graphs.py tests/test_gpu_bounds.py tests/test_gpu_fused.py -q > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-allreduce-sweep 2>/dev/null | grep '^{' >> $O/bench_n1.jsonl; done
BENCH_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none \
  -k regex:"encode_kernel|absmax" -c 4 -f -o $O/n1_encode python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-allreduce-sweep > $O/ncu.log 2>&1
