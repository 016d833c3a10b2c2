#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (codec kernels, emulated ring
# on both wire protocols, direct reduce-scatter, fused variants, star).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_sanitize}
mkdir -p $O
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  timeout ${TMO:-1200} /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 100 --error-exitcode 9 \
    python tools/sanitize_cases.py > $O/$tool.log 2>&1
  echo "exit $?" >> $O/$tool.log
done
