#!/bin/bash
# codec kernels vs grid size (CTAs per SM cap), one GPU
cd "$(dirname "$0")/.."
for g in ${GRIDS:-4 5 8 16}; do
  echo "== grid_per_sm=$g"
  PIPESGD_CU_GRID_PER_SM=$g timeout 120 python tools/kernel_micro.py 2>/dev/null
done
