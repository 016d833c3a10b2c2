#!/bin/bash
# libpipesgd variants for the LL-threshold A/B (PIPESGD_LIB=...)
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
for t in ${THRESHOLDS:-0 16384 65536}; do
  nvcc $F -DPIPESGD_LL_BLOCK=$t -o variants/lib_ll$t.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu &
done
wait
ls variants
