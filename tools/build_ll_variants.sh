#!/bin/bash
# libpipesgd variants for the LL-threshold A/B (PIPESGD_LIB=...):
# THRESHOLDS = "block:region ..." in elements
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
for t in ${THRESHOLDS:-262144:262144 1048576:1048576}; do
  b=${t%%:*}; r=${t##*:}
  nvcc $F -DPIPESGD_LL_BLOCK=$b -DPIPESGD_LL_REGION=$r -o variants/lib_ll$b.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu &
done
wait
ls variants
