#!/bin/bash
# libpipesgd variants for the LL-threshold A/B (PIPESGD_LIB=...): HOPS = bytes per hop
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
for h in ${HOPS:-524288 1048576}; do
  nvcc $F -DPIPESGD_LL_HOP_BYTES=$h -o variants/lib_ll$h.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu &
done
wait
ls variants
