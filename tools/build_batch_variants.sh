#!/bin/bash
# libpipesgd variants for the flag-protocol batch / LL threshold A/B (PIPESGD_LIB=variants/lib_<name>.so)
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
b() { name=$1; shift; nvcc $F "$@" -o variants/lib_$name.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu & }
b b512 -DPIPESGD_RING_BATCH=512
b b256 -DPIPESGD_RING_BATCH=256
b llhop1 -DPIPESGD_LL_HOP_BYTES=1048576u
b b256_llhop1 -DPIPESGD_RING_BATCH=256 -DPIPESGD_LL_HOP_BYTES=1048576u
wait
ls -la variants
