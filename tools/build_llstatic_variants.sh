#!/bin/bash
# LL chunk scheduling (static stride vs phase counter) and LL slot size variants (PIPESGD_LIB=variants/lib_<name>.so)
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
b() { name=$1; shift; nvcc $F "$@" -o variants/lib_$name.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu & }
b lldyn -DPIPESGD_LL_STATIC=0
b llreg4s -DPIPESGD_LL_REGION_BYTES=4194304u -DPIPESGD_LL_HOP_BYTES=1572864u
b llreg8s -DPIPESGD_LL_REGION_BYTES=8388608u -DPIPESGD_LL_HOP_BYTES=4194304u
wait
