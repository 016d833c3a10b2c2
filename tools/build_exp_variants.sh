#!/bin/bash
# Timing-only experiment variants (PIPESGD_LIB=variants/lib_<name>.so); not for parity.
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
b() { name=$1; shift; nvcc $F "$@" -o variants/lib_$name.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu & }
b nofence -DPIPESGD_EXP_NOFENCE
b nofence_llhop1 -DPIPESGD_EXP_NOFENCE -DPIPESGD_LL_HOP_BYTES=1048576u
wait
