#!/bin/bash
# Direct reduce-scatter scheduling variants (PIPESGD_LIB=variants/lib_<name>.so)
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
b() { name=$1; shift; nvcc $F "$@" -o variants/lib_$name.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu & }
b flagstatic -DPIPESGD_FLAG_STATIC=1
b interleave -DPIPESGD_DIRECT_INTERLEAVE=1
b flagstatic_interleave -DPIPESGD_FLAG_STATIC=1 -DPIPESGD_DIRECT_INTERLEAVE=1
wait
