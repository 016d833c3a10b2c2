#!/bin/bash
# quant8 groups per lane / register budget variants (PIPESGD_LIB=variants/lib_<name>.so)
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
b() { name=$1; shift; nvcc $F "$@" -o variants/lib_$name.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu & }
b q8u2_m3 -DPIPESGD_Q8_UNROLL=2 -DPIPESGD_RING_MINBLOCKS=3
b q8u2_m2 -DPIPESGD_Q8_UNROLL=2 -DPIPESGD_RING_MINBLOCKS=2
b m3 -DPIPESGD_RING_MINBLOCKS=3
wait
