#!/bin/bash
# libpipesgd variants for the ring batch / register-budget A/B (PIPESGD_LIB=...)
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
for v in ${VARIANTS:-"1024 4 1" "2048 2 1" "2048 2 2"}; do set -- $v
  nvcc $F -DPIPESGD_RING_BATCH=$1 -DPIPESGD_RING_MINBLOCKS=$2 -DPIPESGD_Q8_UNROLL=$3 -o variants/lib_r_b$1_m$2_q$3.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu &
done
wait
ls variants
