#!/bin/bash
# libpipesgd variants for the quant8 pass-unroll A/B: VARIANTS = "load:fold ..."
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
for v in ${VARIANTS:-1:1 4:1 4:2 2:1}; do
  l=${v%%:*}; f=${v##*:}
  nvcc $F -DPIPESGD_Q8_LOAD_UNROLL=$l -DPIPESGD_Q8_FOLD_UNROLL=$f -o variants/lib_q8_l${l}_f${f}.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu &
done
wait
ls variants
