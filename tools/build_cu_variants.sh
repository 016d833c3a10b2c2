#!/bin/bash
# libpipesgd variants for the codec-kernel A/B (tools/kernel_micro.py)
cd "$(dirname "$0")/.."
C=paper_1811_03619_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -Xcompiler -fPIC -shared -I$C"
mkdir -p variants
# (the round-1 A/B also built the previous codec_kernels.cu as lib_old.so from git history:
#  git show <rev>:paper_1811_03619_b200/csrc/codec_kernels.cu > <dir>/codec_kernels.cu)
for v in "16 1" "16 4" "32 1" "8 1" "8 4"; do set -- $v
  nvcc $F -DPIPESGD_CU_ELEMS=$1 -DPIPESGD_CU_MINB=$2 -o variants/lib_e$1_m$2.so $C/ring.cu $C/star.cu $C/comm.cu $C/codec_kernels.cu $C/calib.cu &
done
wait
ls variants
