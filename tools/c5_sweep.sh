#!/bin/bash
# ring sweep 1 KB - 1 GB fp32 (2^8..2^28 elements) plus
# non-divisible sizes, x {none, trunc16, quant8} x p in {2, 4}, NCCL fp32
# allreduce beside it, replica bit-identity checked, SM clocks per series,
# Eq. 5 prediction per row (GPU-calibrated alpha / beta / gamma / S) and the
# reference's CPU ring (baseline/_ref, p threads) up to 2^24 elements. JSON lines.
cd "$(dirname "$0")/.."
O=${OUT:-gpurun_out/c5}
mkdir -p $O
S=""
for k in $(seq 8 28); do S="$S,$((1 << k))"; done
S="${S#,},4099,1048579,16777219"
NG=$(nvidia-smi -L | wc -l)
for np in 2 4; do
  [ $np -gt $NG ] && continue
  echo "== p=$np"
  timeout 1500 torchrun --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29513 tools/ring_sweep.py \
    --sizes $S --iters 20 --warmup 5 --check --nccl --clocks --eq5 --cpu-ref-max ${CPU_MAX:-16777216} \
    > $O/c5_p$np.log 2>&1
  grep '^{' $O/c5_p$np.log > $O/c5_p$np.jsonl
done
