#!/bin/bash
# ncu NVLink + DRAM counters of the real P2P ring kernel on GPU 0 (p = $1 GPUs,
# one process; see tools/ring_nvlink_ncu.py). Two single-pass metric lists so
# no launch is ever replayed while its peers wait.
cd "$(dirname "$0")/.."
P=${1:-2}
OUT=gpurun_out/ring_ncu_p$P
mkdir -p $OUT
timeout 300 python tools/ring_nvlink_ncu.py $P > $OUT/plain.jsonl 2> $OUT/plain.err || { echo "plain run failed"; exit 1; }
timeout 600 ncu --devices 0 -k regex:ring_allreduce --clock-control none --cache-control none \
  --metrics nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum \
  --csv --log-file $OUT/nvl.csv python tools/ring_nvlink_ncu.py $P > $OUT/ncu_nvl.jsonl 2> $OUT/ncu_nvl.err
echo "ncu nvl rc=$?"
timeout 600 ncu --devices 0 -k regex:ring_allreduce --clock-control none --cache-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --csv --log-file $OUT/dram.csv python tools/ring_nvlink_ncu.py $P > $OUT/ncu_dram.jsonl 2> $OUT/ncu_dram.err
echo "ncu dram rc=$?"
