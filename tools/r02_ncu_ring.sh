#!/bin/bash
# ncu --set full (source counters) of one emulated ring call per codec at the
# C3 gradient size (p ranks in one cooperative launch on GPU 0), fused form.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_ncu_ring}
mkdir -p $O
for c in ${CODECS:-quant8}; do
  P=${P:-4} N=${N:-61100840} CODECS=$c timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:ring_allreduce -c 1 -f -o $O/ring_${c}_p${P:-4} python tools/ring_fused_once.py > $O/ncu_${c}.log 2>&1
  echo "exit $?" >> $O/ncu_${c}.log
done
