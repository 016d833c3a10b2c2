#!/bin/bash
# NCCL's algorithm choice at p = 4 (TUNING log) and its times with / without NVLS and per protocol.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_nccl_algo
mkdir -p $O
T="timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 tools/nccl_algo_probe.py"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING $T > $O/default.log 2>&1
NCCL_NVLS_ENABLE=0 $T > $O/nvls0.log 2>&1
NCCL_NVLS_ENABLE=0 NCCL_PROTO=Simple $T > $O/nvls0_simple.log 2>&1
NCCL_NVLS_ENABLE=0 NCCL_PROTO=LL128 $T > $O/nvls0_ll128.log 2>&1
NCCL_ALGO=Ring NCCL_PROTO=Simple $T > $O/ring_simple.log 2>&1
