"""Measured NVLink bytes of the fused ring (NVML per-GPU NVLink data
counters, paper_1811_03619_b200/nvlink.py) around K back-to-back ring calls,
against the algorithmic wire bytes per rank W = 2(p-1)/p * n * w (LL
protocol: 2W, every 8-byte word carries 4 payload bytes).

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/nvlink_traffic.py

Sizes: the BASELINE configs' gradients (C1 648,010 / C2 4,710,538 / C3
61,100,840 / C4 25,557,032 fp32) and a 256 MiB bucket, every codec. One JSON
line per (size, codec) on rank 0 with every rank's TX/RX deltas per call.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import Codec, ProcessGroupTransport, _lib  # noqa: E402
from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait, partition_blocks  # noqa: E402
from paper_1811_03619_b200.nvlink import NvlinkCounters  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="648010,4710538,25557032,61100840,67108864")
ap.add_argument("--codecs", default="none,trunc16,quant8")
ap.add_argument("--calls", type=int, default=10)
ap.add_argument("--ctas", type=int, default=0)
a = ap.parse_args()
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, p = dist.get_rank(), dist.get_world_size()
sizes = [int(x) for x in a.sizes.split(",")]
ep = ProcessGroupTransport.endpoint(local, max_elems=max(sizes), timeout_s=30.0, ctas=a.ctas)
cnt = NvlinkCounters(local)
s = torch.cuda.current_stream()
for n in sizes:
    x = torch.randn(n, device="cuda")
    y = torch.empty_like(x)
    for cname in a.codecs.split(","):
        codec = Codec.parse(cname)
        w = codec.bytes_per_elem
        plan = (torch.zeros(5, dtype=torch.int64))
        import ctypes
        o = (ctypes.c_int64 * 5)()
        _lib.call("gp_ring_plan", n, p, ep.info()["ctas"], int(codec), 0, n, o)
        ll = bool(o[2])
        for _ in range(2):
            allreduce_into(x, y, ep, codec, 0, s)
        endpoint_wait(ep, n, s)
        dist.barrier()
        cnt.start()
        for _ in range(a.calls):
            allreduce_into(x, y, ep, codec, 0, s)
        endpoint_wait(ep, n, s)
        torch.cuda.synchronize()
        dist.barrier()
        d = cnt.delta()
        blocks = partition_blocks(n, p)
        wire = (sum(blocks[(rank - t) % p][1] for t in range(p - 1)) +
                sum(blocks[(rank + 1 - t) % p][1] for t in range(p - 1))) * w
        rec = {"rank": rank, "tx_per_call": d.get("data_tx", 0) / a.calls, "rx_per_call": d.get("data_rx", 0) / a.calls,
               "raw_tx_per_call": d.get("raw_tx", 0) / a.calls, "algorithmic_wire_per_call": wire,
               "expected_on_wire": wire * (2 if ll else 1)}
        allr = [None] * p
        dist.all_gather_object(allr, rec)
        if rank == 0:
            tx = sum(r["tx_per_call"] for r in allr) / p
            exp = sum(r["expected_on_wire"] for r in allr) / p
            print(json.dumps({"p": p, "n": n, "codec": cname, "protocol": "LL" if ll else "flag", "calls": a.calls,
                              "mean_tx_bytes_per_call": tx, "algorithmic_wire_bytes": sum(
                                  r["algorithmic_wire_per_call"] for r in allr) / p,
                              "expected_bytes_incl_protocol": exp, "measured_over_expected": tx / exp if exp else None,
                              "ranks": allr}), flush=True)
dist.barrier()
dist.destroy_process_group()
