"""Ring AllReduce sweep under torchrun: fused compressed ring vs NCCL.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/ring_sweep.py [--sizes ...]

One process per GPU, inboxes shared over CUDA IPC (ProcessGroupTransport).
Prints one JSON line per (size, codec) on rank 0: device time per call
(CUDA events on the launching stream, max over ranks), fp32-equivalent bus
bandwidth 2(p-1)/p*4n/t (nccl-tests convention), wire bus bandwidth
2(p-1)/p*w*n/t, and NCCL all_reduce on the same buffer for comparison.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1811_03619_b200 import Codec, ProcessGroupTransport  # noqa: E402
from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait  # noqa: E402


def timed(fn, iters, warmup, stream):
    for _ in range(warmup):
        fn()
    stream.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(2_000_000)  # host enqueues the whole series before the clock starts
    a.record(stream)
    for _ in range(iters):
        fn()
    b.record(stream)
    b.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=str, default="256,4096,65536,1048576,4194304,16777216,67108864,268435456")
    ap.add_argument("--codecs", type=str, default="none,trunc16,quant8")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--nccl", action="store_true")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, p = dist.get_rank(), dist.get_world_size()
    sizes = [int(s) for s in args.sizes.split(",")]
    ep = ProcessGroupTransport.endpoint(local, max_elems=max(sizes), timeout_s=20.0, ctas=args.ctas)
    stream = torch.cuda.current_stream()
    for n in sizes:
        g = torch.Generator(device="cuda").manual_seed(1000 * rank + n % 997)
        x = torch.randn(n, device="cuda", generator=g)
        out = torch.empty_like(x)
        for cname in args.codecs.split(","):
            codec = Codec.parse(cname)
            it = max(3, min(args.iters, int(4e9 // max(1, 8 * n))))

            def run():
                allreduce_into(x, out, ep, codec, 0, stream)

            t = timed(run, it, args.warmup, stream)
            endpoint_wait(ep, n, stream)
            rec = {"p": p, "n": n, "bytes": 4 * n, "codec": cname, "ms": t * 1e3,
                   "busbw_gbs": 2 * (p - 1) / p * 4 * n / t / 1e9,
                   "wire_busbw_gbs": 2 * (p - 1) / p * codec.bytes_per_elem * n / t / 1e9,
                   "ctas": ep.info()["ctas"]}
            if args.check:  # every rank holds the same bits (oracle parity: tests/test_gpu_ring.py)
                allreduce_into(x, out, ep, codec, 0, stream)
                endpoint_wait(ep, n, stream)
                ref = out.clone()
                dist.broadcast(ref, 0)
                same = torch.tensor([int(torch.equal(ref.view(torch.int32), out.view(torch.int32)))], device="cuda")
                dist.all_reduce(same, op=dist.ReduceOp.MIN)
                rec["replicas_bit_identical"] = bool(same.item())
            if rank == 0:
                print(json.dumps(rec), flush=True)
        if args.nccl:
            y = x.clone()
            t = timed(lambda: dist.all_reduce(y), max(3, min(args.iters, int(4e9 // max(1, 8 * n)))), args.warmup, stream)
            if rank == 0:
                print(json.dumps({"p": p, "n": n, "bytes": 4 * n, "codec": "nccl", "ms": t * 1e3,
                                  "busbw_gbs": 2 * (p - 1) / p * 4 * n / t / 1e9}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
