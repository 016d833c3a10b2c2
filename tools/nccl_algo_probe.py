"""Which algorithm / protocol NCCL picks for fp32 all_reduce at the C5 sizes on
this box (NCCL_DEBUG_SUBSYS=TUNING log lines), and its time with NVLink SHARP
(in-switch reduction) on and off, beside our ring (codec none). Run under
torchrun; env NCCL_NVLS_ENABLE=0/1 is set by the driver script."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, p = dist.get_rank(), dist.get_world_size()
s = torch.cuda.current_stream()
for n in [1 << 18, 1 << 20, 1 << 21, 1 << 22, 1 << 24, 1 << 26, 1 << 28]:
    y = torch.randn(n, device="cuda")
    it = 20 if n < (1 << 24) else 8
    for _ in range(5):
        dist.all_reduce(y)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)
    a.record(s)
    for _ in range(it):
        dist.all_reduce(y)
    b.record(s)
    b.synchronize()
    t = torch.tensor([a.elapsed_time(b) / it], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"p": p, "n": n, "bytes": 4 * n, "nccl_us": t.item() * 1e3,
                          "nvls": os.environ.get("NCCL_NVLS_ENABLE", "default"),
                          "algo_env": os.environ.get("NCCL_ALGO", ""), "proto_env": os.environ.get("NCCL_PROTO", "")}),
              flush=True)
dist.destroy_process_group()
