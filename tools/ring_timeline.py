"""Per-warp timeline of one ring call (torchrun, one process per GPU).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/ring_timeline.py --n 4194304 --codec trunc16

Prints, for rank 0, percentiles over warps of each phase stamp relative to
the earliest kernel start on that GPU (us), plus the CUDA-event time of the
same call, so launch overhead / flag latency / streaming time separate.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import Codec, ProcessGroupTransport, _lib  # noqa: E402
from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--numel", type=int, default=1 << 22)
ap.add_argument("--codec", default="trunc16", help="comma list")
ap.add_argument("--ctas", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--fused", default="0", help="comma list; 1 = engine form: precompress + compressed slot output")
a = ap.parse_args()
SLOTS = 44  # csrc/ring.cuh kTraceSlots
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, p = dist.get_rank(), dist.get_world_size()
ep = ProcessGroupTransport.endpoint(local, max_elems=a.numel, ctas=a.ctas, timeout_s=20)
G = ep.info()["ctas"]
W = G * 4
tr = torch.zeros(W * SLOTS, dtype=torch.int64, device="cuda")
x = torch.randn(a.numel, device="cuda") * 1e-2
y = torch.empty_like(x)
names = {0: "start", 1: "send0_done", 2: "q8_max_barrier_open", 35: "ag_first_in", 36: "end"}
for s_ in range(p - 1):
    names.update({3 + 4 * s_: f"s{s_}_first_in", 4 + 4 * s_: f"s{s_}_q8_passA_done",
                  5 + 4 * s_: f"s{s_}_q8_barrier_open", 6 + 4 * s_: f"s{s_}_done"})
if p == 2:
    names.update({37: "fold_first_grab", 38: "fold_first_data_done", 39: "fold_first_published",
                  40: "send_first_data_done", 41: "send_first_published", 42: "ag_first_grab"})
s = torch.cuda.current_stream()
for cname in a.codec.split(","):
    codec = Codec.parse(cname)
    slot = torch.empty(a.numel * codec.bytes_per_elem, dtype=torch.uint8, device="cuda")
    slot_scale = torch.empty(1, device="cuda")
    for fused in [int(f) for f in a.fused.split(",")]:
        kw = dict(precompress=True, slot=slot, slot_scale=slot_scale) if fused else {}
        for _ in range(3):
            allreduce_into(x, y, ep, codec, 0, s, **kw)
        endpoint_wait(ep, a.numel, s)
        res = []
        for rep in range(a.reps):
            tr.zero_()
            _lib.call("gp_comm_set_trace", ep._comm, tr.data_ptr())
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            allreduce_into(x, y, ep, codec, 0, s, **kw)
            e1.record(s)
            endpoint_wait(ep, a.numel, s)
            _lib.call("gp_comm_set_trace", ep._comm, None)
            t = tr.view(W, SLOTS).cpu().numpy().astype(np.int64)
            t0 = t[:, 0][t[:, 0] > 0].min()
            row = {"event_us": round(e0.elapsed_time(e1) * 1e3, 1),
                   "kernel_span_us": round((t[:, 36].max() - t0) / 1e3, 1),
                   "start_spread_us": round((t[:, 0][t[:, 0] > 0].max() - t0) / 1e3, 1)}
            for k, nm in sorted(names.items()):
                v = t[:, k]
                v = v[v > 0]
                if v.size and k:
                    q = np.percentile((v - t0) / 1e3, [0, 50, 90, 100])
                    row[nm] = [round(float(z), 1) for z in q]
            res.append(row)
        if rank == 0:
            print(json.dumps({"n": a.numel, "codec": cname, "p": p, "ctas": G, "fused": fused,
                              "stamps": "us from the first warp start: [min, p50, p90, max] over warps",
                              "reps": res[-2:]}), flush=True)
dist.barrier()
dist.destroy_process_group()
