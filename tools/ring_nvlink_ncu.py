"""The fused ring at p = 2 (or 4) in ONE process, for ncu's NVLink and DRAM
counters of the real P2P kernel on GPU 0.

Every call is enqueued on the other ranks' devices first and on GPU 0 last
(allreduce_into is asynchronous), so when ncu intercepts GPU 0's launch its
peers' kernels are already queued on their own GPUs and the ring completes
in a single pass. Run ncu with --devices 0, a single-pass metric list and
-k regex:ring_allreduce, e.g. (tools/ring_nvlink_ncu.sh):

  ncu --devices 0 -k regex:ring_allreduce --clock-control none --cache-control none \
      --metrics nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,gpu__time_duration.sum \
      --csv --log-file out.csv python tools/ring_nvlink_ncu.py 2

Sizes: the C1 / C2 / C4 / C3 gradients and a 256 MiB bucket, every codec;
each case runs twice (the second call is the one to read). Without ncu the
script prints the event-timed duration of GPU 0's call per case.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import GpuTransport  # noqa: E402
from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
SIZES = {"C1": 648_010, "C2": 4_710_538, "C4": 25_557_032, "C3": 61_100_840, "256MiB": 1 << 26}
if len(sys.argv) > 2:
    SIZES = {k: v for k, v in SIZES.items() if k in sys.argv[2].split(",")}
ctas = int(os.environ.get("RING_CTAS", "0"))
tr = GpuTransport(p, timeout_s=10.0, max_elems=max(SIZES.values()), ctas=ctas)
streams = [torch.cuda.Stream(device=r) for r in range(p)]
for name, n in SIZES.items():
    xs = [torch.randn(n, device=f"cuda:{r}") for r in range(p)]
    ys = [torch.empty_like(x) for x in xs]
    for codec in ("none", "trunc16", "quant8"):
        for rep in range(2):
            for r in range(p):
                torch.cuda.synchronize(r)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            for r in list(range(1, p)) + [0]:  # GPU 0 last
                with torch.cuda.device(r):
                    if r == 0:
                        e0.record(streams[0])
                    allreduce_into(xs[r], ys[r], tr.endpoint(r), codec, rep, streams[r])
                    if r == 0:
                        e1.record(streams[0])
            for r in range(p):
                endpoint_wait(tr.endpoint(r), n, streams[r])
            w = {"none": 4, "trunc16": 2, "quant8": 1}[codec]
            print(json.dumps({"case": name, "n": n, "p": p, "codec": codec, "rep": rep,
                              "us_gpu0": e0.elapsed_time(e1) * 1e3,
                              "wire_bytes_per_rank": 2 * (p - 1) * n * w // p}), flush=True)
    del xs, ys
tr.close()
