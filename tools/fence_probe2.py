"""Pull-model ingredients at mid sizes: (a) a local copy with a release per
chunk (does a system-scope fence on LOCAL stores cost what it costs on NVLink
stores?), (b) two GPUs pulling from each other at once (remote loads, local
stores), contiguous per-warp chunks, 512-thread CTAs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import GpuTransport, _lib  # noqa: E402

tr = GpuTransport(2, max_elems=1024)
NBMAX = 64 << 20
REPS = 20
a = [torch.empty(NBMAX, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
b = [torch.empty(NBMAX, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
ctr = [torch.zeros(REPS, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)]
flags = [torch.zeros(1 << 20, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)]
st = [torch.cuda.Stream(device=d) for d in (0, 1)]


def run(nb, mode, chunk, ctas, where):
    us = []
    for rep in range(2):
        evs = []
        for d in (0, 1):
            ctr[d].zero_()
        for d in (0, 1):
            torch.cuda.synchronize(d)
        for d in (0, 1):
            if where == "local":
                dst, src, fl = b[d], a[d], flags[d]
            elif where == "push":
                dst, src, fl = b[1 - d], a[d], flags[1 - d]
            else:  # pull: remote src, local dst
                dst, src, fl = b[d], a[1 - d], flags[d]
            with torch.cuda.device(d), torch.cuda.stream(st[d]):
                torch.cuda._sleep(1_000_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st[d])
                for k in range(REPS):
                    _lib.call("gp_calib_p2p_copy_ex", dst.data_ptr(), src.data_ptr(), nb, ctas, mode, chunk,
                              ctr[d][k:k + 1].data_ptr(), fl.data_ptr(), st[d].cuda_stream)
                e1.record(st[d])
                evs.append((e0, e1))
        for s in st:
            s.synchronize()
        us = [round(e0.elapsed_time(e1) * 1e3 / REPS, 1) for e0, e1 in evs]
    return max(us)


for nb in (2 << 20, 8 << 20, 64 << 20):
    for chunk in (4096, 16384):
        row = {"bytes": nb, "ctas_512thr": 148, "chunk": chunk}
        for where in ("local", "push", "pull"):
            pull = 1 if where == "pull" else 0
            for name, mode in (("plain", 2), ("release", 6)):
                t = run(nb, mode | pull, chunk, 148, where)
                row[f"{where}_{name}_us"] = t
        print(json.dumps(row), flush=True)
