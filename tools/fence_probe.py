"""What a system-scope release per chunk costs at mid sizes, and whether one
fence per CTA (all its warps' chunks) instead of one per warp recovers it.
Two GPUs push to each other at once (calib p2p_copy_kernel, 512-thread CTAs):
contiguous per-warp chunks with no publish / a st.release.sys per chunk /
a CTA barrier + one fence + relaxed flag stores per CTA round."""
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


def run(nb, mode, chunk, ctas):
    us = []
    for rep in range(2):
        evs = []
        for d in (0, 1):
            ctr[d].zero_()
        for d in (0, 1):
            torch.cuda.synchronize(d)
        for d in (0, 1):
            with torch.cuda.device(d), torch.cuda.stream(st[d]):
                torch.cuda._sleep(1_000_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st[d])
                for k in range(REPS):
                    _lib.call("gp_calib_p2p_copy_ex", b[1 - d].data_ptr(), a[d].data_ptr(), nb, ctas, mode, chunk,
                              ctr[d][k:k + 1].data_ptr(), flags[1 - d].data_ptr(), st[d].cuda_stream)
                e1.record(st[d])
                evs.append((e0, e1))
        for s in st:
            s.synchronize()
        us = [round(e0.elapsed_time(e1) * 1e3 / REPS, 1) for e0, e1 in evs]
    return max(us)


for nb in (2 << 20, 8 << 20, 64 << 20):
    for ctas in (37, 148):
        for chunk in (4096, 16384):
            row = {"bytes": nb, "ctas_512thr": ctas, "chunk": chunk}
            for name, mode in (("contig", 2), ("release_per_warp", 6), ("fence_per_cta", 8)):
                t = run(nb, mode, chunk, ctas)
                row[name + "_us"] = t
                row[name + "_gbs"] = round(nb / t / 1e3, 1)
            print(json.dumps(row), flush=True)
