"""Bidirectional NVLink push at ring-phase sizes (1-38 MB): how long does one
kernel launch take to move S bytes each way between 2 GPUs? Series of R
back-to-back launches per device (both directions at once); per-launch time
= series / R. Modes: 0 interleaved grid-stride, 2 per-warp contiguous chunks
from a counter, 6 chunks + a system-scope release flag per chunk (the ring's
pattern). JSON lines."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import GpuTransport, _lib  # noqa: E402

tr = GpuTransport(2, max_elems=1024)
NB = 64 << 20
a = [torch.ones(NB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
b = [torch.empty(NB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
ctr = [torch.zeros(64, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)]
flags = [torch.zeros(1 << 20, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)]
st = [torch.cuda.Stream(device=d) for d in (0, 1)]
R = 40


def launch(d, size, ctas, mode, chunk, i):
    with torch.cuda.device(d):
        c = ctr[d][i % 64]
        _lib.call("gp_calib_p2p_copy_ex", b[1 - d].data_ptr(), a[d].data_ptr(), size, ctas, mode, chunk,
                  c.data_ptr(), flags[1 - d].data_ptr(), st[d].cuda_stream)


def run(size, ctas, mode, chunk):
    for d in (0, 1):
        ctr[d].zero_()
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    ev = []
    for d in (0, 1):
        with torch.cuda.device(d), torch.cuda.stream(st[d]):
            torch.cuda._sleep(2_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st[d])
            ev.append([e0, e1])
    for i in range(R):
        if i % 64 == 63:
            break
        for d in (0, 1):
            launch(d, size, ctas, mode, chunk, i)
    n = min(R, 63)
    for d in (0, 1):
        ev[d][1].record(st[d])
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    us = [e0.elapsed_time(e1) * 1e3 / n for e0, e1 in ev]
    return max(us)


for size in (1 << 20, 4710538, 9421076, 37684304):
    size = (size + 15) // 16 * 16
    for ctas in (16, 32, 64, 128, 148, 296, 592):
        row = {"bytes": size, "ctas": ctas}
        for mode, chunk, key in ((0, 0, "interleaved"), (2, 10240, "chunk10k"), (6, 10240, "chunk10k+rel"),
                                 (6, 65536, "chunk64k+rel")):
            us = run(size, ctas, mode, chunk)
            row[key] = {"us": round(us, 2), "gbs_each_way": round(size / us / 1e3, 1)}
        print(json.dumps(row), flush=True)
