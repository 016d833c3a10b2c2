"""Mid-size pushes among 4 GPUs (one process, peer access): every GPU sends
`total` bytes (a) all to its ring successor, (b) split evenly over its 3
peers (the direct reduce-scatter's pattern), with and without a
system-scope release per 4 KiB chunk. Calibration copy kernel (512-thread
CTAs), all sends of all GPUs launched at once; time = max over GPUs of the
span from the first launch to the last kernel's end."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import GpuTransport, _lib  # noqa: E402

P = 4
tr = GpuTransport(P, max_elems=1024)
MAX = 32 << 20
src = [torch.empty(MAX, dtype=torch.uint8, device=f"cuda:{d}") for d in range(P)]
dst = [torch.empty(MAX, dtype=torch.uint8, device=f"cuda:{d}") for d in range(P)]
flags = [torch.zeros(1 << 16, dtype=torch.int64, device=f"cuda:{d}") for d in range(P)]
streams = [[torch.cuda.Stream(device=d) for _ in range(3)] for d in range(P)]
REPS = 20
ctr = [torch.zeros(3 * REPS, dtype=torch.int64, device=f"cuda:{d}") for d in range(P)]


def run(total, spread, mode, ctas_total=148):
    for d in range(P):
        ctr[d].zero_()
        torch.cuda.synchronize(d)
    spans = []
    ev = []
    for d in range(P):
        peers = [(d + k) % P for k in (1, 2, 3)] if spread else [(d + 1) % P]
        per = total // len(peers)
        ctas = max(1, ctas_total // len(peers))
        evs = []
        for j, q in enumerate(peers):
            s = streams[d][j]
            with torch.cuda.device(d):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for k in range(REPS):
                    _lib.call("gp_calib_p2p_copy_ex", dst[q].data_ptr() + d * per, src[d].data_ptr() + j * per, per,
                              ctas, mode, 4096, ctr[d][3 * k + j:3 * k + j + 1].data_ptr(), flags[q].data_ptr(),
                              s.cuda_stream)
                e1.record(s)
                evs.append((e0, e1))
        ev.append(evs)
    for d in range(P):
        torch.cuda.synchronize(d)
    for evs in ev:
        spans.append(max(e0.elapsed_time(e1) for e0, e1 in evs) * 1e3 / REPS)
    return max(spans)


for total in (3 << 20, 9 << 20, 24 << 20):
    row = {"bytes_per_gpu": total}
    for spread in (False, True):
        for name, mode in (("plain", 2), ("release", 6)):
            run(total, spread, mode)
            row[f"{'a2a' if spread else 'ring'}_{name}_us"] = round(run(total, spread, mode), 1)
    print(json.dumps(row), flush=True)
