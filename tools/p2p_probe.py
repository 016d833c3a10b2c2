"""NVLink ceilings on this box (2 GPUs, one process): kernel push/pull copy
rates vs CTA count, uni- and bidirectional, copy-engine memcpy, flag
ping-pong latency. Output: JSON lines."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import GpuTransport, _lib  # noqa: E402

tr = GpuTransport(2, max_elems=1024)  # enables peer access both ways
NB = 1 << 30
a = [torch.empty(NB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
b = [torch.empty(NB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
st = [torch.cuda.Stream(device=d) for d in (0, 1)]


def run(dirs, ctas, pull, reps=5):
    # dirs: list of (src_dev, dst_dev); kernel runs on the src device for push,
    # on the dst device for pull.
    ev = []
    for _ in range(2):  # warm-up
        for s, d in dirs:
            dev = d if pull else s
            with torch.cuda.device(dev):
                _lib.call("gp_calib_p2p_copy", b[d].data_ptr(), a[s].data_ptr(), NB, ctas, pull, st[dev].cuda_stream)
    for x in st:
        x.synchronize()
    res = []
    for s, d in dirs:
        dev = d if pull else s
        with torch.cuda.device(dev):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st[dev])
            for _ in range(reps):
                _lib.call("gp_calib_p2p_copy", b[d].data_ptr(), a[s].data_ptr(), NB, ctas, pull, st[dev].cuda_stream)
            e1.record(st[dev])
            ev.append((e0, e1))
    for x in st:
        x.synchronize()
    return [NB * reps / (e0.elapsed_time(e1) / 1e3) / 1e9 for e0, e1 in ev]


for pull in (0, 1):
    for ctas in (8, 16, 32, 64, 96, 148, 296):
        uni = run([(0, 1)], ctas, pull)
        bi = run([(0, 1), (1, 0)], ctas, pull)
        print(json.dumps({"mode": "pull" if pull else "push", "ctas": ctas, "uni_gbs": round(uni[0], 1),
                          "bidir_gbs_each": [round(v, 1) for v in bi]}), flush=True)

# copy engine
for _ in range(2):
    b[1].copy_(a[0])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.device(0):
    e0.record()
    for _ in range(5):
        b[1].copy_(a[0])
    e1.record()
torch.cuda.synchronize()
print(json.dumps({"mode": "memcpy_peer", "gbs": round(NB * 5 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)}))

# ping-pong latency
flags = [torch.zeros(4, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)]
ns = [torch.zeros(1, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)]
iters = 20000
for d in (0, 1):
    with torch.cuda.device(d):
        _lib.call("gp_calib_pingpong", flags[d].data_ptr(), flags[1 - d].data_ptr(), iters, int(d == 0), 0,
                  ns[d].data_ptr(), st[d].cuda_stream)
for x in st:
    x.synchronize()
print(json.dumps({"mode": "pingpong", "round_trip_us": ns[0].item() / iters / 1e3,
                  "one_way_us": ns[0].item() / iters / 2e3}))
