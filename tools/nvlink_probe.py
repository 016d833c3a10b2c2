"""Which NVML NVLink byte counters move, and by how much, around known
traffic: K pushes of a buffer GPU0 -> GPU1 (gp_calib_p2p_copy, one process,
peer access), then K fused ring calls at p = 2 per codec. Prints one JSON
line per probe with the counter deltas of both GPUs next to the algorithmic
bytes. Run: python tools/nvlink_probe.py (2 GPUs)."""
import json
import os
import sys
import threading

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402

from paper_1811_03619_b200 import GpuTransport, _lib  # noqa: E402
from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait  # noqa: E402

pynvml.nvmlInit()
H = [pynvml.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
FIELDS = [138, 139, 140, 141, 202, 204]


def snap():
    out = []
    for h in H:
        d = {}
        for f in FIELDS:
            for scope in [0xFFFFFFFF] + list(range(18)):
                try:
                    v = pynvml.nvmlDeviceGetFieldValues(h, [(f, scope)])[0]
                except pynvml.NVMLError as e:  # noqa: PERF203
                    d[f"{f}@{scope}"] = f"err {e}"
                    continue
                if v.nvmlReturn == 0:
                    d[f"{f}@{scope}"] = int(v.value.ullVal)
                else:
                    d[f"{f}@{scope}"] = f"ret {v.nvmlReturn}"
        out.append(d)
    return out


def diff(a, b):
    res = []
    for x, y in zip(a, b):
        dd = {}
        for k in y:
            if isinstance(y[k], int) and isinstance(x.get(k), int) and y[k] != x[k]:
                dd[k] = y[k] - x[k]
        res.append(dd)
    return res


base = snap()
print(json.dumps({"probe": "fields", "gpu0": {k: v for k, v in base[0].items() if not isinstance(v, int)}}))
tr = GpuTransport(2, max_elems=1 << 26, ctas=592)
nb = 256 << 20
K = 8
src = torch.ones(nb, dtype=torch.uint8, device="cuda:0")
dst = torch.empty(nb, dtype=torch.uint8, device="cuda:1")
s = torch.cuda.Stream(device=0)
torch.cuda.synchronize(0)
a = snap()
with torch.cuda.device(0):
    for _ in range(K):
        _lib.call("gp_calib_p2p_copy", dst.data_ptr(), src.data_ptr(), nb, 148, 0, s.cuda_stream)
    s.synchronize()
b = snap()
print(json.dumps({"probe": "push", "bytes_gpu0_to_gpu1": K * nb, "delta": diff(a, b)}))

n = 1 << 26
for codec, w in (("none", 4), ("trunc16", 2), ("quant8", 1)):
    xs = [torch.randn(n, device=f"cuda:{r}") for r in range(2)]
    ys = [torch.empty_like(x) for x in xs]
    ss = [torch.cuda.Stream(device=r) for r in range(2)]
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    a = snap()

    def run(r):
        with torch.cuda.device(r):
            for _ in range(K):
                allreduce_into(xs[r], ys[r], tr.endpoint(r), codec, 0, ss[r])
            endpoint_wait(tr.endpoint(r), n, ss[r])

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    b = snap()
    print(json.dumps({"probe": f"ring_{codec}", "wire_bytes_per_rank": K * 2 * (2 - 1) // 2 * n * w,
                      "delta": diff(a, b)}))
tr.close()
