"""Calibrate small-kernel timing: our HBM kernels vs torch's copy of the same
bytes, warm (L2-resident, back-to-back) and cold (read-flush subtraction)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import _lib  # noqa: E402
from paper_1811_03619_b200.compression import CodecStatus, encode_async, roundtrip_async  # noqa: E402

n = int(os.environ.get("N", 4710538))
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(dev)
flush = torch.ones(64 << 20, device=dev)
g = torch.randn(n, device=dev)
w = torch.randn(n, device=dev)
loc = torch.empty_like(g)
payload = torch.zeros(n * 2, dtype=torch.uint8, device=dev)
st = CodecStatus(dev)
R = 50


def series(fn, with_flush):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        if with_flush:
            flush.sum()
        e0.record(s)
        for _ in range(R):
            if with_flush:
                flush.sum()
            if fn:
                fn()
        e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / R * 1e3


payload4 = torch.zeros(n * 4, dtype=torch.uint8, device=dev)
sts = [CodecStatus(dev) for _ in range(3)]
for c in range(3):
    encode_async(g, c, payload4, sts[c], s.cuda_stream)
W = {0: 4, 1: 2, 2: 1}
kern = {"torch_copy_37.7MB": lambda: loc.copy_(g)}
for c, nm in ((0, "none"), (1, "trunc16"), (2, "quant8")):
    kern[f"encode_{nm}_{(4 + W[c]) * n / 1e6:.1f}MB"] = (
        lambda c=c: encode_async(g, c, payload4, sts[c], s.cuda_stream))
    kern[f"consume_update_{nm}_{(8 + W[c]) * n / 1e6:.1f}MB"] = (
        lambda c=c: _lib.call("gp_consume_update", w.data_ptr(), c, payload4.data_ptr(),
                              sts[c].scale_view.data_ptr(), n, 1e-3, 2, s.cuda_stream))
kern["roundtrip_trunc16_37.7MB"] = lambda: roundtrip_async(g, 1, loc, st, s.cuda_stream)
base = series(None, True)
series(None, True)
for k, fn in kern.items():
    fn()
    warm = series(fn, False)
    cold = series(fn, True) - series(None, True)
    print(json.dumps({"lib": os.path.basename(os.environ.get("PIPESGD_LIB", "default")), "kernel": k, "n": n, "warm_us": round(warm, 2), "cold_us": round(cold, 2)}), flush=True)
