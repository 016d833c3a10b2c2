"""One process, two GPUs: the calibration push kernel (gp_calib_p2p_copy,
GPU 0 -> GPU 1, 256 MiB) a few times, for ncu's NVLink counters on GPU 0
(the kernel never waits on the peer, so ncu's kernel replay is safe)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import GpuTransport, _lib  # noqa: E402

tr = GpuTransport(2, max_elems=1024)  # peer access both ways
nb = 256 << 20
src = torch.ones(nb, dtype=torch.uint8, device="cuda:0")
dst = torch.empty(nb, dtype=torch.uint8, device="cuda:1")
s = torch.cuda.Stream(device=0)
with torch.cuda.device(0):
    for _ in range(3):
        _lib.call("gp_calib_p2p_copy", dst.data_ptr(), src.data_ptr(), nb, 148, 0, s.cuda_stream)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    _lib.call("gp_calib_p2p_copy", dst.data_ptr(), src.data_ptr(), nb, 148, 0, s.cuda_stream)
    e1.record(s)
    e1.synchronize()
print(f"push 256 MiB GPU0->GPU1: {e0.elapsed_time(e1) * 1e3:.1f} us, {nb / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
tr.close()
