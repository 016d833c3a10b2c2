"""Do `nvidia-smi nvlink -gt d` data counters move with known NVLink traffic?
K pushes of 256 MiB GPU0 -> GPU1 (gp_calib_p2p_copy); prints the per-link
counter deltas of both GPUs (KiB) next to the bytes pushed."""
import json
import os
import re
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import GpuTransport, _lib  # noqa: E402


def counters(gpu):
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(gpu)], capture_output=True, text=True).stdout
    tx = sum(int(v) for v in re.findall(r"Tx:\s*(\d+)", out))
    rx = sum(int(v) for v in re.findall(r"Rx:\s*(\d+)", out))
    return tx, rx, out


before = [counters(g) for g in (0, 1)]
print(json.dumps({"raw_sample": before[0][2][:600]}))
tr = GpuTransport(2, max_elems=1024)
nb, K = 256 << 20, 8
src = torch.ones(nb, dtype=torch.uint8, device="cuda:0")
dst = torch.empty(nb, dtype=torch.uint8, device="cuda:1")
s = torch.cuda.Stream(device=0)
with torch.cuda.device(0):
    for _ in range(K):
        _lib.call("gp_calib_p2p_copy", dst.data_ptr(), src.data_ptr(), nb, 148, 0, s.cuda_stream)
    s.synchronize()
after = [counters(g) for g in (0, 1)]
print(json.dumps({"pushed_bytes": K * nb, "gpu0_tx_delta": after[0][0] - before[0][0],
                  "gpu0_rx_delta": after[0][1] - before[0][1], "gpu1_tx_delta": after[1][0] - before[1][0],
                  "gpu1_rx_delta": after[1][1] - before[1][1], "unit": "as printed by nvidia-smi (KiB)"}))
tr.close()
