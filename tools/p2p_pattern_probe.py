"""Does the ring's access pattern (contiguous per-warp chunks, a release per
chunk) cost NVLink bandwidth? Bidirectional push between 2 GPUs, 1 GiB."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import GpuTransport, _lib  # noqa: E402

tr = GpuTransport(2, max_elems=1024)
NB = 1 << 28
a = [torch.empty(NB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
b = [torch.empty(NB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
ctr = [torch.zeros(1, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)]
flags = [torch.zeros(1 << 20, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)]
st = [torch.cuda.Stream(device=d) for d in (0, 1)]


def run(mode, chunk, ctas, reps=5):
    ev = []
    for rep in range(2):
        evs = []
        for d in (0, 1):
            with torch.cuda.device(d), torch.cuda.stream(st[d]):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st[d])
                for _ in range(reps):
                    ctr[d].zero_()
                    _lib.call("gp_calib_p2p_copy_ex", b[1 - d].data_ptr(), a[d].data_ptr(), NB, ctas, mode, chunk,
                              ctr[d].data_ptr(), flags[1 - d].data_ptr(), st[d].cuda_stream)
                e1.record(st[d])
                evs.append((e0, e1))
        for s in st:
            s.synchronize()
        ev = evs
    return [round(NB * reps / (e0.elapsed_time(e1) / 1e3) / 1e9, 1) for e0, e1 in ev]


for ctas in (32, 148):
    print(json.dumps({"ctas": ctas, "interleaved": run(0, 0, ctas)}), flush=True)
    for chunk in (4096, 16384, 65536, 262144):
        print(json.dumps({"ctas": ctas, "chunk": chunk, "contig": run(2, chunk, ctas),
                          "contig+release": run(6, chunk, ctas)}), flush=True)
