"""One fused ring call per codec (precompress + slot output, the engine's comm
kernel) with p ranks emulated on cuda:0, for ncu. Checks that every rank's
slot and scale are bit-identical (oracle parity: tests/test_gpu_fused.py)."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import Codec, EmulatedTransport  # noqa: E402
from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait  # noqa: E402

p = int(os.environ.get("P", 4))
n = int(os.environ.get("N", 1 << 22))
codecs = [Codec.parse(c) for c in os.environ.get("CODECS", "none,trunc16,quant8").split(",")]
g = np.random.default_rng(0)
ins_np = [(g.normal(0, 1e-2, n)).astype(np.float32) for _ in range(p)]
ins = [torch.from_numpy(x).cuda() for x in ins_np]
tr = EmulatedTransport(p, max_elems=n, timeout_s=60)
for codec in codecs:
    w = codec.bytes_per_elem
    res = [None] * p

    def run(r):
        out = torch.empty(n, device="cuda")
        slot = torch.empty(n * w, dtype=torch.uint8, device="cuda")
        sc = torch.empty(1, device="cuda")
        s = torch.cuda.current_stream()
        allreduce_into(ins[r], out, tr.endpoint(r), codec, 1, s, precompress=True, slot=slot, slot_scale=sc)
        endpoint_wait(tr.endpoint(r), n, s)
        res[r] = (slot.cpu().numpy(), sc.cpu().numpy())

    th = [threading.Thread(target=run, args=(r,)) for r in range(p)]
    [t.start() for t in th]
    [t.join() for t in th]
    for r in range(1, p):
        assert res[r][0].tobytes() == res[0][0].tobytes() and res[r][1].tobytes() == res[0][1].tobytes()
    print(codec.name, "ok", flush=True)
tr.close()
