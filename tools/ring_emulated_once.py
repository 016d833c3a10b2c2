"""Run the fused ring once per codec with p ranks emulated on cuda:0 (for ncu:
`-k regex:ring_allreduce`). Checks that every rank's output is bit-identical
(parity against the oracle lives in tests/test_gpu_ring.py)."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import Codec, EmulatedTransport  # noqa: E402
from paper_1811_03619_b200.collective import ring_allreduce  # noqa: E402

p = int(os.environ.get("P", 4))
n = int(os.environ.get("N", 1 << 24))
codecs = [Codec.parse(c) for c in os.environ.get("CODECS", "none,trunc16,quant8").split(",")]
g = np.random.default_rng(0)
ins = [torch.from_numpy(g.normal(0, 1, n).astype(np.float32)).cuda() for _ in range(p)]
tr = EmulatedTransport(p, max_elems=n, timeout_s=60)
for codec in codecs:
    outs = [None] * p
    th = [threading.Thread(target=lambda r=r: outs.__setitem__(r, ring_allreduce(ins[r], r, p, tr.endpoint(r), codec)))
          for r in range(p)]
    [t.start() for t in th]
    [t.join() for t in th]
    for r in range(1, p):
        assert torch.equal(outs[r].view(torch.int32), outs[0].view(torch.int32)), f"rank {r} differs"
    print(codec.name, "ok", flush=True)
tr.close()
