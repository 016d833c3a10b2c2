"""Small workloads for compute-sanitizer (memcheck / synccheck / racecheck /
initcheck): every codec kernel, the emulated ring (all p ranks in one
cooperative launch on cuda:0) on both wire protocols, the direct
reduce-scatter, the fused variants, and the star collectives. Each output is
checked for replica identity; exits non-zero on any mismatch. Kept small:
the sanitizer slows kernels 10-100x."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_03619_b200 import Codec, EmulatedTransport, compress, decompress  # noqa: E402
from paper_1811_03619_b200 import _lib  # noqa: E402
from paper_1811_03619_b200.collective import (allreduce_into, broadcast_from_root, endpoint_wait,  # noqa: E402
                                              gather_to_root)


def ranks(p, fn):
    out = [None] * p
    th = [threading.Thread(target=lambda r=r: out.__setitem__(r, fn(r))) for r in range(p)]
    [t.start() for t in th]
    [t.join() for t in th]
    return out


g = np.random.default_rng(0)
# codec kernels (encode with absmax, decode, roundtrip, consume_update)
from paper_1811_03619_b200.compression import CodecStatus, roundtrip_async  # noqa: E402
x = torch.from_numpy(g.normal(0, 1, 100_003).astype(np.float32)).cuda()
for c in Codec:
    blk = compress(x, c)
    y = decompress(blk)
    assert y.shape == x.shape
    rt = torch.empty_like(x)
    roundtrip_async(x, c, rt, CodecStatus(x.device))
    assert torch.equal(rt.view(torch.int32), y.view(torch.int32))
    w = x.clone()
    _lib.call("gp_consume_update", w.data_ptr(), int(c), blk.payload.data_ptr(), blk.scale_t.data_ptr(),
              x.numel(), 0.01, 2, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("codec kernels ok", flush=True)

cases = [(2, 1_200_000), (4, 4099), (3, 2_000_001), (8, 777)]  # flag protocol / LL / direct RS (none) / p = 8
for p, n in cases:
    ins = [torch.from_numpy(g.normal(0, 1, n).astype(np.float32)).cuda() for _ in range(p)]
    tr = EmulatedTransport(p, max_elems=n, timeout_s=600)
    for codec in Codec:
        for fused in (False, True):
            def run(r):
                ep = tr.endpoint(r)
                s = ep.stream
                out = torch.empty(n, device="cuda")
                if fused:
                    slot = torch.empty(n * codec.bytes_per_elem, dtype=torch.uint8, device="cuda")
                    sc = torch.empty(1, device="cuda")
                    allreduce_into(ins[r], out, ep, codec, 1, s, precompress=True, slot=slot, slot_scale=sc)
                    endpoint_wait(ep, n, s)
                    return slot.cpu().numpy().tobytes() + sc.cpu().numpy().tobytes()
                allreduce_into(ins[r], out, ep, codec, 1, s)
                endpoint_wait(ep, n, s)
                return out.cpu().numpy().tobytes()
            res = ranks(p, run)
            assert all(r == res[0] for r in res), (p, n, codec, fused)
            print(f"ring p={p} n={n} {codec.name} fused={fused} ok", flush=True)
    v = [ins[r].cpu().numpy() for r in range(p)]
    got = ranks(p, lambda r: gather_to_root(v[r], 0, r, p, tr.endpoint(r)))
    assert got[0] is not None
    got = ranks(p, lambda r: broadcast_from_root(v[0] if r == 0 else None, 0, r, p, tr.endpoint(r)))
    assert all(o.tobytes() == v[0].tobytes() for o in got)
    print(f"star p={p} ok", flush=True)
    tr.close()
print("all sanitizer cases ok")
