"""Back-to-back asynchronous ring calls over real P2P (no host sync between
calls): each rank enqueues a long sequence of calls with mixed sizes (LL
and flag protocols), codecs and fused variants on its own stream, so ranks
drift up to a call apart on the device. Every output must be bit-identical
across ranks and, for a sample, equal the reference (oracle) result --
the cross-call safety argument of DESIGN.md section 3 under load."""

import numpy as np
import pytest
import torch

from helpers import assert_bits_equal, real_transport, run_ranks
from oracle import codec as OC
from oracle import ring as OR

pytestmark = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("seed", [2024, 7])
@pytest.mark.parametrize("p", [2, 4])
def test_async_call_storm_is_exact(P, p, seed):
    from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait
    g = np.random.default_rng(seed)
    calls = []
    for k in range(240):
        n = int(g.choice([1, 37, 4099, 70_001, 300_007, 1_000_003]))
        codec = int(g.integers(0, 3))
        fused = bool(g.integers(0, 4) == 0)
        calls.append((n, codec, fused))
    nmax = max(n for n, _, _ in calls)
    # blocks above 256 KiB take the flag protocol: both protocols interleave
    tr = real_transport(P, p, timeout_s=60.0, max_elems=nmax, ll_max_bytes=256 << 10)
    sample = set(range(0, len(calls), 17))
    base = [g.normal(0, 1, nmax).astype(np.float32) for _ in range(p)]

    def op(r, ep):
        dev = ep.device
        with torch.cuda.device(dev):
            x = torch.from_numpy(base[r]).to(dev)
            s = torch.cuda.Stream(dev)
            outs = []
            with torch.cuda.stream(s):
                for k, (n, codec, fused) in enumerate(calls):
                    xi = x[:n]
                    out = torch.empty(n, device=dev)
                    if fused:
                        w = (4, 2, 1)[codec]
                        slot = torch.empty(max(16, n * w), dtype=torch.uint8, device=dev)
                        sc = torch.empty(1, device=dev)
                        allreduce_into(xi, out, ep, P.Codec(codec), k, s, precompress=True, slot=slot, slot_scale=sc)
                        outs.append(("slot", slot[:n * w], sc))
                    else:
                        allreduce_into(xi, out, ep, P.Codec(codec), k, s)
                        outs.append(("out", out, None))
            endpoint_wait(ep, nmax, s)
            s.synchronize()
            return [(kind, a.cpu().numpy(), None if b is None else b.cpu().numpy()) for kind, a, b in outs]

    try:
        res = run_ranks(tr, op)
    finally:
        tr.close()
    for k, (n, codec, fused) in enumerate(calls):
        for r in range(1, p):
            assert res[r][k][1].tobytes() == res[0][k][1].tobytes(), f"call {k} rank {r} differs"
        if k in sample:
            ins = [b[:n] for b in base]
            if fused:
                summed = OR.ring_allreduce_all([OC.roundtrip(v, codec) for v in ins], codec).outputs[0]
                s_want, pl_want = OC.encode(summed, codec)
                assert res[0][k][1].tobytes() == np.asarray(pl_want).tobytes(), f"call {k} slot"
                if codec == OC.QUANT8:
                    assert np.float32(res[0][k][2][0]).view(np.uint32) == np.float32(s_want).view(np.uint32)
            else:
                want = OR.ring_allreduce_all(ins, codec).outputs[0]
                assert_bits_equal(res[0][k][1], want, f"call {k} n={n} codec={codec}")
