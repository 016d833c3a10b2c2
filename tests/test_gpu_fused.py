"""GPU parity of the fused ring variants:

  precompress : ring(D(C(g_r))) computed from the raw gradients g_r, the
                engine's whole-vector local pre-compress (engine.py:333,
                :355/:400) applied inside the ring's loads;
  slot output : C(ring sum) written as the compressed aggregated slot
                (engine.py:407) by the allgather, its quant8 scale derived
                from the block scales (127 * max_b s_b) with no extra pass.

Bar: bit-exact against the oracle composition of the reference functions
(payload bytes and scale bits), on every rank, for every codec.
"""

import numpy as np
import pytest
import torch

from helpers import assert_bits_equal, real_transport, run_ranks
from oracle import codec as OC
from oracle import ring as OR

pytestmark = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.fixture(scope="module")
def P():
    import paper_1811_03619_b200 as P
    return P


def expected(ins, codec, pre, slot):
    xs = [OC.roundtrip(x, codec) for x in ins] if pre else ins
    summed = OR.ring_allreduce_all(xs, codec).outputs[0]
    if slot:
        return OC.encode(summed, codec)
    return summed


def run_fused(P, tr, ins, codec, pre, slot, devices):
    from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait
    p, n = len(ins), ins[0].size
    w = P.Codec(codec).bytes_per_elem

    def op(r, ep):
        dev = devices[r]
        with torch.cuda.device(dev):
            x = torch.from_numpy(ins[r]).to(dev)
            out = torch.empty_like(x)
            sl = torch.full((n * w,), 0xAB, dtype=torch.uint8, device=dev) if slot else None
            sc = torch.full((1,), -1.0, device=dev) if slot else None
            s = ep.stream  # the rank's own stream (ranks may share a GPU)
            s.wait_stream(torch.cuda.current_stream(dev))
            allreduce_into(x, out, ep, codec, 4, s, precompress=pre, slot=sl, slot_scale=sc)
            endpoint_wait(ep, n, s)
            if slot:
                return sl.cpu().numpy(), sc.cpu().numpy()
            return out.cpu().numpy()

    return run_ranks(tr, op)


def check(res, want, codec, slot, msg):
    for r, got in enumerate(res):
        if slot:
            pl, sc = got
            w_sc, w_pl = want
            assert pl.tobytes() == np.asarray(w_pl).tobytes(), f"{msg} rank {r} payload"
            assert np.float32(sc[0]).view(np.uint32) == np.float32(w_sc).view(np.uint32), f"{msg} rank {r} scale"
        else:
            assert_bits_equal(got, want, f"{msg} rank {r}")


def inputs(p, n, seed, scale_exp=0):
    g = np.random.default_rng(seed)
    return [(g.normal(0, 1, n) * 10.0 ** (scale_exp + g.integers(-2, 3))).astype(np.float32) for _ in range(p)]


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_fused_variants_emulated(P, p):
    n_list = [1, 7, 4099, 1_000_003]
    tr = P.EmulatedTransport(p, timeout_s=60.0, max_elems=max(n_list))
    devs = [torch.device("cuda", 0)] * p
    try:
        for n in n_list:
            for codec in (0, 1, 2):
                ins = inputs(p, n, n * 10 + codec + p, scale_exp=-30 if n == 7 else 0)
                for pre, slot in ((True, False), (False, True), (True, True)):
                    want = expected(ins, codec, pre, slot)
                    res = run_fused(P, tr, ins, codec, pre, slot, devs)
                    check(res, want, codec, slot, f"p={p} n={n} codec={codec} pre={pre} slot={slot}")
    finally:
        tr.close()


@pytest.mark.parametrize("n,ll", [(4_710_538, 0), (150_001, None)])  # flag protocol / LL protocol
@pytest.mark.parametrize("codec", [0, 1, 2])
def test_fused_variants_p2p(P, codec, n, ll):
    p = 4  # per-rank launches: one GPU per rank, or ranks sharing GPUs
    tr = real_transport(P, p, timeout_s=60.0, max_elems=n, ll_max_bytes=ll)
    devs = [tr.endpoint(r).device for r in range(p)]
    try:
        ins = inputs(p, n, 77 + codec, scale_exp=-3)
        for pre, slot in ((True, False), (True, True)):
            want = expected(ins, codec, pre, slot)
            res = run_fused(P, tr, ins, codec, pre, slot, devs)
            check(res, want, codec, slot, f"p2p codec={codec} pre={pre} slot={slot}")
    finally:
        tr.close()


def test_fused_precompress_rejects_nonfinite(P):
    p = 4
    tr = P.EmulatedTransport(p, timeout_s=20.0, max_elems=4096)
    ins = inputs(p, 3000, 5)
    ins[1][2999] = np.inf
    try:
        for codec in (0, 1, 2):
            with pytest.raises(P.CodecError):
                run_fused(P, tr, ins, codec, True, True, [torch.device("cuda", 0)] * p)
    finally:
        tr.close()
