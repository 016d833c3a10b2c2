"""GPU parity of the whole-vector codec kernels (gp_encode/gp_decode/
gp_roundtrip/gp_consume_update) against the reference golden vectors and
the CPU oracle. Bar: bit-exact."""

import os

import numpy as np
import pytest
import torch

from helpers import assert_bits_equal
from oracle import codec as OC
from oracle import engine as OE

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def P():
    import paper_1811_03619_b200 as P
    assert torch.cuda.is_available()
    return P


def test_golden_vectors(P):
    gold = np.load(os.path.join(GOLD, "codec_golden.npz"))
    for i in range(int(gold["count"][0])):
        x = gold[f"x{i}"]
        b = P.compress(torch.from_numpy(x).cuda(), P.Codec.TRUNC16)
        assert np.array_equal(b.payload.cpu().numpy().view("<u2"), gold[f"t16_{i}"]), i
        b = P.compress(torch.from_numpy(x).cuda(), P.Codec.QUANT8)
        assert np.array_equal(b.payload.cpu().numpy().view(np.int8), gold[f"q8_{i}"]), i
        assert np.float32(b.scale).view(np.uint32) == gold[f"q8s_{i}"].view(np.uint32)[0], i
        for codec in P.Codec:
            got = P.decompress(P.compress(torch.from_numpy(x).cuda(), codec)).cpu().numpy()
            assert_bits_equal(got, OC.roundtrip(x, int(codec)), f"case {i} {codec.name}")


def wide_values(n, seed):
    g = np.random.default_rng(seed)
    x = g.normal(0, 1, n) * 10.0 ** g.integers(-45, 38, n)
    x = x.astype(np.float32)
    u = g.integers(0, 2**32, n // 8, dtype=np.uint64).astype(np.uint32)
    u = u[(u & 0x7F800000) != 0x7F800000]  # random finite bit patterns incl. subnormals
    x[: u.size] = u.view(np.float32)
    return x


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 1000, 4099, (1 << 20) + 3])
def test_trunc16_and_none_random_bit_patterns(P, n):
    x = wide_values(n, n)
    for codec in (P.Codec.NONE, P.Codec.TRUNC16):
        b = P.compress(torch.from_numpy(x).cuda(), codec)
        _, want = OC.encode(x, int(codec))
        assert b.payload.cpu().numpy().tobytes() == want.tobytes()


def test_large_vector_all_codecs(P):
    n = 10_000_019
    g = np.random.default_rng(3)
    x = (g.normal(0, 1, n) * 10.0 ** g.integers(-6, 6, n)).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    for codec in P.Codec:
        b = P.compress(xt, codec)
        s, want = OC.encode(x, int(codec))
        assert b.payload.cpu().numpy().tobytes() == want.tobytes(), codec
        assert np.float32(b.scale) == s
        assert_bits_equal(P.decompress(b).cpu().numpy(), OC.decode(int(codec), s, want))


def test_quant8_blocks_at_many_scales(P):
    g = np.random.default_rng(4)
    for e in range(-45, 39, 3):
        for n in (1, 5, 64, 3001):
            x = (g.normal(0, 1, n) * 10.0 ** e).astype(np.float32)
            b = P.compress(torch.from_numpy(x).cuda(), P.Codec.QUANT8)
            s, want = OC.encode(x, OC.QUANT8)
            assert np.float32(b.scale).view(np.uint32) == np.float32(s).view(np.uint32), (e, n)
            assert np.array_equal(b.payload.cpu().numpy().view(np.int8), want), (e, n)


def test_quant8_exact_ties(P):
    # half-steps k+1/2 of a generic scale must round away from zero
    s = OC.quant_scale(3.3)
    ks = np.arange(-127, 128, dtype=np.float64)
    x = np.concatenate([[3.3], np.sign(ks) * (np.abs(ks) + 0.5) * float(s)]).astype(np.float32)
    x = x[np.abs(x) <= np.float32(3.3)]
    b = P.compress(torch.from_numpy(x).cuda(), P.Codec.QUANT8)
    _, want = OC.encode(x, OC.QUANT8)
    assert np.array_equal(b.payload.cpu().numpy().view(np.int8), want)


def test_nonfinite_rejected(P):
    for bad in (np.inf, -np.inf, np.nan):
        for codec in P.Codec:
            with pytest.raises(P.CodecError):
                P.compress(torch.tensor([1.0, bad], device="cuda"), codec)


def test_roundtrip_async_matches(P):
    from paper_1811_03619_b200.compression import CodecStatus, roundtrip_async
    x = wide_values(123_457, 9)
    x[np.abs(x) > 1e30] = 1.0
    xt = torch.from_numpy(x).cuda()
    for codec in P.Codec:
        out = torch.empty_like(xt)
        st = CodecStatus(xt.device)
        roundtrip_async(xt, codec, out, st)
        torch.cuda.synchronize()
        st.raise_if_nonfinite()
        assert_bits_equal(out.cpu().numpy(), OC.roundtrip(x, int(codec)), codec.name)


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_consume_update_matches_reference_sgd(P, p):
    from paper_1811_03619_b200 import _lib
    g = np.random.default_rng(p)
    n = 100_003
    w = g.normal(0, 0.1, n).astype(np.float32)
    total = (g.normal(0, 1, n) * p).astype(np.float32)
    for codec in P.Codec:
        for lr in (0.05, 0.1, 1e-3):
            blk = P.compress(torch.from_numpy(total).cuda(), codec)
            wt = torch.from_numpy(w).cuda()
            _lib.call("gp_consume_update", wt.data_ptr(), int(codec), blk.payload.data_ptr(),
                      blk.scale_t.data_ptr(), n, float(np.float32(lr)), p,
                      torch.cuda.current_stream().cuda_stream)
            s, pl = OC.encode(total, int(codec))
            want = OE.sgd_update(w, OE.aggregate_mean(OC.decode(int(codec), s, pl), p), lr)
            assert_bits_equal(wt.cpu().numpy(), want, f"{codec.name} lr={lr}")
