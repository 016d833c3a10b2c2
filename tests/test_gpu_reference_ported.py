"""The reference's own unit tests, ported to run against the B200 path.

Each test mirrors one in /root/reference/pkg/tests (file:line in its name or
docstring) with the same inputs and the same assertions; only the transport
changes (GPU ring — the emulated ring on one GPU when ranks outnumber GPUs)
and, where the reference compares against its own CPU functions, the CPU
oracle stands in for them.
"""

import struct

import numpy as np
import pytest
import torch

from helpers import run_ranks

pytestmark = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.fixture(scope="module")
def P():
    import paper_1811_03619_b200 as P
    return P


def transport(P, p, **kw):
    if 1 < p <= NGPU:
        return P.GpuTransport(p, max_elems=1 << 16, **kw)
    return P.EmulatedTransport(p, max_elems=1 << 16, **kw)


def random_inputs(p, n, seed):
    rng = np.random.default_rng(seed)
    return [rng.normal(0, 1, n).astype(np.float32) for _ in range(p)]


def assert_sum_close(out, want):
    atol = 1e-6 * max(1.0, float(np.abs(want).max()))
    np.testing.assert_allclose(out, want, rtol=1e-6, atol=atol)


def ring(P, p, ins, codec=0, fn="ring_allreduce", iteration=0):
    tr = transport(P, p)
    try:
        return run_ranks(tr, lambda r, ep: getattr(P, fn)(ins[r], r, p, ep, P.Codec(codec), iteration))
    finally:
        tr.close()


# ---------------------------------------------------- test_collective.py

def test_two_party_sum(P):  # test_collective.py:73-77
    ins = [np.array([1.0, 2.0], np.float32), np.array([3.0, 4.0], np.float32)]
    for out in ring(P, 2, ins):
        assert np.array_equal(out, np.array([4.0, 6.0], np.float32))


def test_matches_direct_sum(P):  # :79-84
    ins = random_inputs(4, 1024, 0)
    want = np.sum(np.stack(ins).astype(np.float64), axis=0)
    for out in ring(P, 4, ins):
        assert_sum_close(out, want)


def test_zeros_survive_quant8(P):  # :86-92
    zero = np.zeros(64, np.float32)
    for out in ring(P, 4, [zero] * 4, codec=2):
        assert np.array_equal(out, zero)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 7, 1024, 4099])
def test_sum_correctness_all_shapes(P, p, n):  # :94-101
    ins = random_inputs(p, n, p * 10_000 + n)
    want = np.sum(np.stack(ins).astype(np.float64), axis=0)
    for out in ring(P, p, ins):
        assert_sum_close(out, want)


def test_all_ranks_bit_identical_lossy(P):  # :103-110
    for codec in (1, 2):
        outs = ring(P, 4, random_inputs(4, 131, 7), codec=codec)
        for out in outs[1:]:
            assert np.array_equal(out, outs[0])


def test_quant8_error_envelope(P):  # :112-120
    p, n = 4, 512
    ins = random_inputs(p, n, 11)
    want = np.sum(np.stack(ins).astype(np.float64), axis=0)
    outs = ring(P, p, ins, codec=2)
    envelope = p * max(np.abs(v).max() for v in ins) / 64.0
    assert np.abs(outs[0].astype(np.float64) - want).max() <= envelope


def test_message_and_byte_accounting(P):  # :122-138
    for p in (2, 4, 8):
        for codec in P.Codec:
            n = 1024
            tr = transport(P, p)

            def op(rank, ep):
                ep.reset_stats()
                P.ring_allreduce(np.full(n, rank + 1.0, np.float32), rank, p, ep, codec)
                return ep.stats.snapshot()

            try:
                stats = run_ranks(tr, op)
            finally:
                tr.close()
            for s in stats:
                assert s.messages == 2 * (p - 1)
                assert s.payload_bytes == 2 * (p - 1) * P.payload_size(codec, n // p)
                assert s.payload_bytes == int(2 * ((p - 1) / p) * P.payload_size(codec, n))


def test_single_rank_is_identity(P):  # :147-151
    tr = P.EmulatedTransport(1, max_elems=16)
    vec = np.array([5.0, -1.0], np.float32)
    assert np.array_equal(P.ring_allreduce(vec, 0, 1, tr.endpoint(0), P.Codec.QUANT8), vec)
    tr.close()


@pytest.mark.parametrize("p", [2, 4, 8])
def test_pipelined_bit_exact_vs_sequential(P, p):  # :154-160
    ins = random_inputs(p, 1000, p)
    a = ring(P, p, ins)
    b = ring(P, p, ins, fn="pipelined_allreduce")
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_pipelined_bit_exact_trunc16_many_cases(P):  # :162-175
    p = 4
    tr = transport(P, p)
    try:
        for case in range(100):
            ins = random_inputs(p, 37, 1000 + case)
            a = run_ranks(tr, lambda r, ep: P.ring_allreduce(ins[r], r, p, ep, P.Codec.TRUNC16, case))
            b = run_ranks(tr, lambda r, ep: P.pipelined_allreduce(ins[r], r, p, ep, P.Codec.TRUNC16, case))
            for x, y in zip(a, b):
                assert np.array_equal(x, y)
    finally:
        tr.close()


def test_criterion_1_oracle_equivalence(P):  # test_acceptance.py:66-106 (cases trimmed 100 -> 20)
    for p in (1, 2, 3, 4, 8):
        tr = transport(P, p)
        try:
            for n in sorted({1, 7, p, 1024, 4099}):
                for case in range(20):
                    rng = np.random.default_rng((p, n, case))
                    vecs = [rng.normal(0, 1, n).astype(np.float32) for _ in range(p)]
                    want = np.sum(np.stack(vecs).astype(np.float64), axis=0)
                    res = run_ranks(tr, lambda r, ep: (P.ring_allreduce(vecs[r], r, p, ep, P.Codec.NONE, case),
                                                       P.pipelined_allreduce(vecs[r], r, p, ep, P.Codec.NONE,
                                                                             case)))
                    for a, b in res:
                        assert_sum_close(a, want)
                        assert np.array_equal(a, b)
        finally:
            tr.close()


# --------------------------------------------------- test_compression.py

def rt(P, vec, codec):
    return P.decompress(P.compress(np.asarray(vec, np.float32), codec)).cpu().numpy()


def test_trunc16_known_answers(P):  # test_compression.py:40-51
    b = P.compress(np.array([1.0], np.float32), P.Codec.TRUNC16)
    assert struct.unpack("<H", b.payload_bytes())[0] == 0x3F80
    b = P.compress(np.array([np.float32(np.pi)], np.float32), P.Codec.TRUNC16)
    assert struct.unpack("<H", b.payload_bytes())[0] == 0x4049
    assert P.decompress(b).cpu().numpy()[0] == np.float32(3.140625)


def test_trunc16_edges_and_error_bound(P):  # :66-88
    mn, mx = np.float32(2.0 ** -126), np.float32(np.finfo(np.float32).max)
    out = rt(P, [0.0, mn, -mn, mx, -mx], P.Codec.TRUNC16)
    assert np.isfinite(out).all() and out[0] == 0.0 and out[1] == mn and out[2] == -mn
    rng = np.random.default_rng(1)
    v = (rng.normal(0, 1, 20_000) * 10.0 ** rng.integers(-20, 20, 20_000)).astype(np.float32)
    v = v[np.abs(v) >= mn]
    o = rt(P, v, P.Codec.TRUNC16)
    rel = np.abs(o.astype(np.float64) - v.astype(np.float64)) / np.abs(v.astype(np.float64))
    assert rel.max() <= 2.0 ** -8


def test_quant8_known_answers(P):  # :92-124
    b = P.compress(np.array([0.0, 1.0, -1.0, 0.5], np.float32), P.Codec.QUANT8)
    assert list(np.frombuffer(b.payload_bytes(), np.int8)) == [0, 127, -127, 64]
    assert b.scale == pytest.approx(1 / 127, rel=1e-4)
    z = P.compress(np.zeros(33, np.float32), P.Codec.QUANT8)
    assert z.scale == 0.0
    assert P.compress(np.array([0.0, 1e-30], np.float32), P.Codec.QUANT8).scale > 0.0
    v = np.array([127.0, 2.5, -2.5, 0.5, -0.5], np.float32)
    assert list(np.frombuffer(P.compress(v, P.Codec.QUANT8).payload_bytes(), np.int8)) == [127, 3, -3, 1, -1]


def test_quant8_half_step_bound(P):  # :103-109
    rng = np.random.default_rng(2)
    for _ in range(20):
        v = (rng.normal(0, 1, 256) * 10.0 ** rng.integers(-3, 4)).astype(np.float32)
        o = rt(P, v, P.Codec.QUANT8)
        assert np.abs(o.astype(np.float64) - v.astype(np.float64)).max() <= np.abs(v).max() / 254.0


@pytest.mark.parametrize("codec", [1, 2])
def test_idempotent_reencoding(P, codec):  # :128-135
    rng = np.random.default_rng(3)
    for _ in range(25):
        v = (rng.normal(0, 1, 97) * 10.0 ** rng.integers(-6, 7)).astype(np.float32)
        once = rt(P, v, codec)
        assert np.array_equal(once, rt(P, once, codec))


@pytest.mark.parametrize("codec", [0, 1, 2])
def test_sign_and_zero_preservation(P, codec):  # :142-150
    v = np.random.default_rng(4).normal(0, 1, 1000).astype(np.float32)
    v[::10] = 0.0
    o = rt(P, v, codec)
    assert np.array_equal(o[::10], np.zeros(100, np.float32))
    nz = o != 0
    assert np.all(np.sign(o[nz]) == np.sign(v[nz]))


def test_empty_vector_and_wire(P):  # :162-217
    for codec in P.Codec:
        b = P.compress(np.zeros(0, np.float32), codec)
        assert b.n_elems == 0 and b.payload_bytes() == b""
        assert P.decompress(b).numel() == 0
        for n in (0, 1, 7, 1024):
            v = np.random.default_rng(n).normal(0, 1, n).astype(np.float32)
            wire = P.serialize_block(P.compress(v, codec))
            assert len(wire) == P.wire_size(codec, n)
        v = np.random.default_rng(8).normal(0, 1, 321).astype(np.float32)
        blk = P.compress(v, codec)
        back = P.deserialize_block(P.serialize_block(blk))
        assert back == blk
    wire = P.serialize_block(P.compress(np.array([2.0], np.float32), P.Codec.QUANT8))
    tag, n_elems, _ = struct.unpack("<BIf", wire[:9])
    assert tag == 2 and n_elems == 1
    with pytest.raises(P.CorruptBlockError):
        P.deserialize_block(P.serialize_block(P.compress(np.ones(4, np.float32), P.Codec.TRUNC16))[:-1])
    bad = bytearray(P.serialize_block(P.compress(np.ones(2, np.float32), P.Codec.NONE)))
    bad[0] = 77
    with pytest.raises(P.CorruptBlockError):
        P.deserialize_block(bytes(bad))


# ------------------------------------------------------- test_engine.py

def test_gradient_buffer_guards(P):  # test_engine.py:363-375
    from paper_1811_03619_b200.engine import GradientBuffer
    buf = GradientBuffer(2)
    buf.put(1, "block")
    with pytest.raises(P.EngineError, match="twice"):
        buf.put(3, "block")
    buf = GradientBuffer(2)
    buf.put(4, "b4")
    assert buf.take(4) == "b4"
    buf.put(6, "b6")


def test_config_validation(P):  # :377-385
    from paper_1811_03619_b200.engine import RunConfig
    with pytest.raises(P.ConfigError):
        RunConfig(mode="ring_async")
    with pytest.raises(P.ConfigError):
        RunConfig(mode="pipe_sgd", depth=1)
    with pytest.raises(P.ConfigError):
        RunConfig(iterations=0)
    with pytest.raises(P.ConfigError):
        RunConfig(learning_rate=0)


def test_batch_exceeding_shard_rejected_and_traffic_stats(P):  # :387-403
    from oracle import engine as OE
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import logistic_model
    data = OE.synthetic_blobs(dim=8, num_classes=2, num_samples=512, seed=1)
    with pytest.raises(P.ConfigError, match="shard"):
        run_inproc_cluster(2, RunConfig(mode="d_sync", iterations=2, batch_size=300), data, logistic_model(8, 2))
    res = run_inproc_cluster(4, RunConfig(mode="d_sync", iterations=4, batch_size=16), data, logistic_model(8, 2))
    for r in res:
        assert r.stats.messages == 4 * 2 * 3


@pytest.mark.parametrize("workers", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", ["d_sync", "pipe_sgd"])
def test_all_modes_complete(P, mode, workers):  # :258-265
    from oracle import engine as OE
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import logistic_model
    data = OE.synthetic_blobs(dim=8, num_classes=2, num_samples=512, seed=1)
    res = run_inproc_cluster(workers, RunConfig(mode=mode, iterations=6, batch_size=8, seed=1), data,
                             logistic_model(8, 2))
    assert len(res) == workers
    for r in res[1:]:
        assert np.array_equal(r.params, res[0].params)
