"""Parity at the BASELINE.json configurations' real sizes.

C1  MNIST MLP 784-500-500-10 (648,010 params), p=4, codec none, Pipe-SGD
    width 2: engine weights bit-exact with the oracle trajectory when the
    oracle supplies the gradients.
C3  AlexNet-sized gradient (61,100,840 fp32), quant8 ring at p=8 (emulated
    on one GPU) and on the real GPUs: every rank bit-identical, and sampled
    every ring block bit-exact with the oracle's fold (block b folds from rank b;
    the block-wide quant8 scale makes each block self-contained, so checking
    whole blocks is exact at full size).
C4  ResNet-50-sized gradient (25,557,032), codec none, p=4 and 8: ranks
    identical, every block bit-exact, and the sum within the reference's
    own tolerance of the float64 direct sum (test_collective.py:50-54).
C2  the bench's CIFAR CNN through the width-2 engine on real GPUs: replicas
    stay bit-identical over steps.
"""

import numpy as np
import pytest
import torch

from helpers import assert_bits_equal, real_transport, run_ranks
from oracle import codec as OC
from oracle import engine as OE
from oracle import ring as OR

pytestmark = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
ALEXNET, RESNET50 = 61_100_840, 25_557_032


@pytest.fixture(scope="module")
def P():
    import paper_1811_03619_b200 as P
    return P


def make_inputs(p, n, scale, seed, device="cuda:0"):
    g = torch.Generator(device=device).manual_seed(seed)
    return [torch.randn(n, device=device, generator=g) * scale for _ in range(p)]


def oracle_block(ins_cpu_block, b, codec):
    """Reference fold of block b (collective.py:96-139): s0 = x_b,
    s_k = fl(x_{b+k} + D(C(s_{k-1}))), out = D(C(s_{p-1}))."""
    p = len(ins_cpu_block)
    s = ins_cpu_block[b].copy()
    for k in range(1, p):
        s = ins_cpu_block[(b + k) % p] + OC.roundtrip(s, codec)
    return OC.roundtrip(s, codec)


def check_blocks(ins, outs, codec):
    """Every rank identical, and EVERY block bit-exact with the oracle's
    fold (blocks are independent: the oracle folds them on threads)."""
    from concurrent.futures import ThreadPoolExecutor
    p, n = len(ins), ins[0].numel()
    parts = OR.partition_blocks(n, p)
    for r in range(1, p):
        assert torch.equal(outs[r].view(torch.int32).to(outs[0].device), outs[0].view(torch.int32)), r
    host = [x.cpu().numpy() for x in ins]
    got = outs[0].cpu().numpy()

    def one(b):
        off, ln = parts[b]
        want = oracle_block([h[off:off + ln] for h in host], b, codec)
        assert_bits_equal(got[off:off + ln], want, f"block {b}")

    with ThreadPoolExecutor(min(p, 8)) as pool:
        list(pool.map(one, range(p)))


def run_emulated(P, ins, codec, p):
    tr = P.EmulatedTransport(p, timeout_s=120.0, max_elems=ins[0].numel())
    try:
        return run_ranks(tr, lambda r, ep: P.ring_allreduce(ins[r], r, p, ep, codec, iteration=1))
    finally:
        tr.close()


def test_c3_alexnet_quant8_p8_emulated(P):
    ins = make_inputs(8, ALEXNET, 1e-3, 3)
    outs = run_emulated(P, ins, P.Codec.QUANT8, 8)
    check_blocks(ins, outs, 2)


def test_c4_resnet50_none_p8_emulated(P):
    ins = make_inputs(8, RESNET50, 1e-2, 4)
    outs = run_emulated(P, ins, P.Codec.NONE, 8)
    check_blocks(ins, outs, 0)
    want = torch.stack(ins).double().sum(0)
    got = outs[0].double()
    atol = 1e-6 * max(1.0, want.abs().max().item())
    assert torch.allclose(got, want, rtol=1e-6, atol=atol)


def test_c4_resnet50_trunc16_p4_emulated(P):
    ins = make_inputs(4, RESNET50, 1e-2, 5)
    outs = run_emulated(P, ins, P.Codec.TRUNC16, 4)
    check_blocks(ins, outs, 1)


@pytest.mark.parametrize("codec,n", [(2, ALEXNET), (0, RESNET50)])
def test_c3_c4_on_real_gpus(P, codec, n):
    """Per-rank launches (one GPU per rank, or ranks sharing GPUs)."""
    p = 4
    base = make_inputs(p, n, 1e-3, 6)
    tr = real_transport(P, p, timeout_s=120.0, max_elems=n)
    ins = [x.to(tr.endpoint(r).device) for r, x in enumerate(base)]
    try:
        outs = run_ranks(tr, lambda r, ep: P.ring_allreduce(ins[r], r, p, ep, P.Codec(codec), iteration=2))
    finally:
        tr.close()
    check_blocks(base, outs, codec)


@pytest.mark.parametrize("codec", [1, 2])
@pytest.mark.parametrize("scale", [1e-38, 1e-6, 1e6, 1e30])
def test_scaled_inputs_on_real_gpus(P, codec, scale):
    """SURVEY 8(d)'s second input variant: N(0,1) x 10^k, here down to where
    quant8 block scales are subnormal (1e-38) and up to 1e30; per-rank
    launches, a non-divisible n, every block bit-exact with the oracle."""
    p, n = 4, 4_194_307
    base = make_inputs(p, n, scale, 11)
    tr = real_transport(P, p, timeout_s=60.0, max_elems=n)
    ins = [x.to(tr.endpoint(r).device) for r, x in enumerate(base)]
    try:
        outs = run_ranks(tr, lambda r, ep: P.ring_allreduce(ins[r], r, p, ep, P.Codec(codec), iteration=5))
    finally:
        tr.close()
    check_blocks(base, outs, codec)


def test_c1_mnist_mlp_pipe_sgd_bit_exact(P):
    """C1: MLP 784-500-500-10, p=4, codec none, width 2, global batch 100."""
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import ModelSpec
    data = OE.synthetic_blobs(dim=784, num_classes=10, num_samples=2000, seed=0)
    net = OE.Net("mlp", (784, 500, 500, 10))
    p, T, bs = 4, 6, 25
    rngs = [np.random.default_rng([0, r]) for r in range(p)]
    shards = [data.shard(r, p) for r in range(p)]

    def grad_fn(rank, t, params):
        b = OE.sample_from_shard(shards[rank], bs, rngs[rank])
        return OE.loss_and_grad(params.cpu().numpy(), net, data, b)

    cfg = RunConfig(mode="pipe_sgd", iterations=T, learning_rate=0.05, codec="none", depth=2, batch_size=bs,
                    seed=0)
    res = run_inproc_cluster(p, cfg, data, ModelSpec("mlp", (784, 500, 500, 10)), grad_fn=grad_fn)
    want = OE.run_trajectory(p, OE.Config(mode="pipe_sgd", iterations=T, learning_rate=0.05, codec=0,
                                          batch_size=bs, seed=0), data, net).params
    assert res[0].params.size == 648_010
    for r in res:
        assert_bits_equal(r.params, want, f"rank {r.rank}")


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs: on one GPU a rank's spinning ring CTAs can starve the peer "
                                     "rank's large cuDNN kernels that the ring is waiting for")
def test_c2_cnn_replicas_stay_identical(P):
    from paper_1811_03619_b200.engine import RankEngine, RunConfig
    from paper_1811_03619_b200.models import FlatModel, build_torch_model
    import threading
    p, T = 2, 6
    tr = real_transport(P, p, timeout_s=60.0, max_elems=5_000_000)
    init_lock = threading.Lock()  # torch's RNG is process-global: seed + init one thread at a time

    def op(r, ep):
        dev = ep.device
        with torch.cuda.device(dev):
            with init_lock:
                torch.manual_seed(0)
                mod, shape, classes = build_torch_model("c2")
            fm = FlatModel(mod, dev)
            g = torch.Generator(device="cpu").manual_seed(100 + r)
            x = torch.randn((64, *shape), generator=g).to(dev)
            y = torch.randint(0, classes, (64,), generator=g).to(dev)
            cfg = RunConfig(mode="pipe_sgd", iterations=T, learning_rate=0.01, codec="trunc16", batch_size=64)
            eng = RankEngine(r, p, ep, fm, cfg, lambda rank, t: (x, y), trace=False)
            eng.run()
            eng.cs.synchronize()
            eng.ms.synchronize()
            ep._check_errors(fm.num_params)
            return fm.params.cpu().numpy()

    try:
        res = run_ranks(tr, op)
    finally:
        tr.close()
    assert_bits_equal(res[1], res[0], "CNN replicas")
