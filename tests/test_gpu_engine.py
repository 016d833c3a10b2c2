"""GPU parity of the width-K Pipe-SGD engine (paper_1811_03619_b200.engine).

* oracle gradients injected -> final weights BIT-EXACT with the reference's
  own trajectories (tests/golden/engine_golden.npz) for d_sync / pipe_sgd,
  every codec, p = 1, 2, 4 (ranks on distinct GPUs when available, else the
  emulated ring on one GPU): checks zero-priming, t-K consumption, the
  whole-vector re-compress of the sum, fl(g/p), fl(w - fl(lr*g)) and drain;
* torch gradients (fp32 on the GPU) -> weights within tolerance of the oracle
  (fp64 math in the reference), tolerance stated below;
* the reference's engine invariants: replicas bit-identical, exactly T+K
  updates with consumed tag t-K, allreduce(t) overlapping compute(t+1).
"""

import os

import numpy as np
import pytest
import torch

from golden.cases import ENGINE_CASES
from helpers import assert_bits_equal
from oracle import engine as OE

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.fixture(scope="module")
def P():
    import paper_1811_03619_b200 as P
    return P


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "engine_golden.npz"))


@pytest.fixture(scope="module")
def blobs():
    return OE.synthetic_blobs(dim=8, num_classes=3, num_samples=512, seed=1)


NETS = {"log": ((8, 3), "logistic"), "mlp": ((8, 16, 12, 3), "mlp")}


def oracle_grad_fn(data, net, p, seed, batch_size):
    """Reference batch stream per rank (engine.py:262-264) + oracle gradients."""
    rngs = [np.random.default_rng([seed, r]) for r in range(p)]
    shards = [data.shard(r, p) for r in range(p)]

    def fn(rank, t, params):
        b = OE.sample_from_shard(shards[rank], batch_size, rngs[rank])
        return OE.loss_and_grad(params.cpu().numpy(), net, data, b)

    return fn


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "unfused"])
@pytest.mark.parametrize("case", ENGINE_CASES, ids=lambda c: c[0])
def test_engine_bit_exact_with_oracle_gradients(P, gold, blobs, case, fused):
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import ModelSpec
    name, m, mode, codec, p, T, K, warm, lr, bs, dec = case
    dims, kind = NETS[m]
    spec = ModelSpec(kind, dims)
    net = OE.Net(kind, dims)
    cfg = RunConfig(mode=mode, iterations=T, learning_rate=lr, codec=codec, depth=K, batch_size=bs,
                    warmup_epochs=warm, seed=7, lr_decay_every=dec, lr_decay_factor=0.5)
    res = run_inproc_cluster(p, cfg, blobs, spec, grad_fn=oracle_grad_fn(blobs, net, p, 7, bs), fused=fused)
    for r in res:
        assert_bits_equal(r.params, gold[name], f"{name} rank {r.rank}")
    losses = [x[2] for x in res[0].metrics]
    np.testing.assert_allclose(losses, gold[name + "_loss"], rtol=1e-6)


# fp32 GPU math vs the reference's fp64-inside math: after T steps of SGD on
# this well-conditioned problem the weights agree to rtol 2e-5 / atol 2e-6
# (codec none). Lossy codecs can flip a rounding boundary, so they get an
# envelope of one trunc16 ulp (2^-8 relative) / one quant8 step instead.
TOL = {0: (2e-5, 2e-6), 1: (0, 4e-3), 2: (0, 2e-2)}


@pytest.mark.parametrize("mode", ["d_sync", "pipe_sgd"])
@pytest.mark.parametrize("codec", [0, 1, 2])
def test_engine_torch_gradients_within_tolerance(P, blobs, mode, codec):
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import ModelSpec
    p = 2
    spec = ModelSpec("mlp", (8, 16, 12, 3))
    cfg = RunConfig(mode=mode, iterations=10, learning_rate=0.05, codec=codec, batch_size=25, seed=3)
    res = run_inproc_cluster(p, cfg, blobs, spec)
    want = OE.run_trajectory(p, OE.Config(mode=mode, iterations=10, learning_rate=0.05, codec=codec,
                                          batch_size=25, seed=3), blobs, OE.Net("mlp", (8, 16, 12, 3))).params
    rtol, atol = TOL[codec]
    for r in res:
        np.testing.assert_allclose(r.params, want, rtol=rtol, atol=atol * max(1.0, np.abs(want).max()))
    for r in res[1:]:
        assert_bits_equal(r.params, res[0].params, "replicas diverged")


def test_staleness_tags_and_replicas(P, blobs):
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import ModelSpec
    depth, T = 2, 25
    cfg = RunConfig(mode="pipe_sgd", iterations=T, batch_size=16, seed=4, depth=depth, codec="quant8")
    res = run_inproc_cluster(2, cfg, blobs, ModelSpec("logistic", (8, 3)))
    for r in res:
        ups = [e for e in r.trace if e.stage == "update"]
        assert len(ups) == T + depth
        for e in ups:
            assert e.consumed_tag == e.iteration - depth
        assert sorted(e.consumed_tag for e in ups if e.consumed_tag >= 1) == list(range(1, T + 1))
        assert r.stats.messages == T * 2 * (2 - 1)
    assert_bits_equal(res[1].params, res[0].params, "replicas")


def test_first_updates_are_noops(P, blobs):
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import ModelSpec, init_params
    spec = ModelSpec("mlp", (8, 16, 3))
    cfg = RunConfig(mode="pipe_sgd", iterations=6, batch_size=16, seed=3, depth=3, snapshot_first=4)
    res = run_inproc_cluster(2, cfg, blobs, spec)
    w0 = init_params(spec, 3)
    snaps = dict(res[0].early_params)
    for t in (1, 2, 3):
        assert_bits_equal(snaps[t], w0, f"update {t}")
    assert not np.array_equal(snaps[4], w0)


@pytest.mark.skipif(NGPU < 2, reason="overlap is measured on two real GPUs")
def test_allreduce_overlaps_next_iteration_compute(P):
    """engine.py overlap contract (test_engine.py:278-307): the ring of
    iteration t runs while iteration t+1 computes."""
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import ModelSpec
    data = OE.synthetic_blobs(dim=1024, num_classes=10, num_samples=8192, seed=0)
    spec = ModelSpec("mlp", (1024, 4096, 4096, 10))
    cfg = RunConfig(mode="pipe_sgd", iterations=20, batch_size=512, seed=3)
    res = run_inproc_cluster(2, cfg, data, spec)
    tr = res[0].trace
    ar = {e.iteration: (e.start_ns, e.end_ns) for e in tr if e.stage == "allreduce"}
    comp = {e.iteration: (e.start_ns, e.end_ns) for e in tr if e.stage == "backward"}
    cand = ov = 0
    for t, (a0, a1) in ar.items():
        if t + 1 in comp:
            cand += 1
            c0, c1 = comp[t + 1]
            ov += min(a1, c1) > max(a0, c0)
    assert cand > 10 and ov >= cand * 0.5, (ov, cand)


@pytest.mark.parametrize("codec", [0, 2])
def test_comm_partition_is_bit_exact(P, codec):
    """The comm stream on a green-context SM partition (RankEngine comm_sms,
    engine.default_comm_partition) changes where the ring runs, not what it
    computes: weights bit-identical to the unpartitioned engine, and the
    partition is really made (one GPU per rank, or both ranks sharing one)."""
    from helpers import real_transport, run_ranks
    from paper_1811_03619_b200.engine import RankEngine, RunConfig
    from paper_1811_03619_b200.models import FlatModel, ModelSpec, SpecNet, init_params
    spec = ModelSpec("mlp", (64, 256, 10))
    p, T = 2, 8

    def train(sms):
        tr = real_transport(P, p, timeout_s=30.0, max_elems=spec.num_params, ctas=32)

        def op(r, ep):
            dev = ep.device
            with torch.cuda.device(dev):
                fm = FlatModel(SpecNet(spec), dev, init_params(spec, 1))
                g = torch.Generator(device="cpu").manual_seed(20 + r)
                x = torch.randn(32, 64, generator=g).to(dev)
                y = torch.randint(0, 10, (32,), generator=g).to(dev)
                cfg = RunConfig(mode="pipe_sgd", iterations=T, learning_rate=0.05, codec=codec, batch_size=32)
                eng = RankEngine(r, p, ep, fm, cfg, lambda rank, t: (x, y), trace=False, comm_sms=sms)
                eng.run()
                eng.cs.synchronize()
                eng.ms.synchronize()
                ep._check_errors(fm.num_params)
                return fm.params.cpu().numpy(), eng.comm_sms

        try:
            return run_ranks(tr, op)
        finally:
            tr.close()

    plain, part = train(0), train(16)
    for r in range(p):
        assert part[r][1] >= 16, "no green-context partition was made"
        assert_bits_equal(part[r][0], plain[r][0], f"rank {r} codec {codec}")


def test_comm_partition_rejects_budget_beyond_partition(P):
    from helpers import real_transport
    from paper_1811_03619_b200.engine import ConfigError, RankEngine, RunConfig
    from paper_1811_03619_b200.models import FlatModel, ModelSpec, SpecNet, init_params
    spec = ModelSpec("mlp", (8, 16, 3))
    tr = real_transport(P, 2, timeout_s=10.0, max_elems=spec.num_params, ctas=256)
    try:
        ep = tr.endpoint(0)
        with torch.cuda.device(ep.device):
            fm = FlatModel(SpecNet(spec), ep.device, init_params(spec, 1))
            with pytest.raises(ConfigError, match="partition"):
                RankEngine(0, 2, ep, fm, RunConfig(mode="pipe_sgd", iterations=2, batch_size=4), lambda r, t: None,
                           trace=False, comm_sms=16)
    finally:
        tr.close()


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_run_process_worker_under_torchrun_bit_exact():
    """One process per GPU (torchrun, CUDA IPC inboxes): run_process_worker
    with oracle gradients reproduces the oracle trajectory bit for bit."""
    import json
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tests", "process_worker_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert res and all(res.values()), res


def test_ps_sync_server_is_last_and_matches_workers(P, blobs):
    """test_engine.py:160-167: the server result comes last, params equal."""
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import ModelSpec
    cfg = RunConfig(mode="ps_sync", iterations=3, batch_size=16, seed=1)
    res = run_inproc_cluster(2, cfg, blobs, ModelSpec("logistic", (8, 3)))
    assert [r.is_server for r in res] == [False, False, True]
    assert_bits_equal(res[0].params, res[2].params, "server vs worker")
    assert res[0].stats.messages == 3 and res[2].stats.messages == 6


def test_star_collectives_match_reference_semantics(P):
    """collective.py:215-280: gather folds local_root + others in rank order;
    broadcast is bit-exact (test_collective.py:178-221)."""
    from helpers import run_ranks
    from paper_1811_03619_b200.collective import broadcast_from_root, gather_to_root
    p = 4
    tr = P.EmulatedTransport(p, timeout_s=30.0, max_elems=1 << 20)
    try:
        g = np.random.default_rng(5)
        ins = [(g.normal(0, 1, 1000_003) * 10.0 ** g.integers(-3, 3)).astype(np.float32) for _ in range(p)]
        for root in (0, 2):
            outs = run_ranks(tr, lambda r, ep: gather_to_root(ins[r], root, r, p, ep))
            want = ins[root].copy()
            for s in range(p):
                if s != root:
                    want = want + ins[s]
            assert_bits_equal(outs[root], want, f"gather root {root}")
            assert all(o is None for r, o in enumerate(outs) if r != root)
        value = g.normal(0, 1, 1_000_000).astype(np.float32)
        outs = run_ranks(tr, lambda r, ep: broadcast_from_root(value if r == 3 else None, 3, r, p, ep))
        for o in outs:
            assert o.tobytes() == value.tobytes()
    finally:
        tr.close()


def test_star_back_to_back_over_nvlink_across_sequence_wrap(P):
    """Real per-rank launches (no shared cooperative launch; one GPU per rank
    or ranks sharing GPUs): back-to-back
    gathers with changing roots and back-to-back broadcasts stay exact,
    because a star call closes only once every reader acknowledged the
    staged bytes; started two calls before the 32-bit call sequence wraps."""
    from helpers import real_transport, run_ranks
    from paper_1811_03619_b200 import _lib
    from paper_1811_03619_b200.collective import broadcast_from_root, gather_to_root
    p = 4
    tr = real_transport(P, p, timeout_s=30.0, max_elems=1 << 20)
    try:
        for r in range(p):
            _lib.call("gp_comm_set_call_counter", tr.endpoint(r)._comm, 0xFFFFFFFF - 2)
        g = np.random.default_rng(9)
        for it in range(6):
            ins = [g.normal(0, 1, 700_001).astype(np.float32) for _ in range(p)]
            root = it % p
            outs = run_ranks(tr, lambda r, ep: gather_to_root(ins[r], root, r, p, ep))
            want = ins[root].copy()
            for s in range(p):
                if s != root:
                    want = want + ins[s]
            assert_bits_equal(outs[root], want, f"gather {it} root {root}")
            value = g.normal(0, 1, 500_000 + it).astype(np.float32)
            outs = run_ranks(tr, lambda r, ep: broadcast_from_root(value if r == root else None, root, r, p, ep))
            for o in outs:
                assert o.tobytes() == value.tobytes()
    finally:
        tr.close()


def test_c1_mnist_mlp_torch_gradients_within_tolerance(P):
    """C1 at its real shape (BASELINE configs[0]): MLP 784-500-500-10
    (648,010 params), p = 4, codec none, Pipe-SGD width 2, batch 25 per rank,
    gradients from torch on the GPU (fp32) against the oracle trajectory
    (numpy, the reference's math). Tolerance after 10 steps: rtol 1e-4 and
    atol 1e-5 x max|w| (fp32 GEMM summation order differs from numpy's)."""
    from paper_1811_03619_b200.engine import RunConfig, run_inproc_cluster
    from paper_1811_03619_b200.models import ModelSpec
    data = OE.synthetic_blobs(dim=784, num_classes=10, num_samples=2000, seed=0)
    p, T = 4, 10
    cfg = RunConfig(mode="pipe_sgd", iterations=T, learning_rate=0.05, codec="none", depth=2, batch_size=25, seed=0)
    res = run_inproc_cluster(p, cfg, data, ModelSpec("mlp", (784, 500, 500, 10)))
    want = OE.run_trajectory(p, OE.Config(mode="pipe_sgd", iterations=T, learning_rate=0.05, codec=0, batch_size=25,
                                          seed=0), data, OE.Net("mlp", (784, 500, 500, 10))).params
    assert res[0].params.size == 648_010
    for r in res:
        np.testing.assert_allclose(r.params, want, rtol=1e-4, atol=1e-5 * max(1.0, np.abs(want).max()))
    for r in res[1:]:
        assert_bits_equal(r.params, res[0].params, "replicas diverged")
