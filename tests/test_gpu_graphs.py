"""CUDA-graph replay of the pipelined step (RankEngine.capture_graphs /
step_graph) computes exactly what the eager engine computes: same weights,
bit for bit, after warm-up + graph steps + drain, for p = 1 and p = 2
(per-rank launches: over NVLink with two GPUs, else both ranks on one GPU),
every codec."""

import numpy as np
import pytest
import torch

from helpers import assert_bits_equal, real_transport, run_ranks

pytestmark = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def train(P, p, codec, graphs, T=12, W=3, mode="pipe_sgd", depth=2, decay=0, comm_sms=0):
    from paper_1811_03619_b200.engine import RankEngine, RunConfig
    from paper_1811_03619_b200.models import FlatModel, ModelSpec, SpecNet, init_params
    spec = ModelSpec("mlp", (64, 128, 10))
    tr = real_transport(P, p, timeout_s=30.0, max_elems=spec.num_params, ctas=64)

    def op(r, ep):
        dev = ep.device
        with torch.cuda.device(dev):
            fm = FlatModel(SpecNet(spec), dev, init_params(spec, 1))
            g = torch.Generator(device="cpu").manual_seed(10 + r)
            x = torch.randn(32, 64, generator=g).to(dev)
            y = torch.randint(0, 10, (32,), generator=g).to(dev)
            cfg = RunConfig(mode=mode, iterations=T + 2, learning_rate=0.05, codec=codec, batch_size=32, depth=depth,
                            lr_decay_every=decay, lr_decay_factor=0.5 if decay else 1.0)
            eng = RankEngine(r, p, ep, fm, cfg, lambda rank, t: (x, y), trace=False, comm_sms=comm_sms)
            pipe = mode == "pipe_sgd"
            step = eng.step if pipe else eng.ps_step if mode == "ps_sync" else eng.step_sync
            with torch.cuda.stream(eng.cs):
                if pipe:
                    eng.prime(1)
                for t in range(1, W + 1):
                    step(t)
                if graphs:
                    eng.capture_graphs((x, y))
                    for t in range(W + 1, T + 1):
                        eng.step_graph(t)
                    eng.drain_graph(T)
                else:
                    for t in range(W + 1, T + 1):
                        step(t)
                    if pipe:
                        eng.drain(T)
                    elif mode == "d_sync":
                        eng.drain_sync()
            eng.cs.synchronize()
            eng.ms.synchronize()
            ep._check_errors(fm.num_params)
            return fm.params.cpu().numpy(), eng.losses[1:T + 1].cpu().numpy()

    try:
        return run_ranks(tr, op)
    finally:
        tr.close()


@pytest.mark.parametrize("mode", ["pipe_sgd", "d_sync", "ps_sync"])
@pytest.mark.parametrize("codec", [0, 1, 2])
@pytest.mark.parametrize("p", [1, 2])
def test_graph_replay_matches_eager(P, p, codec, mode):
    eager = train(P, p, codec, graphs=False, mode=mode)
    graph = train(P, p, codec, graphs=True, mode=mode)
    for r in range(p):
        assert_bits_equal(graph[r][0], eager[r][0], f"p={p} codec={codec} rank {r} weights")
        np.testing.assert_array_equal(graph[r][1], eager[r][1])
    for r in range(1, p):
        assert_bits_equal(graph[r][0], graph[0][0], "replicas")


@pytest.mark.parametrize("codec", [1, 2])
@pytest.mark.parametrize("p", [1, 2])
def test_graph_replay_width_3_matches_eager(P, p, codec):
    eager = train(P, p, codec, graphs=False, depth=3)
    graph = train(P, p, codec, graphs=True, depth=3)
    for r in range(p):
        assert_bits_equal(graph[r][0], eager[r][0], f"width 3 p={p} codec={codec} rank {r}")
        np.testing.assert_array_equal(graph[r][1], eager[r][1])


@pytest.mark.parametrize("mode", ["pipe_sgd", "d_sync"])
@pytest.mark.parametrize("p", [1, 2])
def test_graph_replay_with_lr_decay_matches_eager(P, p, mode):
    """engine.py:287-292 decay under replay: the update graphs read the rate
    from device memory, written before every replay; the drain uses the
    eager engine's per-tag rates."""
    eager = train(P, p, 1, graphs=False, mode=mode, decay=4)
    graph = train(P, p, 1, graphs=True, mode=mode, decay=4)
    for r in range(p):
        assert_bits_equal(graph[r][0], eager[r][0], f"decay {mode} p={p} rank {r}")
        np.testing.assert_array_equal(graph[r][1], eager[r][1])
    const = train(P, p, 1, graphs=True, mode=mode, decay=0)
    assert not np.array_equal(const[0][0], graph[0][0]), "decay had no effect"


@pytest.mark.parametrize("codec", [0, 2])
def test_graph_replay_on_green_context_stream_matches_eager(P, codec):
    """The bench's configuration at N > 1: comm graphs captured and replayed
    on a green-context stream (RankEngine comm_sms) give the eager engine's
    weights bit for bit."""
    eager = train(P, 2, codec, graphs=False)
    # 32 SMs x 4 CTAs hold both ranks' 64-CTA rings when they share one GPU
    graph = train(P, 2, codec, graphs=True, comm_sms=32)
    for r in range(2):
        assert_bits_equal(graph[r][0], eager[r][0], f"green graphs codec={codec} rank {r}")
        np.testing.assert_array_equal(graph[r][1], eager[r][1])
