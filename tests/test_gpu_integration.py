"""The reference's own training loop with the B200 ring underneath.

integration/gradpipe_b200.py is the ctypes module a gradpipe maintainer
would add. With it installed, the UNMODIFIED
reference `run_inproc_cluster` (engine.py:563-618) calls `ring_allreduce`
(engine.py:354-361 d_sync, :399-406 pipe) exactly as before, but every
ring runs as one gp_allreduce launch per rank through the C ABI. The final
weights and traffic stats of every rank must equal a plain reference run
bit for bit. Needs the reference package: baseline/_ref (it travels to the
GPU box) or /root/reference/pkg/src (the build container)."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "gradpipe")):
        sys.path.append(cand)
        break
gradpipe = pytest.importorskip("gradpipe", reason="reference package not available on this box")
sys.path.insert(0, os.path.join(ROOT, "integration"))
import gradpipe_b200  # noqa: E402
from gradpipe.compression import Codec  # noqa: E402
from gradpipe.data import synthetic_blobs  # noqa: E402
from gradpipe.engine import RunConfig, run_inproc_cluster  # noqa: E402
from gradpipe.models import mlp_model  # noqa: E402


@pytest.mark.parametrize("mode,codec,p", [("pipe_sgd", Codec.QUANT8, 4), ("pipe_sgd", Codec.TRUNC16, 2),
                                          ("pipe_sgd", Codec.NONE, 3), ("d_sync", Codec.QUANT8, 2),
                                          ("d_sync", Codec.NONE, 4)])
def test_reference_run_inproc_cluster_on_the_b200_ring_is_bit_exact(mode, codec, p):
    import gradpipe.engine as E
    data = synthetic_blobs(dim=16, num_classes=4, num_samples=1024, seed=3)
    spec = mlp_model(16, (64, 32), 4)
    cfg = RunConfig(mode=mode, iterations=10, learning_rate=0.05, codec=codec, batch_size=32, seed=1)
    plain = run_inproc_cluster(p, cfg, data, spec)
    calls = []
    undo = gradpipe_b200.install(gradpipe)
    real = gradpipe_b200.ring_allreduce_b200
    gradpipe_b200.ring_allreduce_b200 = lambda *a, **k: calls.append(1) or real(*a, **k)
    try:
        assert E.InProcTransport is not gradpipe.transport.InProcTransport
        b200 = run_inproc_cluster(p, cfg, data, spec)
    finally:
        gradpipe_b200.ring_allreduce_b200 = real
        undo()
    assert len(calls) == p * cfg.iterations, "every ring call of the reference loop went through the C ABI"
    for a, b in zip(plain, b200):
        assert a.rank == b.rank
        assert np.array_equal(a.params.view(np.uint32), b.params.view(np.uint32)), f"rank {a.rank} weights"
        assert (a.stats.messages, a.stats.payload_bytes, a.stats.frame_bytes) == \
               (b.stats.messages, b.stats.payload_bytes, b.stats.frame_bytes), f"rank {a.rank} stats"
