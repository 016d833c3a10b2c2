"""Oracle restatement of the reference training engine (TEST INFRASTRUCTURE ONLY).

Restates, for parity runs of the GPU engine:
  * models.py:84-102   `init_params` (zeros; Glorot-uniform MLP weights)
  * models.py:118-195  forward / softmax-CE loss / backward, float64 inside,
                       float32 out
  * models.py:198-204  `sgd_update`  fl(w - fl(f32(lr) * g)), no FMA
  * engine.py:123-129  `aggregate_mean` fl(total / f32(p)), identity at p=1
  * data.py:41-43, :57-63, :66-90  shard / sample_from_shard / synthetic_blobs
  * engine.py:287-292  learning-rate decay
  * engine.py:323-336  local step: grad -> whole-vector D(C(grad))
  * engine.py:340-375  d_sync loop + drain
  * engine.py:379-448  width-K pipe loop: zero-primed slots, ring, whole-vector
                       re-compress of the sum (:407), consume t-K, drain K
  * engine.py:469-478  warm-up switch (sync epochs, drain, fresh pipe buffer)
  * engine.py:503-552  ps_sync: workers send D(C(grad)) (codec NONE on the
                       wire) to the server, which folds them in rank order from
                       its zero vector (collective.py:236-251), takes one SGD
                       step and broadcasts the parameters (:255-280)

Instead of threads and queues the oracle evaluates the data dependencies
directly: every rank's gradient for iteration t depends only on that rank's
parameters after update t, and the update at t consumes the aggregated slot
of t-K (pipe) or t-1 (sync). This yields the same floating-point trajectory
as the reference's threaded engine.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import codec as C
from .ring import ring_allreduce_all

D_SYNC, PIPE_SGD, PS_SYNC = "d_sync", "pipe_sgd", "ps_sync"


# --------------------------------------------------------------------- data

@dataclass(frozen=True)
class Blobs:
    features: np.ndarray  # (N, dim) float32
    labels: np.ndarray    # (N,) int64
    num_classes: int

    @property
    def num_samples(self) -> int:
        return self.features.shape[0]

    def shard(self, rank: int, p: int) -> np.ndarray:
        return np.arange(rank % p, self.num_samples, p)  # data.py:41-43


def synthetic_blobs(dim=64, num_classes=2, num_samples=10_000, separation=3.0, seed=0) -> Blobs:
    """data.py:66-90: orthogonal class centres `separation` sigmas apart."""
    g = np.random.default_rng(seed)
    basis, _ = np.linalg.qr(g.normal(size=(dim, num_classes)))
    centres = basis.T * (separation / np.sqrt(2.0))
    labels = np.arange(num_samples) % num_classes
    x = centres[labels] + g.normal(size=(num_samples, dim))
    return Blobs(x.astype(np.float32), labels.astype(np.int64), num_classes)


def sample_from_shard(shard: np.ndarray, size: int, g: np.random.Generator) -> np.ndarray:
    return shard[g.choice(len(shard), size=size, replace=False)]  # data.py:57-63


# ------------------------------------------------------------------- models

@dataclass(frozen=True)
class Net:
    """layer_dims = (input, hidden..., classes); flat layout W0,b0,W1,b1,...
    with W stored (d_in, d_out) row-major (models.py:57-66)."""
    kind: str            # "logistic" | "mlp"
    layer_dims: tuple

    def layout(self):
        off, out = 0, []
        for din, dout in zip(self.layer_dims[:-1], self.layer_dims[1:]):
            out.append((off, (din, dout)))
            off += din * dout
            out.append((off, (dout,)))
            off += dout
        return out

    @property
    def num_params(self) -> int:
        return sum((a + 1) * b for a, b in zip(self.layer_dims[:-1], self.layer_dims[1:]))


def init_params(net: Net, seed: int = 0) -> np.ndarray:
    w = np.zeros(net.num_params, np.float32)
    if net.kind == "mlp":
        g = np.random.default_rng(seed)
        for off, shape in net.layout():
            if len(shape) == 2:
                lim = np.sqrt(6.0 / (shape[0] + shape[1]))
                w[off:off + shape[0] * shape[1]] = g.uniform(-lim, lim, size=shape).reshape(-1).astype(np.float32)
    return w


def _tensors(w: np.ndarray, net: Net) -> list[np.ndarray]:
    out = []
    for off, shape in net.layout():
        k = int(np.prod(shape))
        out.append(w[off:off + k].reshape(shape).astype(np.float64))
    return out


def _logits(x: np.ndarray, w: np.ndarray, net: Net):
    ts = _tensors(w, net)
    nl = len(ts) // 2
    pre, a = [], x
    for i in range(nl):
        z = a @ ts[2 * i] + ts[2 * i + 1]
        pre.append(z)
        a = np.maximum(z, 0.0) if i < nl - 1 else z
    return a, pre, ts


def _logsoftmax(z: np.ndarray) -> np.ndarray:
    z = z - z.max(axis=1, keepdims=True)
    return z - np.log(np.exp(z).sum(axis=1, keepdims=True))


def loss_and_grad(w: np.ndarray, net: Net, data: Blobs, batch: np.ndarray):
    """Mean softmax CE and its float32 gradient (models.py:155-195)."""
    idx = np.asarray(batch, np.int64)
    x = data.features[idx].astype(np.float64)
    y = data.labels[idx]
    z, pre, ts = _logits(x, w, net)
    lp = _logsoftmax(z)
    loss = float(-lp[np.arange(len(y)), y].mean())
    # backward recomputes the forward exactly as the reference does
    z, pre, ts = _logits(x, w, net)
    pr = np.exp(_logsoftmax(z))
    pr[np.arange(len(y)), y] -= 1.0
    delta = pr / len(y)
    nl = len(ts) // 2
    acts = [x] + [np.maximum(pre[i], 0.0) for i in range(nl - 1)]
    g = np.empty(net.num_params, np.float32)
    lay = net.layout()
    for i in range(nl - 1, -1, -1):
        gw = acts[i].T @ delta
        gb = delta.sum(axis=0)
        wo, bo = lay[2 * i][0], lay[2 * i + 1][0]
        g[wo:wo + gw.size] = gw.reshape(-1).astype(np.float32)
        g[bo:bo + gb.size] = gb.astype(np.float32)
        if i > 0:
            delta = (delta @ ts[2 * i].T) * (pre[i - 1] > 0.0)
    if not np.isfinite(g).all():
        raise ValueError("non-finite gradient")
    return loss, g


def sgd_update(w: np.ndarray, g: np.ndarray, lr: float) -> np.ndarray:
    return (w - np.float32(lr) * g).astype(np.float32)  # models.py:198-204


def aggregate_mean(total: np.ndarray, p: int) -> np.ndarray:
    return total if p == 1 else (total / np.float32(p)).astype(np.float32)  # engine.py:123-129


# ------------------------------------------------------------------- engine

@dataclass
class Config:
    mode: str = D_SYNC
    iterations: int = 10
    learning_rate: float = 0.05
    codec: int = C.NONE
    depth: int = 2
    batch_size: int = 32
    warmup_epochs: int = 0
    seed: int = 0
    lr_decay_every: int = 0
    lr_decay_factor: float = 1.0


@dataclass
class Trajectory:
    params: np.ndarray                   # final params (identical on all ranks)
    losses: list[list[float]]            # [rank][t-1]
    local_grads: dict = field(default_factory=dict)   # (rank, t) -> D(C(grad))
    aggregated: dict = field(default_factory=dict)    # t -> slot the update consumes
    updates: list = field(default_factory=list)       # (iteration, consumed_tag, lr)


def lr_at(cfg: Config, t: int) -> float:
    if cfg.lr_decay_every <= 0:
        return cfg.learning_rate
    return cfg.learning_rate * (cfg.lr_decay_factor ** ((t - 1) // cfg.lr_decay_every))


GradFn = Callable[[int, int, np.ndarray], tuple[float, np.ndarray]]


def run_trajectory(p: int, cfg: Config, data: Blobs | None = None, net: Net | None = None,
                   batch_provider=None, grad_fn: GradFn | None = None,
                   init: np.ndarray | None = None, keep: bool = False) -> Trajectory:
    """Final parameters of a p-worker run (identical on every rank).

    grad_fn(rank, t, params) -> (loss, float32 grad) overrides the built-in
    model; otherwise the model/data restatement above supplies it with the
    engine's per-rank batch stream (engine.py:262-264, :294-297)."""
    if grad_fn is None:
        rngs = [np.random.default_rng([cfg.seed, r]) for r in range(p)]
        shards = [data.shard(r, p) for r in range(p)]

        def grad_fn(r, t, w):
            b = batch_provider(r, t) if batch_provider else sample_from_shard(shards[r], cfg.batch_size, rngs[r])
            return loss_and_grad(w, net, data, b)

        per_epoch = max(1, len(shards[0]) // cfg.batch_size)
    else:
        per_epoch = 1
    w = init_params(net, cfg.seed) if init is None else np.array(init, np.float32, copy=True)
    n = w.size
    T = cfg.iterations
    tr = Trajectory(params=w, losses=[[] for _ in range(p)])

    def update(w, total, tag, t):
        lr = lr_at(cfg, t)
        tr.updates.append((t, tag, lr))
        return sgd_update(w, aggregate_mean(total, p), lr)

    def local_step(t, w):
        grads = []
        for r in range(p):
            loss, g = grad_fn(r, t, w)
            tr.losses[r].append(loss)
            g = C.roundtrip(g, cfg.codec)  # engine.py:333 then decompress at :355/:400
            if keep:
                tr.local_grads[(r, t)] = g
            grads.append(g)
        return grads

    def ring(grads):
        return ring_allreduce_all(grads, cfg.codec).outputs[0]

    def sync_phase(t0, t1, w):
        pending, tag = None, 0
        for t in range(t0, t1 + 1):
            if pending is not None:
                w = update(w, pending, tag, t)
            pending, tag = ring(local_step(t, w)), t
            if keep:
                tr.aggregated[t] = pending
        if pending is not None:
            w = update(w, pending, tag, tag + 1)  # _drain_pending engine.py:368-375
        return w

    def pipe_phase(t0, t1, w):
        K = cfg.depth
        slots = {tag: np.zeros(n, np.float32) for tag in range(t0 - K, t0)}
        for t in range(t0, t1 + 1):
            w = update(w, slots.pop(t - K), t - K, t)
            summed = ring(local_step(t, w))
            slots[t] = C.roundtrip(summed, cfg.codec)  # engine.py:407
            if keep:
                tr.aggregated[t] = slots[t]
        for tag in range(t1 - K + 1, t1 + 1):
            w = update(w, slots.pop(tag), tag, tag + K)
        return w

    def ps_phase(w):
        for t in range(1, T + 1):
            total = np.zeros(n, np.float32)
            for g in local_step(t, w):   # collective.py:236-251: acc starts at the server's zeros
                total = total + g
            w = update(w, total, t, t)   # engine.py:542-545, then broadcast (bit-exact copy)
        return w

    if cfg.mode == PS_SYNC:
        w = ps_phase(w)
    elif cfg.mode == D_SYNC:
        w = sync_phase(1, T, w)
    elif cfg.mode == PIPE_SGD:
        warm = min(T, cfg.warmup_epochs * per_epoch)
        if warm > 0:
            w = sync_phase(1, warm, w)
        if warm < T:
            w = pipe_phase(warm + 1, T, w)
    else:
        raise ValueError(cfg.mode)
    tr.params = w
    return tr
