"""Pipe-SGD training engine on B200: width-K pipeline on two CUDA streams.

Drop-in for the train-step path of /root/reference/pkg/src/gradpipe/engine.py:
`RunConfig` (:80-107), `WorkerResult` (:110-120), `aggregate_mean` (:123-129),
`effective_mode` (:132-136), `GradientBuffer` (:188-235), `run_inproc_cluster`
(:563-618), plus `run_process_worker` (one rank per process under torchrun,
the analogue of `run_tcp_worker`, :621-646).

Reference structure -> B200 structure
  compute thread (:418-431)        -> compute stream: consume(t-K) -> fwd/bwd(t)
                                      -> local pre-compress D(C(grad_t))
  comm thread (:392-412)           -> comm stream: fused ring(t) -> whole-vector
                                      re-compress of the sum into slot t (:407)
  _LocalGradientMailbox (:139-185) -> K device buffers + "local ready" events
  GradientBuffer slots (:188-235)  -> K compressed device slots + "aggregated
                                      ready" events; write-once/take-clears
                                      bookkeeping kept on the host
  _apply_update (:302-307)         -> gp_consume_update: decode slot, fl(g/p),
                                      fl(w - fl(lr*g)) in one HBM pass
One host thread per rank only *enqueues*; the two streams overlap iteration
t's allreduce with iteration t+1's update + forward/backward exactly as in
Alg. 1 (update at t consumes the aggregated gradient of t-K; slots for
tags t_start-K..t_start-1 are zero; K in-flight gradients are drained).
d_sync is the same machinery with depth 1, no re-compress and the compute
stream waiting for the ring every iteration (engine.py:340-375).

By default (fused=True) the local pre-compress and the pipe re-compress are
folded into the single ring kernel of each iteration (gp_allreduce_ex with
GP_RING_PRECOMPRESS | GP_RING_SLOT_OUT). For the steady state,
capture_graphs / step_graph replay the iteration as CUDA graphs (update /
compute / comm per parity, any width, learning-rate decay through a
device-resident rate), bit-identical to the eager step.
"""

from __future__ import annotations

import contextlib
import os
import threading
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _lib
from .collective import allreduce_into
from .compression import Codec, CodecStatus, as_codec, encode_async, roundtrip_async
from .errors import CodecError, ConfigError, EngineError
from .models import FlatModel, ModelSpec, SpecNet, init_params
from .transport import EmulatedTransport, GpuEndpoint, GpuTransport, TrafficStats

MODE_PS_SYNC = "ps_sync"
MODE_D_SYNC = "d_sync"
MODE_PIPE_SGD = "pipe_sgd"
MODES = (MODE_PS_SYNC, MODE_D_SYNC, MODE_PIPE_SGD)

STAGE_UPDATE = "update"
STAGE_FORWARD = "forward"
STAGE_BACKWARD = "backward"
STAGE_COMPRESS = "compress"
STAGE_ALLREDUCE = "allreduce"
STAGE_DECOMPRESS = "decompress"
STAGE_BARRIER = "barrier"
STAGE_IDLE = "idle"


@contextlib.contextmanager
def capture(graph: torch.cuda.CUDAGraph, stream: torch.cuda.Stream):
    """torch.cuda.graph without its device-wide synchronize: a rank sharing
    this GPU with other ranks may be mid-capture (a device sync is illegal
    then) or mid-call (its ring waits for this rank, so a device sync could
    wait on it). Callers synchronize their own streams first."""
    with torch.cuda.stream(stream):
        graph.capture_begin(capture_error_mode="thread_local")
        try:
            yield graph
        finally:
            graph.capture_end()


@dataclass(frozen=True)
class TraceEvent:
    rank: int
    iteration: int
    stage: str
    start_ns: int
    end_ns: int
    consumed_tag: int | None = None


@dataclass(frozen=True)
class RunConfig:
    mode: str = MODE_D_SYNC
    iterations: int = 100
    learning_rate: float = 0.05
    codec: Codec = Codec.NONE
    depth: int = 2  # iteration dependency K (pipe_sgd only)
    batch_size: int = 32
    warmup_epochs: int = 0
    eval_interval: int = 0
    seed: int = 0
    lr_decay_every: int = 0
    lr_decay_factor: float = 1.0
    snapshot_first: int = 0

    def __post_init__(self) -> None:
        if self.mode not in MODES:
            raise ConfigError(f"unknown mode {self.mode!r}")
        if self.iterations < 1:
            raise ConfigError("need at least one iteration")
        if self.learning_rate <= 0:
            raise ConfigError("learning rate must be positive")
        if self.mode == MODE_PIPE_SGD and self.depth < 2:
            raise ConfigError("pipelined training needs depth K >= 2")
        if self.batch_size < 1:
            raise ConfigError("batch size must be >= 1")
        if self.warmup_epochs < 0 or self.eval_interval < 0:
            raise ConfigError("warmup_epochs and eval_interval must be >= 0")
        object.__setattr__(self, "codec", as_codec(self.codec))


@dataclass
class WorkerResult:
    rank: int
    params: np.ndarray
    trace: list[TraceEvent]
    metrics: list[tuple[int, float, float]]  # (iteration, wall_ms, train_loss)
    eval_points: list[tuple[int, np.ndarray]]
    early_params: list[tuple[int, np.ndarray]]
    stats: TrafficStats
    train_seconds: float
    is_server: bool = False
    device_seconds: float = 0.0


def aggregate_mean(total, p: int):
    """Aggregated gradient sum -> mean over the global batch (fp32 division)."""
    if p < 1:
        raise ConfigError("worker count must be >= 1")
    if p == 1:
        return total
    if isinstance(total, torch.Tensor):
        return total / torch.tensor(p, dtype=torch.float32, device=total.device)
    return (np.asarray(total, np.float32) / np.float32(p)).astype(np.float32)


def effective_mode(config: RunConfig, epoch: int) -> str:
    if config.mode != MODE_PIPE_SGD:
        return config.mode
    return MODE_D_SYNC if epoch < config.warmup_epochs else MODE_PIPE_SGD


class GradientBuffer:
    """Depth-K ring of aggregated-gradient slots (engine.py:188-235).

    Host-side bookkeeping with the reference's contract: the slot for tag t
    is written once, `take` clears it, a second write to an occupied slot is
    an EngineError. Each slot carries the CUDA event that marks its device
    data ready, so `take` never blocks the host: the consumer's stream waits."""

    def __init__(self, depth: int, timeout_s: float = 30.0):
        self.depth = depth
        self._slots: list = [None] * depth
        self._lock = threading.Lock()

    def put(self, tag: int, block, ready: torch.cuda.Event | None = None) -> None:
        idx = tag % self.depth
        with self._lock:
            if self._slots[idx] is not None:
                raise EngineError(f"aggregated-gradient slot for iteration {tag} written twice "
                                  f"(still holds iteration {self._slots[idx][0]})")
            self._slots[idx] = (tag, block, ready)

    def take(self, tag: int, stream: torch.cuda.Stream | None = None):
        idx = tag % self.depth
        with self._lock:
            if self._slots[idx] is None:
                raise EngineError(f"aggregated gradient {tag} was never produced")
            slot_tag, block, ready = self._slots[idx]
            if slot_tag != tag:
                raise EngineError(f"slot {idx} holds iteration {slot_tag}, expected {tag}")
            self._slots[idx] = None
        if ready is not None and stream is not None:
            stream.wait_event(ready)
        return block


@dataclass
class _Slot:
    """A compressed aggregated gradient on the device."""
    codec: Codec
    payload: torch.Tensor      # uint8, n * width bytes
    status: CodecStatus        # quant8 scale at status.scale_view


BatchFn = Callable[[int, int], tuple]


class RankEngine:
    """One rank's Pipe-SGD loop on one GPU (enqueue-only host thread)."""

    def __init__(self, rank: int, world: int, endpoint: GpuEndpoint, fm: FlatModel, config: RunConfig,
                 batch_fn: BatchFn, trace: bool = True, grad_fn=None, fused: bool = True, comm_sms: int = 0):
        """fused=True (default): the comm stream runs ONE kernel per iteration —
        the ring with the local pre-compress applied on load and the pipe
        re-compress written as the slot by its allgather (gp_allreduce_ex);
        the raw gradient sits in K alternating buffers. fused=False keeps the
        separate pre-compress / ring / re-compress kernels (reference order)."""
        self.rank, self.world, self.ep, self.fm, self.cfg = rank, world, endpoint, fm, config
        self.fused = fused
        self.batch_fn = batch_fn
        self.grad_fn = grad_fn
        self.dev = fm.params.device
        self.n = fm.num_params
        self.cs = torch.cuda.Stream(self.dev)
        # comm stream priority (COMM_PRIORITY; PIPESGD_COMM_PRIORITY overrides;
        # lower = higher, 0 = same as compute): its CTAs are scheduled ahead of
        # compute CTAs as SMs free up
        prio = int(os.environ.get("PIPESGD_COMM_PRIORITY", COMM_PRIORITY))
        self.ms = torch.cuda.Stream(self.dev, priority=prio)
        # comm_sms > 0: the comm stream lives in a green context of that many
        # SMs (greenctx.py), so the pipelined ring occupies a fixed slice of
        # the GPU; the communicator's CTA budget must fit it (4 CTAs per SM;
        # ranks sharing a GPU share the slice, so their budgets together)
        self.comm_sms = 0
        if comm_sms > 0:
            from .greenctx import green_stream
            try:
                self.ms, self.comm_sms = green_stream(self.dev.index, comm_sms, prio)
            except Exception as err:  # noqa: BLE001 - no green contexts: plain stream, full budget
                import warnings
                warnings.warn(f"green context unavailable ({err}); the comm stream shares every SM")
            if self.comm_sms and world > 1 and endpoint.info()["ctas"] > 4 * self.comm_sms:
                raise ConfigError(f"ring CTA budget {endpoint.info()['ctas']} exceeds the {self.comm_sms}-SM "
                                  f"comm partition ({4 * self.comm_sms} resident CTAs)")
        self.tracing = trace
        self.events: list = []  # (iteration, stage, ev0, ev1, consumed)
        K = max(config.depth, 1)
        self.K = K
        if fused:
            fm.ensure_grad_buffers(K)
        w = config.codec.bytes_per_elem
        with torch.cuda.device(self.dev):
            self.local = [torch.empty(self.n, dtype=torch.float32, device=self.dev) for _ in range(K)]
            self.summed = torch.empty(self.n, dtype=torch.float32, device=self.dev)
            self.slots = [_Slot(config.codec, torch.zeros(self.n * w, dtype=torch.uint8, device=self.dev),
                                CodecStatus(self.dev)) for _ in range(K)]
            # d_sync consumes the raw fp32 sum; at p=1 the reference's ring is an
            # identity copy (collective.py:153-154), so the local buffer is the sum
            if world == 1:
                self.sync_slots = [_Slot(Codec.NONE, self.local[i].view(torch.uint8), CodecStatus(self.dev))
                                   for i in range(K)]
            else:
                self.sync_slots = [_Slot(Codec.NONE, self.summed.view(torch.uint8), CodecStatus(self.dev))] * K
            self.local_status = [CodecStatus(self.dev) for _ in range(K)]
            self.slot_nonfinite = torch.zeros(1, dtype=torch.int32, device=self.dev)
            self.losses = torch.zeros(config.iterations + 2, dtype=torch.float32, device=self.dev)
        self.ev_local = [torch.cuda.Event() for _ in range(K)]
        # gradient buffer i already zero (cleared by the comm stream after the
        # fused ring / encode read it): the next backward into it skips its zero_
        self.grad_clean = [True] * K
        self.buffer = GradientBuffer(K)
        self.iter_done: dict[int, torch.cuda.Event] = {}
        self._pending = None
        self.early_params: list = []
        self.eval_points: list = []
        self.updates_seen = 0

    # ---------------------------------------------------------------- helpers
    def _lr(self, t: int) -> float:
        c = self.cfg
        if c.lr_decay_every <= 0:
            return c.learning_rate
        return c.learning_rate * (c.lr_decay_factor ** ((t - 1) // c.lr_decay_every))

    def reserve_events(self, n: int) -> None:
        """Create n timing events up front: the stage trace then records
        pre-made events instead of creating ~6 per step on the host, which
        matters when the host must enqueue a 0.1 ms step (C1)."""
        self._ev_pool = [torch.cuda.Event(enable_timing=True) for _ in range(n)]

    def _new_event(self):
        pool = getattr(self, "_ev_pool", None)
        return pool.pop() if pool else torch.cuda.Event(enable_timing=True)

    def _ev(self, stream):
        e = self._new_event()
        e.record(stream)
        return e

    def _rec(self, t, stage, e0, e1, consumed=None):
        if self.tracing:
            self.events.append((t, stage, e0, e1, consumed))

    def _consume(self, slot: _Slot, tag: int, t: int) -> None:
        """w <- fl(w - fl(lr * fl(D(slot) / p)))   on the compute stream."""
        lr = float(np.float32(self._lr(t)))
        e0 = self._ev(self.cs) if self.tracing else None
        _lib.call("gp_consume_update", self.fm.params.data_ptr(), int(slot.codec), slot.payload.data_ptr(),
                  slot.status.scale_view.data_ptr(), self.n, lr, self.world, self.cs.cuda_stream)
        if self.tracing:
            self._rec(t, STAGE_UPDATE, e0, self._ev(self.cs), tag)
        self.updates_seen += 1
        if self.updates_seen <= self.cfg.snapshot_first:
            self.early_params.append((t, self.fm.params.clone()))

    def _compute_local(self, t: int) -> None:
        """fwd + bwd (+ whole-vector D(C(grad)) when not fused) (engine.py:323-336)."""
        i = t % self.K
        if self.fused:
            self.fm.use_grad_buffer(i)
        e0 = self._ev(self.cs) if self.tracing else None
        if self.grad_fn is not None:
            self.cs.synchronize()
            loss, g = self.grad_fn(self.rank, t, self.fm.params)
            self.fm.grads.copy_(torch.as_tensor(np.asarray(g, np.float32)).to(self.dev))
            self.losses[t].fill_(float(loss))
        else:
            x, y = self.batch_fn(self.rank, t)
            loss = self.fm.loss_and_grad(x, y, zero=not (self.fused and self.grad_clean[i]))
            self.losses[t].copy_(loss)
        self.grad_clean[i] = False
        e1 = self._ev(self.cs) if self.tracing else None
        if not self.fused:
            roundtrip_async(self.fm.grads, self.cfg.codec, self.local[i], self.local_status[i], self.cs.cuda_stream)
        self.ev_local[i].record(self.cs)
        if self.tracing:
            self._rec(t, STAGE_BACKWARD, e0, e1)
            if not self.fused:
                self._rec(t, STAGE_COMPRESS, e1, self._ev(self.cs))
        if self.cfg.eval_interval and self.rank == 0 and t % self.cfg.eval_interval == 0:
            self.eval_points.append((t, self.fm.params.clone()))

    def _communicate(self, t: int, requant: bool) -> _Slot:
        """Comm stream: ring(local[t]) -> (pipe) C(sum) into slot t."""
        if self.fused:
            return self._communicate_fused(t, requant)
        i = t % self.K
        self.ms.wait_event(self.ev_local[i])
        e0 = self._ev(self.ms) if self.tracing else None
        if self.world > 1:
            allreduce_into(self.local[i], self.summed, self.ep, self.cfg.codec, t, self.ms)
            src = self.summed
        else:
            src = self.local[i]  # p == 1: the ring is the identity (no codec, no copy)
        e1 = self._ev(self.ms) if self.tracing else None
        if requant:
            slot = self.slots[i]
            encode_async(src, self.cfg.codec, slot.payload, slot.status, self.ms.cuda_stream)
        else:
            slot = self.sync_slots[i]
        ready = torch.cuda.Event(enable_timing=self.tracing)
        ready.record(self.ms)
        if self.tracing:
            self._rec(t, STAGE_ALLREDUCE, e0, ready)
            if self.world > 1:
                self._rec(t, "ring", e0, e1)
            if requant:
                self._rec(t, "recompress", e1, ready)
        self.buffer.put(t, slot, ready)
        return slot

    def _communicate_fused(self, t: int, requant: bool) -> _Slot:
        """Comm stream, one kernel: raw grad -> D(C(.)) -> ring -> (pipe) C(sum)
        written straight into slot t (p == 1: C(D(C(g))) == C(g), one encode)."""
        i = t % self.K
        g = self.fm.grad_bufs[i]
        self.ms.wait_event(self.ev_local[i])
        e0 = self._ev(self.ms) if self.tracing else None
        codec = self.cfg.codec
        if requant:
            slot = self.slots[i]
            if self.world > 1:
                allreduce_into(g, self.summed, self.ep, codec, t, self.ms, precompress=True,
                               slot=slot.payload, slot_scale=slot.status.scale_view)
            else:
                encode_async(g, codec, slot.payload, slot.status, self.ms.cuda_stream)
        else:
            slot = self.sync_slots[i]
            if self.world > 1:
                allreduce_into(g, self.summed, self.ep, codec, t, self.ms, precompress=True)
            else:
                roundtrip_async(g, codec, self.local[i], self.local_status[i], self.ms.cuda_stream)
        e1 = self._ev(self.ms) if self.tracing else None
        with torch.cuda.stream(self.ms):  # clean for the backward of t + K (ordered before `ready`)
            g.zero_()
        self.grad_clean[i] = True
        ready = torch.cuda.Event(enable_timing=self.tracing)
        ready.record(self.ms)
        if self.tracing:
            self._rec(t, STAGE_ALLREDUCE, e0, e1)
            self._rec(t, "ring" if self.world > 1 else "recompress", e0, e1)
        self.buffer.put(t, slot, ready)
        return slot

    # ------------------------------------------------------------------ loops
    # Incremental API (used by bench.py to time exactly K steady-state steps):
    #   pipe: prime(t0); step(t) for t0..t1; drain(t1)
    #   sync: step_sync(t) for t0..t1; drain_sync()
    def prime(self, t0: int) -> None:
        """Zero slots for tags t0-K .. t0-1 (engine.py:382-388)."""
        K = self.K
        for tag in range(t0 - K, t0):
            slot = self.slots[tag % K]
            slot.payload.zero_()
            slot.status.t.zero_()
            ev = torch.cuda.Event()
            ev.record(self.cs)
            self.buffer.put(tag, slot, ev)

    def step(self, t: int) -> None:
        """One pipelined iteration: update with slot t-K, compute t, ring t."""
        self._consume(self.buffer.take(t - self.K, self.cs), t - self.K, t)
        self._compute_local(t)
        self._communicate(t, requant=True)
        self._mark(t)

    def drain(self, t1: int) -> None:
        for tag in range(t1 - self.K + 1, t1 + 1):
            self._consume(self.buffer.take(tag, self.cs), tag, tag + self.K)

    def step_sync(self, t: int) -> None:
        if self._pending is not None:
            self._consume(self.buffer.take(self._pending, self.cs), self._pending, t)
        self._compute_local(t)
        self._communicate(t, requant=False)
        self._pending = t
        self._mark(t)

    def drain_sync(self) -> None:
        if self._pending is not None:
            self._consume(self.buffer.take(self._pending, self.cs), self._pending, self._pending + 1)
        self._pending = None

    def sync_phase(self, t0: int, t1: int) -> None:
        """d_sync (engine.py:340-375): update(pending) -> compute -> ring."""
        self._pending = None
        for t in range(t0, t1 + 1):
            self.step_sync(t)
        self.drain_sync()

    def pipe_phase(self, t0: int, t1: int) -> None:
        """pipe_sgd (engine.py:379-448) with zero-primed slots and K-drain."""
        self.prime(t0)
        for t in range(t0, t1 + 1):
            self.step(t)
        self.drain(t1)

    # --------------------------------------------------------- CUDA graphs
    def capture_graphs(self, batch) -> None:
        """Capture the steady-state iteration as CUDA graphs.

        d_sync: K graphs on the compute stream, parity i = t % K: consume the
        sum of t-1 + forward/backward into gradient buffer i + the fused ring
        into the fp32 sum (nothing to overlap, so one stream; same kernels and
        order as step_sync).

        pipe_sgd: for parity i = t % K: update graph i (compute stream) =
        consume slot i; compute graph i = forward/backward of `batch` into
        gradient buffer i; comm graph i (comm stream) = the fused ring from
        gradient buffer i into slot i.

        Update, compute and comm are separate graphs (one extra graph launch
        per step) so CUDA events between them time each of our kernels inside
        the timed region.
        Replays are linked by events between the streams, so iteration t's
        ring still overlaps iteration t+1's compute. The ring kernel reads its
        call sequence number on the device, so every replay is a new call.
        Requirements: pipe or d_sync mode, fused path, real GPU transport,
        static batch tensors (refilled in place by the caller). Learning-rate
        decay works: the update graphs read the rate from device memory."""
        cfg = self.cfg
        if not self.fused or cfg.mode not in (MODE_PIPE_SGD, MODE_D_SYNC, MODE_PS_SYNC) or self.grad_fn is not None:
            raise ConfigError("graph mode needs fused pipe_sgd, d_sync or ps_sync and a model")
        if cfg.eval_interval or cfg.snapshot_first:
            # their host-side snapshots live in the eager step (engine.py run()
            # keeps them); a replayed step would silently skip them
            raise ConfigError("graph mode does not take eval_interval / snapshot_first snapshots; run eagerly")
        if type(self.ep).__name__ == "EmulatedEndpoint":
            raise ConfigError("graph mode needs one GPU per rank (the emulated ring rendezvouses on the host)")
        # one (x, y) for every parity, or a list of K (x, y): compute graph i
        # reads batch i (double-buffered inputs prefetched on a copy stream)
        batches = list(batch) if isinstance(batch, list) else [batch] * self.K
        if len(batches) != self.K:
            raise ConfigError(f"need {self.K} per-parity batches, got {len(batches)}")
        # the update graphs read the learning rate from device memory, written
        # before each replay with lr_at(t) (engine.py:287-292 decay)
        self.lr_dev = torch.full((1,), float(np.float32(cfg.learning_rate)), dtype=torch.float32, device=self.dev)
        lr = self.lr_dev
        self.static_loss = [torch.zeros((), dtype=torch.float32, device=self.dev) for _ in range(self.K)]
        self.g_update, self.g_compute, self.g_comm = [], [], []
        self.ev_agg = [torch.cuda.Event() for _ in range(self.K)]
        # this rank's streams only: a device-wide sync could wait on a peer
        # rank's ring that shares the GPU and waits for this rank's next call
        torch.cuda.current_stream(self.dev).synchronize()
        self.cs.synchronize()
        self.ms.synchronize()
        # the ring's iteration tag (the reference's _expect check, collective.py:52-64)
        # is read from device memory by the captured launches; written with t
        # before every comm replay
        self.tag_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)
        if self.world > 1:
            _lib.call("gp_comm_set_iteration_source", self.ep._comm, self.tag_dev.data_ptr())
        try:
            if cfg.mode == MODE_D_SYNC:
                self._capture_sync_graphs(batches, lr)
            elif cfg.mode == MODE_PS_SYNC:
                self._capture_ps_graphs(batches, lr)
            else:
                self._capture_pipe_graphs(batches, lr)
        finally:
            if self.world > 1:
                _lib.call("gp_comm_set_iteration_source", self.ep._comm, None)

    def _capture_pipe_graphs(self, batches, lr) -> None:
        cfg = self.cfg
        for i in range(self.K):
            slot = self.slots[i]
            gu = torch.cuda.CUDAGraph()
            with capture(gu, self.cs):
                _lib.call("gp_consume_update_dev", self.fm.params.data_ptr(), int(slot.codec), slot.payload.data_ptr(),
                          slot.status.scale_view.data_ptr(), self.n, lr.data_ptr(), self.world, self.cs.cuda_stream)
            self.g_update.append(gu)
            gc = torch.cuda.CUDAGraph()
            with capture(gc, self.cs):
                self.fm.use_grad_buffer(i)
                self.static_loss[i].copy_(self.fm.loss_and_grad(*batches[i], zero=False))
            gm = torch.cuda.CUDAGraph()
            with capture(gm, self.ms):
                g = self.fm.grad_bufs[i]
                if self.world > 1:
                    allreduce_into(g, self.summed, self.ep, cfg.codec, 0, self.ms, precompress=True,
                                   slot=slot.payload, slot_scale=slot.status.scale_view)
                else:
                    encode_async(g, cfg.codec, slot.payload, slot.status, self.ms.cuda_stream)
            self.g_compute.append(gc)
            self.g_comm.append(gm)
        self.graph_ready_tag = {}

    def _capture_sync_graphs(self, batches, lr) -> None:
        K, codec = self.K, self.cfg.codec
        for i in range(K):
            pend = self.sync_slots[(i - 1) % K]  # holds the sum of t-1 when t % K == i
            gu = torch.cuda.CUDAGraph()
            with capture(gu, self.cs):
                _lib.call("gp_consume_update_dev", self.fm.params.data_ptr(), int(Codec.NONE), pend.payload.data_ptr(),
                          pend.status.scale_view.data_ptr(), self.n, lr.data_ptr(), self.world, self.cs.cuda_stream)
            gc = torch.cuda.CUDAGraph()
            with capture(gc, self.cs):
                self.fm.use_grad_buffer(i)
                self.static_loss[i].copy_(self.fm.loss_and_grad(*batches[i], zero=False))
            gm = torch.cuda.CUDAGraph()
            with capture(gm, self.cs):
                g = self.fm.grad_bufs[i]
                if self.world > 1:
                    allreduce_into(g, self.summed, self.ep, codec, 0, self.cs, precompress=True)
                else:
                    roundtrip_async(g, codec, self.local[i], self.local_status[i], self.cs.cuda_stream)
            self.g_update.append(gu)
            self.g_compute.append(gc)
            self.g_comm.append(gm)
        self.graph_pending = None

    def _capture_ps_graphs(self, batches, lr) -> None:
        """ps_sync as graphs, parity i = t % K: compute (forward/backward into
        gradient buffer i, zeroing it first like the eager step), compress
        (local D(C(grad))) and the star round (gather to the root, the root's
        SGD step with the device-resident rate, broadcast of the parameters)
        -- ps_step's kernels in ps_step's order. The star kernels read their
        call sequence on the device, so every replay is a new call; the
        iteration tag they carry is the capture step's, the same on every rank."""
        K, codec, root = self.K, self.cfg.codec, 0
        for i in range(K):
            gc = torch.cuda.CUDAGraph()
            with capture(gc, self.cs):
                self.fm.use_grad_buffer(i)
                self.static_loss[i].copy_(self.fm.loss_and_grad(*batches[i]))
            gz = torch.cuda.CUDAGraph()
            with capture(gz, self.cs):
                roundtrip_async(self.fm.grad_bufs[i], codec, self.local[i], self.local_status[i], self.cs.cuda_stream)
            gm = torch.cuda.CUDAGraph()
            with capture(gm, self.cs):
                self.ep._star(self.local[i], self.summed if self.rank == root else None, self.n, root, 0, True, 0,
                              self.cs)
                if self.rank == root:
                    _lib.call("gp_consume_update_dev", self.fm.params.data_ptr(), int(Codec.NONE),
                              self.summed.data_ptr(), self.local_status[i].scale_view.data_ptr(), self.n,
                              lr.data_ptr(), self.world, self.cs.cuda_stream)
                self.ep._star(self.fm.params, self.fm.params, self.n, root, 1, False, 0, self.cs)
            self.g_compute.append(gc)
            self.g_update.append(gz)  # the compress graph
            self.g_comm.append(gm)

    def _step_graph_ps(self, t: int) -> None:
        i = t % self.K
        tr = self.tracing
        self._set_lr(t)
        e0 = self._ev(self.cs) if tr else None
        self.g_compute[i].replay()
        self.losses[t].copy_(self.static_loss[i])
        e1 = self._ev(self.cs) if tr else None
        self.g_update[i].replay()
        e2 = self._ev(self.cs) if tr else None
        self.g_comm[i].replay()
        if tr:
            e3 = self._ev(self.cs)
            self._rec(t, STAGE_BACKWARD, e0, e1)
            self._rec(t, STAGE_COMPRESS, e1, e2)
            self._rec(t, STAGE_ALLREDUCE, e2, e3)
        self.updates_seen += 1
        self._mark(t)

    def _step_graph_sync(self, t: int) -> None:
        """d_sync by replay: the graph consumes t-1 itself, so only an eager
        predecessor (the warm-up's last step) has to be waited for."""
        i = t % self.K
        if self.graph_pending is None:
            if self._pending is None or self._pending != t - 1:
                raise ConfigError("d_sync graph replay needs the eager step t-1 just before")
            self.buffer.take(self._pending, self.cs)
            self._pending = None
        elif self.graph_pending != t - 1:
            raise ConfigError("d_sync graph steps must be consecutive")
        tr = self.tracing
        self._set_lr(t)
        e0 = self._ev(self.cs) if tr else None
        self.g_update[i].replay()
        e1 = self._ev(self.cs) if tr else None
        self.g_compute[i].replay()
        self.losses[t].copy_(self.static_loss[i])
        e2 = self._ev(self.cs) if tr else None
        if self.world > 1:
            self.tag_dev.fill_(t)
        self.g_comm[i].replay()
        e3 = self._ev(self.cs) if tr else None
        self.fm.grad_bufs[i].zero_()  # clean for the backward of t + K
        if tr:
            self._rec(t, STAGE_UPDATE, e0, e1, t - 1)
            self._rec(t, STAGE_BACKWARD, e1, e2)
            self._rec(t, STAGE_ALLREDUCE, e2, e3)
            self._rec(t, "ring" if self.world > 1 else "compress", e2, e3)
        self.graph_pending = t
        self._mark(t)

    def step_graph(self, t: int) -> None:
        """One iteration by graph replay (after prime / eager warm-up)."""
        if self.cfg.mode == MODE_D_SYNC:
            self._step_graph_sync(t)
            return
        if self.cfg.mode == MODE_PS_SYNC:
            self._step_graph_ps(t)
            return
        i = t % self.K
        prev = self.graph_ready_tag.pop(i, None)
        if prev is not None:
            self.cs.wait_event(self.ev_agg[i])
        else:  # slot i still holds the eager pipeline's tag t-K: wait for it
            self.buffer.take(t - self.K, self.cs)
        tr = self.tracing
        self._set_lr(t)
        e0 = self._ev(self.cs) if tr else None
        self.g_update[i].replay()
        eu = self._ev(self.cs) if tr else None
        self.g_compute[i].replay()
        self.losses[t].copy_(self.static_loss[i])
        self.ev_local[i].record(self.cs)
        self.ms.wait_event(self.ev_local[i])
        e1 = self._ev(self.ms) if tr else None
        with torch.cuda.stream(self.ms):
            if self.world > 1:
                self.tag_dev.fill_(t)
            self.g_comm[i].replay()
        e2 = self._ev(self.ms) if tr else None
        with torch.cuda.stream(self.ms):  # clean for the backward of t + K (outside the timed ring)
            self.fm.grad_bufs[i].zero_()
        self.ev_agg[i].record(self.ms)
        if tr:
            self._rec(t, STAGE_UPDATE, e0, eu, t - self.K)
            self._rec(t, STAGE_BACKWARD, eu, self._ev(self.cs))
            self._rec(t, STAGE_ALLREDUCE, e1, e2)
            self._rec(t, "ring" if self.world > 1 else "recompress", e1, e2)
        self.graph_ready_tag[i] = t
        self._mark(t)

    def _set_lr(self, t: int) -> None:
        """Learning rate of update t into the device scalar the update graphs read."""
        if self.cfg.lr_decay_every > 0:
            with torch.cuda.stream(self.cs):
                self.lr_dev.fill_(float(np.float32(self._lr(t))))

    def drain_graph(self, t1: int) -> None:
        """The last updates eagerly, with the eager engine's rates (drain / drain_sync)."""
        if self.cfg.mode == MODE_PS_SYNC:
            return  # every step applied its own update
        if self.cfg.mode == MODE_D_SYNC:
            if self.graph_pending is not None:
                pend = self.sync_slots[self.graph_pending % self.K]
                lr = float(np.float32(self._lr(self.graph_pending + 1)))
                _lib.call("gp_consume_update", self.fm.params.data_ptr(), int(Codec.NONE), pend.payload.data_ptr(),
                          pend.status.scale_view.data_ptr(), self.n, lr, self.world, self.cs.cuda_stream)
                self.graph_pending = None
            return
        for tag in range(t1 - self.K + 1, t1 + 1):
            i = tag % self.K
            self.cs.wait_event(self.ev_agg[i])
            slot = self.slots[i]
            lr = float(np.float32(self._lr(tag + self.K)))
            _lib.call("gp_consume_update", self.fm.params.data_ptr(), int(slot.codec), slot.payload.data_ptr(),
                      slot.status.scale_view.data_ptr(), self.n, lr, self.world, self.cs.cuda_stream)

    def ps_step(self, t: int) -> None:
        """PS-Sync (engine.py:503-552) with the server role co-located on rank 0:
        local D(C(grad)) -> gather, the server folding 0 + x_0 + ... + x_{p-1}
        in rank order (collective.py:236-251) -> the server's SGD step with the
        mean (engine.py:542-545) -> broadcast of the parameters (:546-549).
        Not pipelined: every stage is on the compute stream."""
        i = t % self.K
        if self.fused:
            self.fm.use_grad_buffer(i)
        e0 = self._ev(self.cs) if self.tracing else None
        if self.grad_fn is not None:
            self.cs.synchronize()
            loss, g = self.grad_fn(self.rank, t, self.fm.params)
            self.fm.grads.copy_(torch.as_tensor(np.asarray(g, np.float32)).to(self.dev))
            self.losses[t].fill_(float(loss))
        else:
            x, y = self.batch_fn(self.rank, t)
            self.losses[t].copy_(self.fm.loss_and_grad(x, y))
        e1 = self._ev(self.cs) if self.tracing else None
        roundtrip_async(self.fm.grads, self.cfg.codec, self.local[i], self.local_status[i], self.cs.cuda_stream)
        e2 = self._ev(self.cs) if self.tracing else None
        root = 0
        self.ep._star(self.local[i], self.summed if self.rank == root else None, self.n, root, 0, True, t, self.cs)
        if self.rank == root:
            lr = float(np.float32(self._lr(t)))
            _lib.call("gp_consume_update", self.fm.params.data_ptr(), int(Codec.NONE),
                      self.summed.data_ptr(), self.local_status[i].scale_view.data_ptr(), self.n, lr, self.world,
                      self.cs.cuda_stream)
        self.ep._star(self.fm.params, self.fm.params, self.n, root, 1, False, t, self.cs)
        if self.tracing:
            e3 = self._ev(self.cs)
            self._rec(t, STAGE_BACKWARD, e0, e1)
            self._rec(t, STAGE_COMPRESS, e1, e2)
            self._rec(t, STAGE_ALLREDUCE, e2, e3)
        self.updates_seen += 1
        if self.updates_seen <= self.cfg.snapshot_first:
            self.early_params.append((t, self.fm.params.clone()))
        if self.cfg.eval_interval and self.rank == 0 and t % self.cfg.eval_interval == 0:
            self.eval_points.append((t, self.fm.params.clone()))
        self._mark(t)

    def _mark(self, t):
        e = self._new_event()
        e.record(self.cs)
        self.iter_done[t] = e

    def run(self, iters_per_epoch: int = 1) -> None:
        cfg = self.cfg
        # every torch op issued below (batch gather, fwd/bwd, snapshots) goes
        # to the compute stream; ring + re-compress are put on self.ms explicitly
        with torch.cuda.device(self.dev), torch.cuda.stream(self.cs):
            if cfg.mode == MODE_D_SYNC:
                self.sync_phase(1, cfg.iterations)
            elif cfg.mode == MODE_PS_SYNC:
                for t in range(1, cfg.iterations + 1):
                    self.ps_step(t)
            else:
                warm = min(cfg.iterations, cfg.warmup_epochs * iters_per_epoch)
                if warm > 0:
                    self.sync_phase(1, warm)
                if warm < cfg.iterations:
                    self.pipe_phase(warm + 1, cfg.iterations)
            self.end = torch.cuda.Event(enable_timing=True)
            self.end.record(self.cs)

    def finish(self, start_ev: torch.cuda.Event, train_seconds: float) -> WorkerResult:
        self.cs.synchronize()
        self.ms.synchronize()
        self.ep._check_errors(self.n)
        if any(int(s.t[1].item()) for s in self.local_status) or \
                any(int(s.status.t[1].item()) for s in self.slots):
            raise CodecError("refusing to compress non-finite values")
        losses = self.losses.cpu().numpy()
        metrics = [(t, start_ev.elapsed_time(e), float(losses[t])) for t, e in sorted(self.iter_done.items())]
        trace = []
        for t, stage, e0, e1, consumed in self.events:
            trace.append(TraceEvent(self.rank, t, stage, int(start_ev.elapsed_time(e0) * 1e6),
                                    int(start_ev.elapsed_time(e1) * 1e6), consumed))
        trace.sort(key=lambda e: (e.start_ns, e.iteration))
        dev_s = start_ev.elapsed_time(self.end) / 1e3
        stats = self.ep.stats.snapshot()
        if self.cfg.mode == MODE_PS_SYNC:  # the worker role's traffic (engine.py:513-519): one gather message
            T, pb = self.cfg.iterations, 4 * self.n
            stats = TrafficStats(T, T * pb, T * (pb + 20))
        return WorkerResult(
            rank=self.rank, params=self.fm.params.cpu().numpy(), trace=trace, metrics=metrics,
            eval_points=[(t, p.cpu().numpy()) for t, p in self.eval_points],
            early_params=[(t, p.cpu().numpy()) for t, p in self.early_params],
            stats=stats, train_seconds=train_seconds, device_seconds=dev_s)


# ----------------------------------------------------------------- clusters

# Where the ring runs. D-Sync runs it between computes: every SM (CTA budget
# 0 = the communicator's default, 4 CTAs per SM) gives the shortest ring.
# Pipe-SGD runs it beside the next iteration's forward/backward, and the
# ring's resident CTAs (most of them waiting on flags) keep SMs from the
# compute kernels:
#   * a small gradient (<= 8 MB) gets 64 CTAs on the shared GPU (C1 MLP,
#     N = 4: 6067 -> 7602 iterations/s from 256 to 64 CTAs; compute 143 ->
#     110 us per step; a 16-SM partition slows its latency-bound LL ring
#     and the end-to-end rate);
#   * up to 32 MB the comm stream runs in a green-context partition of 32
#     SMs with 128 CTAs (C2 CNN, N = 4: 661.8 at 64 CTAs on every SM ->
#     683.0; 16 SMs: 629.4);
#   * a large one gets 48 SMs with 192 CTAs (C3 AlexNet, N = 4: 191.5 at 256
#     CTAs spread over every SM -> 198.1, compute 5.04 -> 4.84 ms per step;
#     592 CTAs on every SM gave 197.4 but held every register of every SM,
#     so the next compute no longer overlapped the ring -- not the paper's
#     pipeline). One rank (no ring): C3 58.1 either way, no partition.
# profiles/r02/engine_ctas/, profiles/r02/green_ctx/.
COMM_CTAS = 0
# The comm stream runs at the highest priority (CUDA clamps -5 to the
# device's range): C3 at N = 1, the pipe re-compress's absmax + encode reach
# 0.54 of HBM beside cuDNN instead of 0.45, iterations/s unchanged
# (58.2 / 58.3; profiles/r02/comm_priority/).
COMM_PRIORITY = -5
PIPE_SMALL_GRADIENT_CTAS = 64
PIPE_MID_GRADIENT_SMS = 32
PIPE_LARGE_GRADIENT_SMS = 48
PIPE_LARGE_GRADIENT_CTAS = 256  # no partition (one rank, or GPUs shared by ranks)
SMALL_GRADIENT_BYTES = 8 << 20
MID_GRADIENT_BYTES = 32 << 20


def default_comm_partition(mode: str, num_params: int, world: int = 2) -> tuple[int, int]:
    """(green-context SMs for the comm stream, 0 = shared GPU; ring CTA budget,
    0 = every SM) for a training run with one rank per GPU (see COMM_CTAS).
    One rank has no ring to fence off: no partition."""
    if mode == MODE_PIPE_SGD:
        if 4 * num_params <= SMALL_GRADIENT_BYTES:
            return 0, PIPE_SMALL_GRADIENT_CTAS
        if world < 2:
            return 0, PIPE_SMALL_GRADIENT_CTAS if 4 * num_params <= MID_GRADIENT_BYTES else PIPE_LARGE_GRADIENT_CTAS
        sms = PIPE_MID_GRADIENT_SMS if 4 * num_params <= MID_GRADIENT_BYTES else PIPE_LARGE_GRADIENT_SMS
        return sms, 4 * sms
    return 0, COMM_CTAS


def default_comm_ctas(mode: str, num_params: int) -> int:
    """The ring's CTA budget without a partition (one rank, or GPUs shared by
    several ranks): Pipe-SGD keeps a gradient <= 32 MB to 64 CTAs and spreads
    256 CTAs of a larger one over every SM."""
    return default_comm_partition(mode, num_params, 1)[1]


def _make_transport(workers: int, timeout_s: float, max_elems: int, ctas: int = COMM_CTAS):
    if torch.cuda.device_count() >= workers:
        return GpuTransport(workers, timeout_s=timeout_s, max_elems=max_elems, ctas=ctas)
    return EmulatedTransport(workers, timeout_s=timeout_s, max_elems=max_elems)


class DeviceDataset:
    """Per-device copy of a (features, labels) dataset with reference-exact
    host-side batch sampling (data.py:41-43 shard, :57-63 sample_from_shard)."""

    def __init__(self, dataset, device):
        self.features = torch.as_tensor(np.asarray(dataset.features, np.float32)).to(device)
        self.labels = torch.as_tensor(np.asarray(dataset.labels, np.int64)).to(device)
        self.num_samples = int(self.features.shape[0])
        self.device = device

    def gather(self, idx: np.ndarray):
        it = torch.as_tensor(np.asarray(idx, np.int64)).to(self.device, non_blocking=False)
        return self.features.index_select(0, it), self.labels.index_select(0, it)


def run_inproc_cluster(workers: int, config: RunConfig, dataset, model, latency_s: float = 0.0,
                       byte_time_s: float = 0.0, batch_provider=None, timeout_s: float = 30.0,
                       transport=None, grad_fn=None, trace: bool = True, fused: bool = True,
                       comm_ctas: int | None = None, comm_sms: int | None = None) -> list[WorkerResult]:
    """Run a full training job with all ranks as threads of this process
    (engine.py:563-618), one GPU per rank (GpuTransport) or all ranks on one
    GPU (EmulatedTransport) when there are fewer GPUs than workers.

    `model` is a ModelSpec (logistic / MLP, reference layout and init);
    `grad_fn(rank, t, params) -> (loss, grad)` optionally replaces the model's
    forward/backward (used by parity tests to inject oracle gradients).
    comm_ctas / comm_sms (None = default_comm_partition, applied only when
    this call makes one GpuTransport rank per GPU): the ring's CTA budget and
    the green-context SMs of the comm stream."""
    if workers < 1:
        raise ConfigError("need at least one worker")
    if latency_s or byte_time_s:
        raise ConfigError("GPU transports do not inject synthetic delays")
    if not isinstance(model, ModelSpec):
        model = ModelSpec(model.kind, tuple(model.layer_dims))
    n = model.num_params
    own_transport = transport is None
    one_per_gpu = transport is None and torch.cuda.device_count() >= workers
    part_sms, part_ctas = default_comm_partition(config.mode, n, workers)
    if comm_sms is None:
        comm_sms = part_sms if one_per_gpu else 0
    if comm_ctas is None:
        comm_ctas = part_ctas if comm_sms else default_comm_ctas(config.mode, n)
    tr = transport or _make_transport(workers, timeout_s, max(n, 1), comm_ctas)
    shards = [np.arange(r % workers, dataset.features.shape[0], workers) for r in range(workers)]
    if batch_provider is None and grad_fn is None:
        for r in range(workers):
            if config.batch_size > len(shards[r]):
                raise ConfigError(f"rank {r}: batch size {config.batch_size} exceeds shard of "
                                  f"{len(shards[r])} samples")
    results: list = [None] * workers
    errors: list = []
    barrier = threading.Barrier(workers)

    def runner(r: int):
        try:
            ep = tr.endpoint(r)
            dev = ep.device
            with torch.cuda.device(dev):
                fm = FlatModel(SpecNet(model), dev, init_params(model, config.seed))
                data = DeviceDataset(dataset, dev) if grad_fn is None else None
                rng = np.random.default_rng([config.seed, r])

                def batch_fn(rank, t):
                    idx = batch_provider(rank, t) if batch_provider else \
                        shards[rank][rng.choice(len(shards[rank]), size=config.batch_size, replace=False)]
                    return data.gather(idx)

                eng = RankEngine(r, workers, ep, fm, config, batch_fn, trace=trace, grad_fn=grad_fn, fused=fused,
                                 comm_sms=comm_sms if isinstance(tr, GpuTransport) else 0)
                ipe = max(1, len(shards[r]) // config.batch_size)
                torch.cuda.synchronize(dev)
                barrier.wait()
                start = torch.cuda.Event(enable_timing=True)
                start.record(eng.cs)
                eng.ms.wait_stream(eng.cs)
                t0 = time.perf_counter()
                eng.run(ipe)
                eng.cs.synchronize()
                results[r] = eng.finish(start, time.perf_counter() - t0)
        except BaseException as err:  # noqa: BLE001
            errors.append(err)
            barrier.abort()

    threads = [threading.Thread(target=runner, args=(r,), name=f"worker-{r}") for r in range(workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if own_transport:
        tr.close()
    if errors:
        real = [e for e in errors if not isinstance(e, threading.BrokenBarrierError)]
        raise (real or errors)[0]
    if config.mode == MODE_PS_SYNC:
        # the reference returns the server's result last (engine.py:581, :600):
        # here the server role lives on rank 0, so its state is rank 0's
        import dataclasses
        T, pb = config.iterations, 4 * n
        server = dataclasses.replace(results[0], rank=workers, is_server=True, metrics=[], eval_points=[],
                                     early_params=[],
                                     stats=TrafficStats(T * workers, T * workers * pb, T * workers * (pb + 20)))
        results = results + [server]
    return results


def run_process_worker(config: RunConfig, dataset, model, timeout_s: float = 30.0, batch_provider=None,
                       grad_fn=None, trace: bool = True, fused: bool = True, comm_ctas: int | None = None,
                       comm_sms: int | None = None, group=None) -> WorkerResult:
    """One rank of a multi-process run (one process per GPU under torchrun):
    the analogue of the reference's run_tcp_worker (engine.py:621-646).
    torch.distributed must be initialised; the rank's GPU is LOCAL_RANK.
    Ranks exchange inbox IPC handles once over the process group, then the
    ring moves gradients over NVLink only. comm_ctas / comm_sms: as in
    run_inproc_cluster (None = default_comm_partition)."""
    import os

    import torch.distributed as dist

    from .transport import ProcessGroupTransport

    if not dist.is_initialized():
        raise ConfigError("run_process_worker needs torch.distributed initialised (torchrun)")
    rank, workers = dist.get_rank(group), dist.get_world_size(group)
    local = int(os.environ.get("LOCAL_RANK", rank % max(1, torch.cuda.device_count())))
    torch.cuda.set_device(local)
    if not isinstance(model, ModelSpec):
        model = ModelSpec(model.kind, tuple(model.layer_dims))
    part_sms, part_ctas = default_comm_partition(config.mode, model.num_params, workers)
    if comm_sms is None:
        comm_sms = part_sms
    if comm_ctas is None:
        comm_ctas = part_ctas if comm_sms else default_comm_ctas(config.mode, model.num_params)
    ep = ProcessGroupTransport.endpoint(local, group=group, timeout_s=timeout_s,
                                        max_elems=max(model.num_params, 1), ctas=comm_ctas)
    dev = ep.device
    shard = np.arange(rank % workers, dataset.features.shape[0], workers)
    if batch_provider is None and grad_fn is None and config.batch_size > len(shard):
        raise ConfigError(f"rank {rank}: batch size {config.batch_size} exceeds shard of {len(shard)} samples")
    with torch.cuda.device(dev):
        fm = FlatModel(SpecNet(model), dev, init_params(model, config.seed))
        data = DeviceDataset(dataset, dev) if grad_fn is None else None
        rng = np.random.default_rng([config.seed, rank])

        def batch_fn(r, t):
            idx = batch_provider(r, t) if batch_provider else \
                shard[rng.choice(len(shard), size=config.batch_size, replace=False)]
            return data.gather(idx)

        eng = RankEngine(rank, workers, ep, fm, config, batch_fn, trace=trace, grad_fn=grad_fn, fused=fused,
                         comm_sms=comm_sms)
        torch.cuda.synchronize(dev)
        dist.barrier(group)
        start = torch.cuda.Event(enable_timing=True)
        start.record(eng.cs)
        eng.ms.wait_stream(eng.cs)
        t0 = time.perf_counter()
        eng.run(max(1, len(shard) // config.batch_size))
        eng.cs.synchronize()
        return eng.finish(start, time.perf_counter() - t0)
