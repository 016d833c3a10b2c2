"""GPU transports: NVLink/NVSwitch peer memory instead of queues and sockets.

Drop-in for the endpoint side of /root/reference/pkg/src/gradpipe/transport.py.
The reference moves serialized blocks through per-pair FIFO channels
(`InProcTransport`, :150-177; `TcpEndpoint`, :192-305) and counts outgoing
traffic per endpoint (`TrafficStats`, :52-61, :85-91). Here the fused ring
kernel writes straight into the successor's inbox over NVLink, so `send` /
`recv` do not exist; what remains is the endpoint bookkeeping the callers
use — `rank`, `world_size`, `timeout_s`, `latency_s`, `byte_time_s`,
`stats`, `reset_stats()`, `close()` — with identical accounting (data
messages, codec payload bytes without the 9-byte header, frame bytes with
the 11-byte frame header).

Three ways to build endpoints:
  * GpuTransport(world_size)            one process, rank r on cuda:r, peer
                                        access between all pairs (mirrors
                                        InProcTransport: p threads, one per rank);
                                        devices=[0, 0, ...] puts several ranks on
                                        one GPU, each still with its own inbox and
                                        its own ring launch (SMs split between them)
  * EmulatedTransport(world_size)       p ranks on ONE GPU: the ranks' calls
                                        rendezvous and one cooperative launch
                                        runs the whole ring (parity at p > #GPUs)
  * ProcessGroupTransport.endpoint()    one process per GPU under torchrun;
                                        inboxes shared through CUDA IPC handles
                                        exchanged over torch.distributed
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import torch

from . import _lib
from .errors import CodecError, CollectiveError, ConfigError

DEFAULT_TIMEOUT_S = 30.0
DEFAULT_MAX_ELEMS = 1 << 26  # 256 MiB of fp32 per allreduce; inbox ~ 2x that per rank


@dataclass
class TrafficStats:
    """Outgoing-traffic counters for one endpoint (data messages only)."""

    messages: int = 0
    payload_bytes: int = 0
    frame_bytes: int = 0

    def snapshot(self) -> "TrafficStats":
        return TrafficStats(self.messages, self.payload_bytes, self.frame_bytes)


_PHASE = {0: "reduce-scatter", 1: "allgather", 2: "reduce-scatter barrier"}


def _comm_create(rank: int, world: int, device: int, max_elems: int) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _lib.call("gp_comm_create", rank, world, device, max_elems, ctypes.byref(h))
    return h


class GpuEndpoint:
    """One rank's view of the GPU ring (the reference's Endpoint surface)."""

    def __init__(self, rank: int, world_size: int, device: torch.device, comm, timeout_s: float,
                 vrank_of=None, transport=None):
        if not 0 <= rank < world_size:
            raise ConfigError(f"rank {rank} outside [0, {world_size})")
        self.rank = rank
        self.world_size = world_size
        self.device = device
        self.timeout_s = timeout_s
        self.latency_s = 0.0       # no injected delay: the link is real
        self.byte_time_s = 0.0
        self._comm = comm
        self._transport = transport
        self._stats_base = TrafficStats()
        self._poisoned: str | None = None
        self._stream: torch.cuda.Stream | None = None
        self.closed = False

    # -- reference Endpoint surface -------------------------------------
    @property
    def stats(self) -> TrafficStats:
        raw = self._raw_stats()
        b = self._stats_base
        return TrafficStats(raw.messages - b.messages, raw.payload_bytes - b.payload_bytes,
                            raw.frame_bytes - b.frame_bytes)

    def reset_stats(self) -> None:
        self._stats_base = self._raw_stats()

    def close(self) -> None:
        self.closed = True

    def send(self, *a, **k):  # pragma: no cover - documented absence
        raise CollectiveError("GPU endpoints have no point-to-point send; the ring kernel moves the data")

    recv = send

    def info(self) -> dict:
        """Communicator facts: CTAs per rank, inbox bytes, calls issued."""
        o = (ctypes.c_int64 * 8)()
        _lib.call("gp_comm_info", self._comm, o)
        keys = ("rank", "world", "device", "max_elems", "ctas", "inbox_bytes", "seq", "mode")
        return dict(zip(keys, [int(v) for v in o]))

    @property
    def stream(self) -> torch.cuda.Stream:
        """The rank's own stream for the blocking entry points: ranks that share
        a GPU must not queue their ring launches behind each other on one
        stream (each waits for the others' flags)."""
        if self._stream is None:
            self._stream = torch.cuda.Stream(self.device)
        return self._stream

    # -- internals --------------------------------------------------------
    def _raw_stats(self) -> TrafficStats:
        s = _lib.GpStats()
        _lib.call("gp_get_stats", self._comm, self.rank, ctypes.byref(s))
        return TrafficStats(int(s.messages), int(s.payload_bytes), int(s.frame_bytes))

    def _launch(self, x: torch.Tensor, out: torch.Tensor | None, codec: int, iteration: int,
                stream: torch.cuda.Stream, flags: int = 0, slot: torch.Tensor | None = None,
                slot_scale: torch.Tensor | None = None) -> None:
        if self._poisoned:
            raise CollectiveError(f"endpoint {self.rank} is unusable after an earlier failure: {self._poisoned}")
        _lib.call("gp_allreduce_ex", self._comm, x.data_ptr(), _ptr(out), _ptr(slot), _ptr(slot_scale),
                  x.numel(), int(codec), int(flags), int(iteration) & 0xFFFFFFFF, stream.cuda_stream)

    def _star(self, x: torch.Tensor, out: torch.Tensor | None, n: int, root: int, mode: int, zero_first: bool,
              iteration: int, stream: torch.cuda.Stream) -> None:
        """Star collective (mode 0 gather-sum to root, 1 broadcast from root)."""
        if self._poisoned:
            raise CollectiveError(f"endpoint {self.rank} is unusable after an earlier failure: {self._poisoned}")
        if mode == 0:
            _lib.call("gp_gather_sum", self._comm, x.data_ptr(), _ptr(out), n, int(root), int(zero_first),
                      int(iteration) & 0xFFFFFFFF, stream.cuda_stream)
        else:
            _lib.call("gp_broadcast", self._comm, x.data_ptr(), _ptr(out), n, int(root),
                      int(iteration) & 0xFFFFFFFF, stream.cuda_stream)

    def _check_errors(self, n: int) -> None:
        """After the launching stream completed: raise what the device latched."""
        e = _lib.GpError()
        _lib.call("gp_comm_poll_error", self._comm, ctypes.byref(e))
        if e.kind:
            raise self._poison(raise_for(e, self.world_size, n, self.timeout_s))

    def _poison(self, err: Exception) -> Exception:
        if isinstance(err, CollectiveError):
            self._poisoned = str(err)
        return err


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def raise_for(e, p: int, n: int, timeout_s: float) -> Exception:
    """Map a device error word to the reference's exception and message shape
    (collective.py:52-64, :106, :157-161; compression.py:108-109)."""
    if e.kind == _lib.GP_FAIL_NONFINITE:
        return CodecError("refusing to compress non-finite values")
    phase = _PHASE.get(e.phase, "ring")
    pred = (e.rank - 1) % p
    if e.kind == _lib.GP_FAIL_TIMEOUT:
        why = "aborted after a peer failed" if e.detail == 1 else f"timed out after {timeout_s:g}s"
        return CollectiveError(f"{phase} step {e.step} (rank {e.rank} <- {pred}): {why}"
                               + (f" waiting for block {e.block}" if e.block >= 0 else ""))
    if e.kind == _lib.GP_FAIL_HEADER:
        from .collective import partition_blocks
        want = partition_blocks(n, p)[e.block][1] if 0 <= e.block < p else -1
        return CollectiveError(f"{phase} step {e.step}: block {e.block} has {e.detail} elems, expected "
                               f"{want} or a different iteration tag (unequal vector lengths across ranks?)")
    if e.kind == _lib.GP_FAIL_BOUNDS:
        return CollectiveError(f"bounds-checked build: rank {e.rank} accessed outside its buffers "
                               f"(address low bits {e.detail & 0xFFFFFFFF:#010x})")
    return CollectiveError(f"{phase} step {e.step}: device error kind {e.kind}")


def _set_protocol(comm, ll_max_bytes: int | None) -> None:
    """ll_max_bytes (every rank the same): LL protocol only for blocks whose
    payload fits it, 0 = flag protocol always; None = the library default
    (LL up to 2 MiB blocks). Results are bit-identical either way."""
    if ll_max_bytes is not None:
        if ll_max_bytes < 0:
            raise ConfigError("ll_max_bytes must be >= 0")
        _lib.call("gp_comm_set_protocol", comm, int(ll_max_bytes))


class GpuTransport:
    """In-process ring over p GPUs (rank r on devices[r]); threads play ranks,
    exactly like the reference's InProcTransport (transport.py:150-177).

    Ranks may share a GPU (devices with repeats): every rank still launches
    its own ring kernel on its own stream and reaches the others' inboxes
    through plain device pointers, so the per-rank launch path (flag / LL
    protocols, graph replay, sequence wrap) runs on a one-GPU box too; the
    device's SMs are split so that all ranks' launches co-reside."""

    def __init__(self, world_size: int, latency_s: float = 0.0, byte_time_s: float = 0.0,
                 timeout_s: float = DEFAULT_TIMEOUT_S, devices=None, max_elems: int = DEFAULT_MAX_ELEMS,
                 ctas: int = 0, ll_max_bytes: int | None = None):
        if world_size < 1:
            raise ConfigError("need at least one rank")
        if latency_s or byte_time_s:
            raise ConfigError("GPU transports do not inject synthetic delays (latency_s/byte_time_s)")
        devices = list(range(world_size)) if devices is None else list(devices)
        if len(devices) != world_size:
            raise ConfigError("need one device per rank")
        if torch.cuda.device_count() < max(devices) + 1:
            raise ConfigError(f"{world_size} ranks need {max(devices) + 1} GPUs, "
                              f"found {torch.cuda.device_count()}")
        self.world_size = world_size
        self.timeout_s = timeout_s
        self.max_elems = max_elems
        self._comms = [_comm_create(r, world_size, devices[r], max_elems) for r in range(world_size)]
        for c in self._comms:
            _lib.call("gp_comm_set_tuning", c, int(ctas), float(timeout_s))
            _set_protocol(c, ll_max_bytes)
        # chunk size, and so every flag index, follows the CTA budget G: all
        # ranks must agree even when their devices' caps differ
        g = min(ep_ctas(c) for c in self._comms)
        for c in self._comms:
            if ep_ctas(c) != g:
                _lib.call("gp_comm_set_tuning", c, int(g), 0.0)
        if len({ep_ctas(c) for c in self._comms}) != 1:
            raise ConfigError("ranks disagree on the ring's CTA budget")
        if world_size > 1:
            arr = (ctypes.c_void_p * world_size)(*[c.value for c in self._comms])
            _lib.call("gp_comm_connect_local", arr, world_size)
        self._eps = [GpuEndpoint(r, world_size, torch.device("cuda", devices[r]), self._comms[r],
                                 timeout_s, transport=self) for r in range(world_size)]

    def endpoint(self, rank: int) -> GpuEndpoint:
        return self._eps[rank]

    def close(self) -> None:
        for c in self._comms:
            _lib.load().gp_comm_destroy(c)
        self._comms = []


class _Generation:
    def __init__(self):
        self.slots: dict[int, tuple] = {}
        self.done: torch.cuda.Event | None = None
        self.n = 0
        self.error: Exception | None = None
        self.polled = False
        self.launched = False


class EmulatedEndpoint(GpuEndpoint):
    """Endpoint of an EmulatedTransport: its calls rendezvous with the other
    virtual ranks; the last arrival launches the ring for everyone."""

    def _launch(self, x, out, codec, iteration, stream, flags=0, slot=None, slot_scale=None):
        self._gen = self._transport._arrive(self.rank, x, out, codec, iteration, stream, flags, slot, slot_scale)

    def _star(self, x, out, n, root, mode, zero_first, iteration, stream):
        self._gen = self._transport._arrive(self.rank, x, out, -1 - mode, iteration, stream,
                                            (int(root) << 1) | int(bool(zero_first)), None, None, n=n)

    def _check_errors(self, n: int) -> None:
        self._transport._finish(getattr(self, "_gen", None))


class EmulatedTransport:
    """p ranks of the ring on one GPU, one cooperative launch per allreduce.

    Ranks call from p threads exactly like InProcTransport endpoints. Every
    call is stream-ordered: the launch waits on each rank's stream (event) and
    each rank's stream waits on the launch, so callers never block on the GPU
    unless they ask to (ring_allreduce does). Used for parity at p = 3/4/8 on
    a single B200 without separately launched kernels that wait on each other."""

    def __init__(self, world_size: int, latency_s: float = 0.0, byte_time_s: float = 0.0,
                 timeout_s: float = DEFAULT_TIMEOUT_S, device: int = 0,
                 max_elems: int = DEFAULT_MAX_ELEMS // 4, ctas: int = 0, ll_max_bytes: int | None = None):
        if latency_s or byte_time_s:
            raise ConfigError("GPU transports do not inject synthetic delays")
        self.world_size = world_size
        self.timeout_s = timeout_s
        self.device = torch.device("cuda", device)
        h = ctypes.c_void_p()
        _lib.call("gp_comm_create_emulated", world_size, device, max_elems, ctypes.byref(h))
        self._comm = h
        _lib.call("gp_comm_set_tuning", h, int(ctas), float(timeout_s))
        _set_protocol(h, ll_max_bytes)
        self._cv = threading.Condition()
        self._cur = _Generation()
        self._poll_lock = threading.Lock()
        self._eps = [EmulatedEndpoint(r, world_size, self.device, h, timeout_s, transport=self)
                     for r in range(world_size)]
        self._stream = torch.cuda.Stream(self.device)

    def endpoint(self, rank: int) -> EmulatedEndpoint:
        return self._eps[rank]

    def _arrive(self, rank, x, out, codec, iteration, stream, flags=0, slot=None, slot_scale=None,
                n=None) -> _Generation:
        """codec >= 0: ring allreduce; -1: gather-sum, -2: broadcast (flags =
        root << 1 | zero_first)."""
        ev = torch.cuda.Event()
        ev.record(stream)
        with self._cv:
            gen = self._cur
            if rank in gen.slots:
                raise CollectiveError(f"rank {rank} entered the same collective twice")
            gen.slots[rank] = (x, out, int(codec), int(iteration), x.numel() if n is None else int(n), ev,
                               int(flags), slot, slot_scale)
            if len(gen.slots) == self.world_size:
                self._launch_all(gen)
                self._cur = _Generation()
                self._cv.notify_all()
            else:
                ok = self._cv.wait_for(lambda: gen.launched, timeout=self.timeout_s)
                if not ok:
                    gen.slots.pop(rank, None)
                    raise CollectiveError(f"reduce-scatter step 0 (rank {rank} <- {(rank - 1) % self.world_size}): "
                                          f"timed out after {self.timeout_s:g}s")
        if gen.error is None and gen.done is not None:
            stream.wait_event(gen.done)
        return gen

    def _launch_all(self, gen: _Generation):
        p = self.world_size
        args = [gen.slots[r] for r in range(p)]
        gen.launched = True
        if len({a[4] for a in args}) != 1 or len({a[2] for a in args}) != 1 or len({a[3] for a in args}) != 1 \
                or len({a[6] for a in args}) != 1:
            gen.error = CollectiveError("reduce-scatter step 0: ranks disagree on vector length, codec or "
                                        "iteration (unequal vector lengths across ranks?)")
            return
        gen.n = args[0][4]
        ins = (ctypes.c_void_p * p)(*[a[0].data_ptr() for a in args])
        outs = (ctypes.c_void_p * p)(*[_ptr(a[1]) for a in args])
        slots = (ctypes.c_void_p * p)(*[_ptr(a[7]) for a in args])
        scales = (ctypes.c_void_p * p)(*[_ptr(a[8]) for a in args])
        for a in args:
            self._stream.wait_event(a[5])
            for t in (a[0], a[1], a[7], a[8]):
                if t is not None:
                    t.record_stream(self._stream)
        op, fl, it = args[0][2], args[0][6], args[0][3] & 0xFFFFFFFF
        if op >= 0:
            _lib.call("gp_allreduce_emulated_ex", self._comm, ins, outs, slots, scales, gen.n, op, fl, it,
                      self._stream.cuda_stream)
        elif op == -1:
            _lib.call("gp_gather_sum_emulated", self._comm, ins, outs, gen.n, fl >> 1, fl & 1, it,
                      self._stream.cuda_stream)
        else:
            _lib.call("gp_broadcast_emulated", self._comm, ins, outs, gen.n, fl >> 1, it, self._stream.cuda_stream)
        gen.done = torch.cuda.Event()
        gen.done.record(self._stream)
        gen.slots = {}

    def _finish(self, gen: _Generation | None):
        if gen is None:
            return
        if gen.error is None and not gen.polled:
            gen.done.synchronize()
            with self._poll_lock:
                if not gen.polled:
                    e = _lib.GpError()
                    _lib.call("gp_comm_poll_error", self._comm, ctypes.byref(e))
                    if e.kind:
                        gen.error = raise_for(e, self.world_size, gen.n, self.timeout_s)
                    gen.polled = True
        if gen.error is not None:
            raise gen.error

    def close(self) -> None:
        if self._comm:
            torch.cuda.synchronize(self.device)
            _lib.load().gp_comm_destroy(self._comm)
            self._comm = None


def exchange_handles(handle: bytes, max_elems: int, device: int, group=None, ctas: int = 0) -> bytes:
    """All-gather every rank's 64-byte inbox IPC handle over the process
    group (any backend) and validate that the communicator geometry agrees;
    returns the rank-ordered handle blob gp_comm_connect_ipc expects."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gathered = [None] * world
    dist.all_gather_object(gathered, (bytes(handle), int(max_elems), int(device), _host_id(), int(ctas)),
                           group=group)
    if len({g[1] for g in gathered}) != 1:
        raise ConfigError("all ranks must create the transport with the same max_elems")
    if len({g[4] for g in gathered}) != 1:
        raise ConfigError("all ranks must give the ring the same CTA budget (chunking depends on it)")
    if len({g[3] for g in gathered}) != 1:
        raise ConfigError("ProcessGroupTransport spans one node only (NVLink peer memory)")
    if len({g[2] for g in gathered}) != world:
        raise ConfigError("ProcessGroupTransport needs a distinct GPU per rank")
    if any(len(g[0]) != 64 for g in gathered):
        raise ConfigError("malformed IPC handle")
    return b"".join(g[0] for g in gathered)


def ep_ctas(comm) -> int:
    o = (ctypes.c_int64 * 8)()
    _lib.call("gp_comm_info", comm, o)
    return int(o[4])


def _host_id() -> str:
    import socket
    return socket.gethostname()


class ProcessGroupTransport:
    """One rank per process (torchrun), inboxes mapped through CUDA IPC.

    The IPC handles travel over the existing torch.distributed process group
    (any backend); after that no collective of torch.distributed is used on
    the data path."""

    @staticmethod
    def endpoint(device: int | None = None, group=None, timeout_s: float = DEFAULT_TIMEOUT_S,
                 max_elems: int = DEFAULT_MAX_ELEMS, ctas: int = 0, ll_max_bytes: int | None = None) -> GpuEndpoint:
        import torch.distributed as dist

        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        comm = _comm_create(rank, world, device, max_elems)
        _lib.call("gp_comm_set_tuning", comm, int(ctas), float(timeout_s))
        _set_protocol(comm, ll_max_bytes)
        if world > 1:
            h = ctypes.create_string_buffer(64)
            _lib.call("gp_comm_ipc_handle", comm, h)
            blob = exchange_handles(h.raw, int(max_elems), int(device), group, ctas=ep_ctas(comm))
            _lib.call("gp_comm_connect_ipc", comm, blob)
            dist.barrier(group)
        return GpuEndpoint(rank, world, torch.device("cuda", device), comm, timeout_s)
