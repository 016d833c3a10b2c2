"""gradpipe_b200 -- the module a gradpipe maintainer adds (as gradpipe/_b200.py)
to route the reference's ring AllReduce through libpipesgd.so's C ABI.

Pure ctypes against include/pipesgd.h (no import of this repository's
Python package); torch only allocates device buffers and streams.

    import gradpipe, gradpipe_b200
    undo = gradpipe_b200.install(gradpipe)
    gradpipe.engine.run_inproc_cluster(...)   # the reference's own loop, B200 ring underneath
    undo()

install() swaps the names the reference's engine resolves at call time:
  * gradpipe.engine.InProcTransport (engine.py:49, :582) -> B200Transport:
    same constructor (world_size, latency_s, byte_time_s, timeout_s) and
    endpoint surface (rank, world_size, timeout_s, latency_s, byte_time_s,
    stats, reset_stats, close; transport.py:64-113), one communicator per
    rank (ranks round-robin over the visible GPUs);
  * gradpipe.engine.ring_allreduce / gradpipe.collective.ring_allreduce
    (engine.py:354-361, :399-406 -> collective.py:143-163) -> a wrapper that
    sends B200 endpoints to gp_allreduce and every other endpoint to the
    original function;
  * gradpipe.engine.barrier (engine.py:454, the run-start barrier;
    collective.py:283-297) -> gp_comm_barrier for B200 endpoints.
Everything else -- codecs, the pipelined loop, GradientBuffer, SGD -- stays
the reference's own numpy code, so the run's final weights must equal a
plain reference run bit for bit (tests/test_gpu_integration.py).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIPESGD_LIB") or os.path.join(HERE, "..", "paper_1811_03619_b200", "libpipesgd.so")

_vp, _u64, _i, _u32, _d = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_double


class _Error(ctypes.Structure):  # gp_error
    _fields_ = [(k, ctypes.c_int32) for k in ("kind", "phase", "step", "block", "rank", "detail")]


class _Stats(ctypes.Structure):  # gp_stats
    _fields_ = [(k, ctypes.c_uint64) for k in ("messages", "payload_bytes", "frame_bytes")]


_lib = None


def lib():
    """Bind the entry points this shim uses (signatures from include/pipesgd.h)."""
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB_PATH)
        sigs = {
            "gp_comm_create": [_i, _i, _i, _u64, ctypes.POINTER(_vp)],
            "gp_comm_connect_local": [ctypes.POINTER(_vp), _i],
            "gp_comm_set_tuning": [_vp, _i, _d],
            "gp_allreduce": [_vp, _vp, _vp, _u64, _i, _u32, _vp],
            "gp_comm_poll_error": [_vp, ctypes.POINTER(_Error)],
            "gp_comm_barrier": [_vp, _i, _vp, _vp],
            "gp_get_stats": [_vp, _i, ctypes.POINTER(_Stats)],
            "gp_comm_destroy": [_vp],
            "gp_last_error_string": [],
        }
        for name, args in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_char_p if name == "gp_last_error_string" else _i
        _lib = L
    return _lib


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: {lib().gp_last_error_string().decode()}")


class B200Endpoint:
    """One rank's endpoint (the reference's Endpoint surface, transport.py:64-113)."""

    def __init__(self, transport, rank):
        import torch
        self.rank, self.world_size = rank, transport.world_size
        self.latency_s, self.byte_time_s, self.timeout_s = 0.0, 0.0, transport.timeout_s
        self.comm, self.device = transport.comms[rank], torch.device("cuda", transport.devices[rank])
        self.stream = torch.cuda.Stream(self.device)
        self._base = (0, 0, 0)
        self._stats_cls = transport.stats_cls

    def _raw(self):
        s = _Stats()
        _check(lib().gp_get_stats(self.comm, self.rank, ctypes.byref(s)), "gp_get_stats")
        return int(s.messages), int(s.payload_bytes), int(s.frame_bytes)

    @property
    def stats(self):
        return self._stats_cls(*[a - b for a, b in zip(self._raw(), self._base)])

    def reset_stats(self):
        self._base = self._raw()

    def close(self):
        pass

    def send(self, *a, **k):
        raise NotImplementedError("the B200 ring moves the data inside gp_allreduce")

    recv = send


class B200Transport:
    """Drop-in for gradpipe.transport.InProcTransport(world_size, latency_s,
    byte_time_s, timeout_s) (transport.py:150-177)."""

    max_elems = 1 << 22  # fp32 elements per allreduce the inboxes are sized for

    def __init__(self, world_size, latency_s=0.0, byte_time_s=0.0, timeout_s=30.0):
        import torch
        from gradpipe.transport import TrafficStats
        if latency_s or byte_time_s:
            raise ValueError("B200Transport moves real bytes over NVLink: no injected delays")
        self.world_size, self.timeout_s, self.stats_cls = world_size, timeout_s, TrafficStats
        ng = torch.cuda.device_count()
        self.devices = [r % ng for r in range(world_size)]
        self.comms = []
        for r in range(world_size):
            h = _vp()
            _check(lib().gp_comm_create(r, world_size, self.devices[r], self.max_elems, ctypes.byref(h)),
                   "gp_comm_create")
            _check(lib().gp_comm_set_tuning(h, 0, float(timeout_s)), "gp_comm_set_tuning")
            self.comms.append(h)
        if world_size > 1:
            arr = (_vp * world_size)(*[c.value for c in self.comms])
            _check(lib().gp_comm_connect_local(arr, world_size), "gp_comm_connect_local")
        self._eps = [B200Endpoint(self, r) for r in range(world_size)]

    def endpoint(self, rank):
        return self._eps[rank]

    def close(self):
        for c in self.comms:
            lib().gp_comm_destroy(c)
        self.comms = []


def ring_allreduce_b200(local, rank, p, endpoint, codec, iteration=0):
    """collective.py:143-163 through gp_allreduce: numpy in, new numpy out."""
    import torch
    from gradpipe.errors import CodecError, CollectiveError
    if endpoint.rank != rank or endpoint.world_size != p:
        raise CollectiveError(f"endpoint is rank {endpoint.rank}/{endpoint.world_size}, caller claims {rank}/{p}")
    dev, s = endpoint.device, endpoint.stream
    with torch.cuda.device(dev):
        x = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float32)).to(dev)
        out = torch.empty_like(x)
        s.wait_stream(torch.cuda.current_stream(dev))
        rc = lib().gp_allreduce(endpoint.comm, x.data_ptr(), out.data_ptr(), x.numel(), int(codec),
                                int(iteration) & 0xFFFFFFFF, s.cuda_stream)
        if rc != 0:
            raise CollectiveError(lib().gp_last_error_string().decode())
        s.synchronize()
        e = _Error()
        _check(lib().gp_comm_poll_error(endpoint.comm, ctypes.byref(e)), "gp_comm_poll_error")
        if e.kind == 1:  # GP_FAIL_NONFINITE
            raise CodecError("refusing to compress non-finite values")
        if e.kind:
            raise CollectiveError(f"ring step {e.step} (rank {e.rank} <- {(e.rank - 1) % p}): device failure "
                                  f"kind {e.kind}")
        return out.cpu().numpy()


def barrier_b200(rank, p, endpoint):
    """collective.py:283-297 through gp_comm_barrier (all-to-all flag barrier
    over the GPUs): no rank returns before all have entered."""
    import torch
    from gradpipe.errors import CollectiveError
    if endpoint.rank != rank or endpoint.world_size != p:
        raise CollectiveError("endpoint does not match caller's rank/size")
    with torch.cuda.device(endpoint.device):
        ns = torch.zeros(1, dtype=torch.int64, device=endpoint.device)
        _check(lib().gp_comm_barrier(endpoint.comm, 1, ns.data_ptr(), endpoint.stream.cuda_stream), "gp_comm_barrier")
        endpoint.stream.synchronize()
        if int(ns.item()) == -1:
            raise CollectiveError(f"barrier (rank {rank}): timed out after {endpoint.timeout_s:g}s")


def install(gradpipe):
    """Route the reference engine's ring through the B200 C ABI; returns undo()."""
    import gradpipe.collective as C
    import gradpipe.engine as E
    orig_ring, orig_transport = C.ring_allreduce, E.InProcTransport

    def ring_allreduce(local, rank, p, endpoint, codec=C.Codec.NONE, iteration=0):
        if isinstance(endpoint, B200Endpoint):
            return ring_allreduce_b200(local, rank, p, endpoint, codec, iteration)
        return orig_ring(local, rank, p, endpoint, codec, iteration)

    live = []

    def transport(*a, **k):
        tr = B200Transport(*a, **k)
        live.append(tr)
        return tr

    orig_barrier = E.barrier

    def barrier(rank, p, endpoint, generation=0):
        if isinstance(endpoint, B200Endpoint):
            return barrier_b200(rank, p, endpoint)
        return orig_barrier(rank, p, endpoint, generation)

    C.ring_allreduce = E.ring_allreduce = ring_allreduce
    E.InProcTransport = transport
    E.barrier = barrier

    def undo():
        C.ring_allreduce = E.ring_allreduce = orig_ring
        E.InProcTransport = orig_transport
        E.barrier = orig_barrier
        for tr in live:
            tr.close()

    return undo
