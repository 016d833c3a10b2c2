"""Ring AllReduce with fused compression over NVLink — drop-in for
gradpipe.collective's ring path.

Reference: /root/reference/pkg/src/gradpipe/collective.py
  partition_blocks      :35-49   (identical)
  ring_allreduce        :143-163 (same signature, same arithmetic, same bits)
  pipelined_allreduce   :166-212 (same result; on the GPU the chunked ring
                                  kernel always overlaps transfer with codec
                                  work, so both names run the same kernel)

Every hop's compress -> send -> recv -> decompress -> add of the reference
is one pass of the fused kernel in csrc/ring.cu. Inputs may be CUDA tensors
(result: a new CUDA tensor on the endpoint's GPU) or numpy arrays (result:
a new numpy array, like the reference). The input is never mutated.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .compression import Codec, as_codec
from .errors import CollectiveError
from .transport import GpuEndpoint


def partition_blocks(n_elems: int, p: int) -> list[tuple[int, int]]:
    """p contiguous (offset, length) blocks covering [0, n_elems); the first
    n_elems % p blocks take one extra element (collective.py:35-49)."""
    base, extra = divmod(n_elems, p)
    out, off = [], 0
    for i in range(p):
        ln = base + (1 if i < extra else 0)
        out.append((off, ln))
        off += ln
    return out


def _check_rank_args(local, rank: int, p: int, endpoint: GpuEndpoint) -> None:
    if endpoint.rank != rank or endpoint.world_size != p:
        raise CollectiveError(
            f"endpoint is rank {endpoint.rank}/{endpoint.world_size}, caller claims {rank}/{p}")
    if getattr(local, "ndim", 1) != 1:
        raise CollectiveError("collectives operate on 1-D vectors")


def _device_input(local, device: torch.device) -> torch.Tensor:
    if isinstance(local, torch.Tensor):
        t = local.detach()
        if t.device != device:
            t = t.to(device)
    else:
        t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float32)).to(device)
    if t.dtype != torch.float32:
        t = t.float()
    if not t.is_contiguous() or t.data_ptr() % 16:
        t = t.contiguous().clone()
    return t


def _rank_stream(endpoint: GpuEndpoint) -> torch.cuda.Stream:
    """The endpoint's own stream, ordered after the caller's current stream
    (which produced the inputs). Blocking calls run there so that ranks
    sharing a GPU never serialise their launches on one stream."""
    s = endpoint.stream
    s.wait_stream(torch.cuda.current_stream(endpoint.device))
    return s


def allreduce_into(x: torch.Tensor, out: torch.Tensor | None, endpoint: GpuEndpoint, codec=Codec.NONE,
                   iteration: int = 0, stream: torch.cuda.Stream | None = None, precompress: bool = False,
                   slot: torch.Tensor | None = None, slot_scale: torch.Tensor | None = None) -> None:
    """Stream-ordered, non-blocking form used by the pipelined engine:
    enqueue the fused ring on `stream` (default: current stream of the
    endpoint's device). Errors surface at `endpoint_wait`.

    precompress=True: x is the raw local gradient; the ring applies the
      engine's whole-vector D(C(x)) while loading it (engine.py:333).
    slot=...: write C(sum) (whole-vector codec, engine.py:407) into the uint8
      `slot` and its scale into `slot_scale` instead of the fp32 sum; `out`
      is then scratch (needed for quant8 at p > 1)."""
    s = stream if stream is not None else torch.cuda.current_stream(endpoint.device)
    flags = (_lib.GP_RING_PRECOMPRESS if precompress else 0) | (_lib.GP_RING_SLOT_OUT if slot is not None else 0)
    endpoint._launch(x, out, as_codec(codec), iteration, s, flags, slot, slot_scale)


def endpoint_wait(endpoint: GpuEndpoint, n: int, stream: torch.cuda.Stream | None = None) -> None:
    s = stream if stream is not None else torch.cuda.current_stream(endpoint.device)
    s.synchronize()
    endpoint._check_errors(n)


def ring_allreduce(local, rank: int, p: int, endpoint: GpuEndpoint, codec: Codec = Codec.NONE,
                   iteration: int = 0):
    """Elementwise sum of all ranks' vectors, identical on every rank."""
    _check_rank_args(local, rank, p, endpoint)
    codec = as_codec(codec)
    as_numpy = not isinstance(local, torch.Tensor)
    dev = endpoint.device
    with torch.cuda.device(dev):
        x = _device_input(local, dev)
        out = torch.empty_like(x)
        s = _rank_stream(endpoint)
        allreduce_into(x, out, endpoint, codec, iteration, s)
        endpoint_wait(endpoint, x.numel(), s)
    return out.cpu().numpy() if as_numpy else out


def pipelined_allreduce(local, rank: int, p: int, endpoint: GpuEndpoint, codec: Codec = Codec.NONE,
                        iteration: int = 0):
    """Bit-identical to ring_allreduce for every codec (collective.py:166-212).
    The fused kernel streams each ring block in chunks, so the transfer of
    chunk c overlaps the decode/add/encode of chunk c-1 by construction."""
    return ring_allreduce(local, rank, p, endpoint, codec, iteration)


# ------------------------------------------------------------------ star

def gather_to_root(local, root: int, rank: int, p: int, endpoint: GpuEndpoint, iteration: int = 0):
    """Root returns the elementwise sum local_root + x_0 + x_1 + ... in rank
    order (src != root), others return None (collective.py:215-252)."""
    _check_rank_args(local, rank, p, endpoint)
    as_numpy = not isinstance(local, torch.Tensor)
    dev = endpoint.device
    with torch.cuda.device(dev):
        x = _device_input(local, dev)
        out = torch.empty_like(x) if rank == root else None
        s = _rank_stream(endpoint)
        endpoint._star(x, out, x.numel(), root, 0, False, iteration, s)
        endpoint_wait(endpoint, x.numel(), s)
    if out is None:
        return None
    return out.cpu().numpy() if as_numpy else out


def broadcast_from_root(value, root: int, rank: int, p: int, endpoint: GpuEndpoint, iteration: int = 0):
    """Bit-exact copy of the root's vector on every rank (collective.py:255-280).
    Non-roots pass None; the length travels first as one bit-copied element."""
    if endpoint.rank != rank or endpoint.world_size != p:
        raise CollectiveError("endpoint does not match caller's rank/size")
    if rank == root and value is None:
        raise CollectiveError("broadcast root has no value")
    as_numpy = rank == root and not isinstance(value, torch.Tensor)
    dev = endpoint.device
    with torch.cuda.device(dev):
        hdr = torch.zeros(4, dtype=torch.int32, device=dev)
        if rank == root:
            x = _device_input(value, dev)
            hdr[0] = x.numel()
        s = _rank_stream(endpoint)
        got = torch.empty_like(hdr)
        endpoint._star(hdr.view(torch.float32), got.view(torch.float32), 4, root, 1, False, iteration, s)
        endpoint_wait(endpoint, 4, s)
        n = int(got[0].item())
        if rank != root:
            x = torch.empty(n, dtype=torch.float32, device=dev)
            as_numpy = not isinstance(value, torch.Tensor) if value is not None else True
        out = torch.empty_like(x)
        s = _rank_stream(endpoint)
        endpoint._star(x, out, n, root, 1, False, iteration, s)
        endpoint_wait(endpoint, n, s)
    return out.cpu().numpy() if as_numpy else out
