"""Gradient codecs on the GPU — drop-in for gradpipe.compression.

Same names and meanings as /root/reference/pkg/src/gradpipe/compression.py:
`Codec` (:37-56), `CompressedBlock` (:59-72), `payload_size` (:75-79),
`wire_size` (:82-84), `compress` (:103-136), `decompress` (:141-151),
`serialize_block` / `deserialize_block` (:154-172).

Differences that follow from living on a B200:
  * vectors are CUDA float32 tensors (numpy input is copied to the current
    device; `decompress` of a block made from numpy still returns a tensor);
  * `CompressedBlock.payload` is a uint8 device tensor and the quant8 scale
    stays on the device (`scale_t`); `.scale` reads it back on demand;
  * the encode/decode math runs in libpipesgd.so (csrc/codec.cuh), bit-exact
    with the reference — there is no CPU fallback.
"""

from __future__ import annotations

import enum
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import CodecError, CorruptBlockError

HEADER = struct.Struct("<BIf")
HEADER_BYTES = HEADER.size  # 9


class Codec(enum.IntEnum):
    """Closed codec enumeration; numeric values are the wire tags."""

    NONE = 0
    TRUNC16 = 1
    QUANT8 = 2

    @classmethod
    def parse(cls, name: str) -> "Codec":
        try:
            return _CODEC_NAMES[name.strip().lower()]
        except KeyError:
            raise CodecError(f"unknown codec {name!r}") from None

    @property
    def bytes_per_elem(self) -> int:
        return _WIDTH[self]


_CODEC_NAMES = {"none": Codec.NONE, "trunc16": Codec.TRUNC16, "quant8": Codec.QUANT8}
_WIDTH = {Codec.NONE: 4, Codec.TRUNC16: 2, Codec.QUANT8: 1}


def as_codec(codec) -> Codec:
    if isinstance(codec, str):
        return Codec.parse(codec)
    try:
        return Codec(int(codec))
    except ValueError:
        raise CodecError(f"unknown codec {codec!r}") from None


@dataclass(frozen=True, eq=False)
class CompressedBlock:
    """An encoded vector resident on the GPU.

    payload: uint8 CUDA tensor of n_elems * codec.bytes_per_elem bytes
    scale_t: 1-element float32 CUDA tensor (quant8 scale; 0 otherwise)
    """

    codec: Codec
    n_elems: int
    payload: torch.Tensor
    scale_t: torch.Tensor

    def __post_init__(self) -> None:
        expected = self.n_elems * self.codec.bytes_per_elem
        if self.payload.numel() != expected:
            raise CorruptBlockError(
                f"{self.codec.name} block of {self.n_elems} elems needs "
                f"{expected} payload bytes, got {self.payload.numel()}"
            )

    @property
    def scale(self) -> float:
        return float(self.scale_t.item())

    def payload_bytes(self) -> bytes:
        return self.payload.cpu().numpy().tobytes()

    def __eq__(self, other) -> bool:
        return (isinstance(other, CompressedBlock) and self.codec == other.codec
                and self.n_elems == other.n_elems
                and np.float32(self.scale).tobytes() == np.float32(other.scale).tobytes()
                and self.payload_bytes() == other.payload_bytes())


def payload_size(codec: Codec, n_elems: int) -> int:
    """Codec payload bytes for n_elems, excluding the block header."""
    if n_elems < 0:
        raise CodecError(f"negative element count {n_elems}")
    return n_elems * as_codec(codec).bytes_per_elem


def wire_size(codec: Codec, n_elems: int) -> int:
    """Exact serialized size of a block, header included."""
    return HEADER_BYTES + payload_size(codec, n_elems)


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def to_device_vector(vec, device=None) -> torch.Tensor:
    """1-D contiguous, 16-byte aligned float32 CUDA tensor view/copy of vec."""
    if isinstance(vec, torch.Tensor):
        t = vec
        if t.device.type != "cuda":
            t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
    else:
        arr = np.ascontiguousarray(vec, dtype=np.float32)
        t = torch.from_numpy(arr).to(device or torch.device("cuda", torch.cuda.current_device()))
    if t.dim() != 1:
        raise CodecError("can only compress 1-D vectors")
    if t.dtype != torch.float32:
        t = t.float()
    if not t.is_contiguous() or t.data_ptr() % 16:
        t = t.contiguous().clone()
    return t


class CodecStatus:
    """Device-resident gp_codec_status (16 bytes) for async codec calls."""

    def __init__(self, device):
        self.t = torch.zeros(4, dtype=torch.int32, device=device)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def scale_view(self) -> torch.Tensor:
        return self.t[2:3].view(torch.float32)

    def raise_if_nonfinite(self) -> None:
        if int(self.t[1].item()) != 0:
            raise CodecError("refusing to compress non-finite values")


def encode_async(x: torch.Tensor, codec: Codec, payload: torch.Tensor, status: CodecStatus,
                 stream: int | None = None) -> None:
    """Stream-ordered encode of x into payload; scale lands in status."""
    s = _stream_ptr(x.device) if stream is None else stream
    _lib.call("gp_encode", int(as_codec(codec)), x.data_ptr(), x.numel(), payload.data_ptr(), status.ptr, s)


def compress(vec, codec: Codec) -> CompressedBlock:
    """Encode a float32 vector under the given codec (blocking, like the
    reference: a non-finite input raises CodecError)."""
    codec = as_codec(codec)
    x = to_device_vector(vec)
    n = x.numel()
    payload = torch.empty(max(n * codec.bytes_per_elem, 0), dtype=torch.uint8, device=x.device)
    status = CodecStatus(x.device)
    encode_async(x, codec, payload, status)
    torch.cuda.current_stream(x.device).synchronize()
    status.raise_if_nonfinite()
    return CompressedBlock(codec, n, payload, status.scale_view.clone())


def decompress_into(block: CompressedBlock, out: torch.Tensor, stream: int | None = None) -> torch.Tensor:
    s = _stream_ptr(out.device) if stream is None else stream
    _lib.call("gp_decode", int(block.codec), block.payload.data_ptr(), block.scale_t.data_ptr(),
              block.n_elems, out.data_ptr(), s)
    return out


def decompress(block: CompressedBlock) -> torch.Tensor:
    """Reconstruct the float32 vector a block encodes (CUDA tensor)."""
    out = torch.empty(block.n_elems, dtype=torch.float32, device=block.payload.device)
    return decompress_into(block, out)


def roundtrip_async(x: torch.Tensor, codec: Codec, out: torch.Tensor, status: CodecStatus,
                    stream: int | None = None) -> torch.Tensor:
    """out = D(C(x)) in one pass (two for quant8), no payload materialised."""
    s = _stream_ptr(x.device) if stream is None else stream
    _lib.call("gp_roundtrip", int(as_codec(codec)), x.data_ptr(), out.data_ptr(), x.numel(), status.ptr, s)
    return out


def serialize_block(block: CompressedBlock) -> bytes:
    return HEADER.pack(int(block.codec), block.n_elems, block.scale) + block.payload_bytes()


def deserialize_block(buf: bytes, device=None) -> CompressedBlock:
    if len(buf) < HEADER_BYTES:
        raise CorruptBlockError(f"block of {len(buf)} bytes is shorter than header")
    tag, n_elems, scale = HEADER.unpack_from(buf)
    try:
        codec = Codec(tag)
    except ValueError:
        raise CorruptBlockError(f"unknown codec tag {tag}") from None
    payload = buf[HEADER_BYTES:]
    if len(payload) != payload_size(codec, n_elems):
        raise CorruptBlockError(
            f"{codec.name} block advertises {n_elems} elems but carries "
            f"{len(payload)} payload bytes"
        )
    dev = device or torch.device("cuda", torch.cuda.current_device())
    pl = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(dev) if payload else \
        torch.empty(0, dtype=torch.uint8, device=dev)
    sc = torch.tensor([scale], dtype=torch.float32, device=dev)
    return CompressedBlock(codec, n_elems, pl, sc)
