"""Oracle restatement of the reference codecs (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/gradpipe/compression.py:
  * codec tags NONE=0 / TRUNC16=1 / QUANT8=2 and widths 4/2/1 B  (:37-56)
  * wire header `<BIf` = 9 bytes                                 (:33-34)
  * `_quant_scale`                                                (:87-100)
  * `compress` finite check + three encoders                     (:103-136)
  * `decompress`                                                  (:141-151)

An encoded block is the triple (codec, scale, payload) where payload is a
numpy array of the wire element type (<f4 / <u2 / i1). `scale` is a
numpy float32 (0 for every codec but quant8).
"""

from __future__ import annotations

import numpy as np

NONE, TRUNC16, QUANT8 = 0, 1, 2
WIDTH = {NONE: 4, TRUNC16: 2, QUANT8: 1}
HEADER_BYTES = 9  # u8 tag | u32 n_elems | f32 scale   (compression.py:33-34)


class OracleCodecError(ValueError):
    """Mirrors gradpipe.errors.CodecError for the oracle."""


def quant_scale(vmax: float) -> np.float32:
    """max|v|/127 snapped down to a 17-significant-bit float32.

    compression.py:87-100: divide in float64, round to float32, clear the
    low 7 mantissa bits, and step one grid point down when the snapped
    value still overshoots (only while the bit pattern is >= 0x100).
    """
    bits = int(np.array([vmax / 127.0], dtype=np.float32).view(np.uint32)[0])
    bits &= 0xFFFFFF80
    snapped = float(np.array([bits], dtype=np.uint32).view(np.float32)[0])
    if snapped * 127.0 > vmax and bits >= 0x100:
        bits -= 0x80
    return np.array([bits], dtype=np.uint32).view(np.float32)[0]


def trunc16_halfwords(x: np.ndarray) -> np.ndarray:
    """Top halfword of each float32, low half rounded to nearest-even,
    with the +-inf halfword clamped to +-0x7F7F (compression.py:114-124)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    hi = u >> 16
    lo = u & 0xFFFF
    bump = (lo > 0x8000) | ((lo == 0x8000) & ((hi & 1) == 1))
    hi = hi + bump.astype(np.uint64)
    at_inf = (hi & 0x7FFF) == 0x7F80
    hi = hi - at_inf.astype(np.uint64)
    return hi.astype("<u2")


def quant8_codes(x: np.ndarray, scale: np.float32) -> np.ndarray:
    """Half-away-from-zero codes of x/scale, clipped to [-127, 127]
    (compression.py:131-135). Evaluated in float64 like the reference,
    including the scale==0 case where x/0 gives +-inf (-> +-127) and
    0/0 gives NaN, which numpy casts to code 0 on x86."""
    q = np.asarray(x, dtype=np.float64) / float(scale) if float(scale) != 0.0 else None
    if q is None:
        with np.errstate(divide="ignore", invalid="ignore"):
            q = np.asarray(x, dtype=np.float64) / 0.0
        codes = np.where(np.isnan(q), 0.0, np.sign(q) * 127.0)
        return codes.astype(np.int8)
    mag = np.floor(np.abs(q) + 0.5)
    return np.clip(np.sign(q) * mag, -127, 127).astype(np.int8)


def encode(vec: np.ndarray, codec: int) -> tuple[np.float32, np.ndarray]:
    """Encode one float32 block. Raises OracleCodecError on NaN/Inf
    for every codec (compression.py:108-109)."""
    v = np.ascontiguousarray(vec, dtype=np.float32).reshape(-1)
    if not np.isfinite(v).all():
        raise OracleCodecError("refusing to compress non-finite values")
    if codec == NONE:
        return np.float32(0.0), v.astype("<f4").copy()
    if codec == TRUNC16:
        return np.float32(0.0), trunc16_halfwords(v)
    if codec == QUANT8:
        if v.size == 0:
            return np.float32(0.0), np.zeros(0, np.int8)
        vmax = float(np.abs(v).max())
        if vmax == 0.0:
            return np.float32(0.0), np.zeros(v.size, np.int8)
        s = quant_scale(vmax)
        return s, quant8_codes(v, s)
    raise OracleCodecError(f"unknown codec {codec!r}")


def decode(codec: int, scale: np.float32, payload: np.ndarray) -> np.ndarray:
    """compression.py:141-151: identity / halfword<<16 / code*scale (fp32)."""
    if codec == NONE:
        return np.asarray(payload, dtype="<f4").astype(np.float32)
    if codec == TRUNC16:
        return (np.asarray(payload, dtype="<u2").astype(np.uint32) << 16).view(np.float32)
    if codec == QUANT8:
        return np.asarray(payload, dtype=np.int8).astype(np.float32) * np.float32(scale)
    raise OracleCodecError(f"unknown codec {codec!r}")


def roundtrip(vec: np.ndarray, codec: int) -> np.ndarray:
    """D(C(vec)) — the whole-vector local pre-compress of engine.py:333/:355."""
    s, pl = encode(vec, codec)
    return decode(codec, s, pl)


def payload_bytes(codec: int, n: int) -> int:
    return int(n) * WIDTH[codec]
