"""Oracle restatement of the reference ring AllReduce (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/gradpipe/collective.py:
  * `partition_blocks`                        (:35-49)
  * `_ring_allreduce_impl` reduce-scatter     (:96-115)
  * `_ring_allreduce_impl` allgather          (:117-139)
  * `ring_allreduce` p==1 identity copy       (:143-154)
and the per-endpoint traffic accounting of transport.py:85-91
(payload bytes exclude the 9-byte block header, frame bytes add the
11-byte `<IBIH` frame header to the serialized block).

All p ranks are simulated step-synchronously in one thread: at ring step s
every rank first emits its message, then every rank consumes the message of
its predecessor. Within a step a rank sends block (r-s)%p and receives
block (r-s-1)%p, which are distinct, so this order reproduces the
reference's arithmetic bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import codec as C

FRAME_HEADER_BYTES = 11  # transport.py:37  `<IBIH`


def partition_blocks(n: int, p: int) -> list[tuple[int, int]]:
    """(offset, length) of p contiguous blocks; the first n % p blocks are
    one element longer (collective.py:35-49)."""
    base, extra = divmod(int(n), int(p))
    out, off = [], 0
    for b in range(p):
        ln = base + (b < extra)
        out.append((off, ln))
        off += ln
    return out


@dataclass
class Stats:
    messages: int = 0
    payload_bytes: int = 0
    frame_bytes: int = 0

    def count(self, codec: int, n_elems: int) -> None:
        pb = C.payload_bytes(codec, n_elems)
        self.messages += 1
        self.payload_bytes += pb
        self.frame_bytes += FRAME_HEADER_BYTES + C.HEADER_BYTES + pb


@dataclass
class Message:
    phase: str          # "rs" | "ag"
    step: int
    block: int
    scale: np.float32
    payload: np.ndarray

    @property
    def wire_bytes(self) -> int:
        return C.HEADER_BYTES + self.payload.nbytes


@dataclass
class RingResult:
    outputs: list[np.ndarray]
    stats: list[Stats]
    sent: list[list[Message]] = field(default_factory=list)


def ring_allreduce_all(inputs: list[np.ndarray], codec: int = C.NONE,
                       keep_messages: bool = False) -> RingResult:
    """Run the reference ring for all ranks at once; returns per-rank
    outputs (bit-identical across ranks) and per-rank traffic stats."""
    p = len(inputs)
    n = int(np.asarray(inputs[0]).size)
    if any(np.asarray(v).size != n for v in inputs):
        raise ValueError("unequal vector lengths across ranks")
    if p == 1:
        return RingResult([np.array(inputs[0], np.float32, copy=True)], [Stats()], [[]])
    blocks = partition_blocks(n, p)
    acc = [np.array(v, dtype=np.float32, copy=True).reshape(-1) for v in inputs]
    stats = [Stats() for _ in range(p)]
    sent: list[list[Message]] = [[] for _ in range(p)]

    def view(r: int, b: int) -> np.ndarray:
        off, ln = blocks[b]
        return acc[r][off:off + ln]

    # reduce-scatter (collective.py:96-115)
    for s in range(p - 1):
        msgs = []
        for r in range(p):
            b = (r - s) % p
            sc, pl = C.encode(view(r, b), codec)
            msgs.append(Message("rs", s, b, sc, pl))
            stats[r].count(codec, blocks[b][1])
            if keep_messages:
                sent[r].append(msgs[-1])
        for r in range(p):
            m = msgs[(r - 1) % p]
            want = (r - s - 1) % p
            assert m.block == want
            tgt = view(r, want)
            tgt += C.decode(codec, m.scale, m.payload)

    # allgather (collective.py:117-139): the owner encodes once, the bytes
    # travel verbatim around the ring and everyone decodes the same bytes.
    out = [np.empty(n, np.float32) for _ in range(p)]
    wire = []
    for r in range(p):
        own = (r + 1) % p
        sc, pl = C.encode(view(r, own), codec)
        wire.append(Message("ag", -1, own, sc, pl))
        off, ln = blocks[own]
        out[r][off:off + ln] = C.decode(codec, sc, pl)
    for s in range(p - 1):
        msgs = []
        for r in range(p):
            m = wire[r]
            assert m.block == (r + 1 - s) % p
            msgs.append(Message("ag", s, m.block, m.scale, m.payload))
            stats[r].count(codec, blocks[m.block][1])
            if keep_messages:
                sent[r].append(msgs[-1])
        for r in range(p):
            m = msgs[(r - 1) % p]
            assert m.block == (r - s) % p
            off, ln = blocks[m.block]
            out[r][off:off + ln] = C.decode(codec, m.scale, m.payload)
            wire[r] = m
    return RingResult(out, stats, sent)


def ring_fold(inputs: list[np.ndarray], codec: int = C.NONE) -> np.ndarray:
    """Closed form of the same result: block b is a
    left fold starting at rank b, s_0 = x_b, s_k = fl(x_{b+k} + D(C(s_{k-1}))),
    and every rank returns D(C(s_{p-1})). Used to cross-check the simulation."""
    p = len(inputs)
    n = int(np.asarray(inputs[0]).size)
    if p == 1:
        return np.array(inputs[0], np.float32, copy=True)
    out = np.empty(n, np.float32)
    for b, (off, ln) in enumerate(partition_blocks(n, p)):
        s = np.array(inputs[b][off:off + ln], np.float32, copy=True)
        for k in range(1, p):
            s = np.asarray(inputs[(b + k) % p][off:off + ln], np.float32) + C.roundtrip(s, codec)
        out[off:off + ln] = C.roundtrip(s, codec)
    return out
