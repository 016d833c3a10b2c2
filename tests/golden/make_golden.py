"""Generate golden vectors by running the REAL reference package.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `gradpipe` from /root/reference/pkg/src, runs its codecs, its
threaded ring AllReduce over its InProcTransport, and its in-process training
engine, and writes the inputs and outputs as small .npz fixtures next to this
script. The fixtures travel to the GPU box; this script does not need to.
"""

from __future__ import annotations

import os
import sys
import threading
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from gradpipe.collective import ring_allreduce  # noqa: E402
from gradpipe.compression import Codec, compress  # noqa: E402
from gradpipe.data import synthetic_blobs  # noqa: E402
from gradpipe.engine import RunConfig, run_inproc_cluster  # noqa: E402
from gradpipe.models import logistic_model, mlp_model  # noqa: E402
from gradpipe.transport import InProcTransport  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
F32 = np.float32


def f32_from_bits(bits):
    return np.array(bits, dtype=np.uint32).view(np.float32)


def codec_cases() -> list[np.ndarray]:
    """Blocks exercising every rounding/edge rule of compression.py."""
    cases = []
    fmax = np.finfo(np.float32).max
    mn = F32(2.0 ** -126)
    cases.append(np.array([0.0, -0.0, mn, -mn, fmax, -fmax, 1.0, np.pi, -np.pi], F32))
    # trunc16 ties / near-ties / overflow clamp around 0x7F7F_xxxx
    bits = []
    for hi in (0x3F80, 0x3F81, 0x7F7F, 0xFF7F, 0x0001, 0x8001, 0x4049):
        for lo in (0x0000, 0x7FFF, 0x8000, 0x8001, 0xFFFF):
            bits.append((hi << 16) | lo)
    cases.append(f32_from_bits(bits))
    # subnormals
    cases.append(f32_from_bits([1, 2, 3, 0x7F, 0x80, 0x81, 0x7FFFFF, 0x807FFFFF, 0x80000001]))
    # quant8 pins from test_compression.py
    cases.append(np.array([0.0, 1.0, -1.0, 0.5], F32))
    cases.append(np.array([127.0, 2.5, -2.5, 0.5, -0.5], F32))
    cases.append(np.zeros(33, F32))
    # quant8 tiny-vmax blocks (scale snaps to 0 or to a subnormal grid)
    cases.append(f32_from_bits([0, 1, 0x80000001, 2]))
    cases.append(f32_from_bits([0, 63, 0x8000003F]))
    cases.append(f32_from_bits([64, 0, 1, 0x80000040]))
    cases.append(f32_from_bits([127 * 128, 1, 0x80000005, 5000]))
    cases.append(f32_from_bits([0x00800000 * 3 + 17, 0x7, 0x80001234]))
    # crafted quant8 ties: scale=1 exact and half-steps of a generic scale
    s = float(compress(np.array([3.3], F32), Codec.QUANT8).scale)
    ks = np.arange(-127, 128, dtype=np.float64)
    ties = (np.sign(ks) * (np.abs(ks) + 0.5) * s).astype(F32)
    cases.append(np.concatenate([np.array([3.3], F32), ties[np.abs(ties) <= 3.3]]))
    # random blocks over many magnitudes
    g = np.random.default_rng(20240601)
    for e in (-40, -30, -12, -6, 0, 3, 6, 20, 30, 37):
        cases.append((g.normal(0, 1, 257) * 10.0 ** e).astype(F32))
    mixed = (g.normal(0, 1, 4099) * 10.0 ** g.integers(-20, 20, 4099)).astype(F32)
    cases.append(mixed)
    return cases


def make_codec():
    out = {}
    cases = codec_cases()
    for i, x in enumerate(cases):
        out[f"x{i}"] = x
        b1 = compress(x, Codec.TRUNC16)
        out[f"t16_{i}"] = np.frombuffer(b1.payload, "<u2").copy()
        b2 = compress(x, Codec.QUANT8)
        out[f"q8_{i}"] = np.frombuffer(b2.payload, np.int8).copy()
        out[f"q8s_{i}"] = np.array([b2.scale], F32)
    out["count"] = np.array([len(cases)])
    np.savez_compressed(os.path.join(OUT, "codec_golden.npz"), **out)
    print("codec cases:", len(cases))


def run_ranks(p, fn, timeout_s=30.0):
    tr = InProcTransport(p, timeout_s=timeout_s)
    res, errs = [None] * p, []

    def go(r):
        try:
            res[r] = fn(r, tr.endpoint(r))
        except BaseException as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=go, args=(r,)) for r in range(p)]
    [t.start() for t in th]
    [t.join() for t in th]
    if errs:
        raise errs[0]
    return res


class Recorder:
    """Wrap an endpoint to log (block_index, wire length) of every send."""

    def __init__(self, ep):
        self.ep, self.log = ep, []

    def __getattr__(self, k):
        return getattr(self.ep, k)

    def send(self, dst, payload, msg_type=0, iteration=0, block_index=0):
        self.log.append((block_index, len(payload)))
        return self.ep.send(dst, payload, msg_type, iteration, block_index)


def ring_inputs(p, n, variant):
    g = np.random.default_rng((p, n, variant))
    mag = {0: 1.0, 1: 1e-6, 2: 1e6, 3: 1e-39}[variant]
    return [(g.normal(0, 1, n) * mag).astype(F32) for _ in range(p)]


def make_ring():
    out = {}
    keys = []
    for p in (2, 3, 4, 8):
        for n in (1, 5, 7, 10, 64, 1000, 4099):
            for variant in ((0, 1, 2, 3) if n in (1000, 4099) else (0,)):
                ins = ring_inputs(p, n, variant)
                for codec in Codec:
                    def op(r, ep):
                        rec = Recorder(ep)
                        y = ring_allreduce(ins[r], r, p, rec, codec, iteration=3)
                        s = ep.stats.snapshot()
                        return y, rec.log, (s.messages, s.payload_bytes, s.frame_bytes)

                    res = run_ranks(p, op)
                    for y, _, _ in res[1:]:
                        assert y.tobytes() == res[0][0].tobytes()
                    k = f"p{p}_n{n}_v{variant}_c{int(codec)}"
                    out[k + "_out"] = res[0][0]
                    out[k + "_stats"] = np.array([r[2] for r in res], np.int64)
                    out[k + "_log"] = np.array([r[1] for r in res], np.int64)
                    keys.append(k)
                out[f"p{p}_n{n}_v{variant}_in"] = np.stack(ins)
    out["keys"] = np.array(keys)
    np.savez_compressed(os.path.join(OUT, "ring_golden.npz"), **out)
    print("ring cases:", len(keys))


from cases import ENGINE_CASES  # noqa: E402


def make_engine():
    data = synthetic_blobs(dim=8, num_classes=3, num_samples=512, seed=1)
    models = {"log": logistic_model(8, 3), "mlp": mlp_model(8, (16, 12), 3)}
    out = {}
    for name, m, mode, codec, p, T, K, warm, lr, bs, dec in ENGINE_CASES:
        cfg = RunConfig(mode=mode, iterations=T, learning_rate=lr, codec=Codec(codec),
                        depth=K, batch_size=bs, warmup_epochs=warm, seed=7,
                        lr_decay_every=dec, lr_decay_factor=0.5)
        res = run_inproc_cluster(p, cfg, data, models[m])
        for r in res[1:]:  # workers and, in ps_sync, the server (last result)
            assert r.params.tobytes() == res[0].params.tobytes()
        out[name] = res[0].params
        out[name + "_loss"] = np.array([x[2] for x in res[0].metrics])
    np.savez_compressed(os.path.join(OUT, "engine_golden.npz"), **out)
    print("engine cases:", len(ENGINE_CASES))


if __name__ == "__main__":
    warnings.simplefilter("ignore")
    make_codec()
    make_ring()
    make_engine()
