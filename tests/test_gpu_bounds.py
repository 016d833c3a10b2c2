"""Memory-safety checks (the pool has no compute-sanitizer):

* the bounds-checked library (libpipesgd_checked.so, csrc/ring.cu
  ring_access_ok) runs every ring variant with each payload / vector / LL /
  flag access checked against its buffer or inbox slot, and a negative
  control proves a deliberate out-of-bounds store is caught;
* guard bands: every kernel of the product library writes exactly its
  output bytes -- canary bytes around the outputs stay untouched (odd sizes,
  every codec, codec kernels, the update, the ring's fp32 and slot outputs).
"""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from helpers import real_transport, run_ranks

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1811_03619_b200", "libpipesgd_checked.so")


def run_checked(extra_env=None):
    env = dict(os.environ, PIPESGD_LIB=CHECKED, **(extra_env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_worker.py")], env=env,
                          capture_output=True, text=True, timeout=900)


def test_bounds_checked_build_runs_every_ring_variant_clean():
    assert os.path.exists(CHECKED), "build the checked library: __graft_entry__.build()"
    r = run_checked()
    assert r.returncode == 0 and "CHECKED OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_bounds_checked_build_catches_a_deliberate_overrun():
    r = run_checked({"PIPESGD_CHECKED_SELFTEST": "1"})
    assert r.returncode == 0 and "SELFTEST CAUGHT" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


CANARY = 0xA5
PAD = 4096


def guarded(nbytes, dev="cuda:0"):
    """A view of nbytes inside a canary-filled buffer (16-byte aligned)."""
    buf = torch.full((nbytes + 2 * PAD,), CANARY, dtype=torch.uint8, device=dev)
    return buf, buf[PAD:PAD + nbytes]


def assert_guards(buf, nbytes, what):
    b = buf.cpu().numpy()
    lo, hi = b[:PAD], b[PAD + nbytes:]
    assert (lo == CANARY).all() and (hi == CANARY).all(), \
        f"{what}: bytes outside the output changed ({np.flatnonzero(lo != CANARY)[:4]}, " \
        f"{np.flatnonzero(hi != CANARY)[:4]})"


@pytest.mark.parametrize("n", [1, 5, 17, 4099, 100_003])
@pytest.mark.parametrize("codec", [0, 1, 2])
def test_codec_kernels_write_only_their_outputs(P, n, codec):
    from paper_1811_03619_b200 import _lib
    from paper_1811_03619_b200.compression import CodecStatus, roundtrip_async
    w = P.Codec(codec).bytes_per_elem
    x = torch.randn(n, device="cuda")
    pbuf, pay = guarded(n * w)
    st = CodecStatus(x.device)
    _lib.call("gp_encode", codec, x.data_ptr(), n, pay.data_ptr(), st.ptr, torch.cuda.current_stream().cuda_stream)
    obuf, out = guarded(4 * n)
    _lib.call("gp_decode", codec, pay.data_ptr(), st.scale_view.data_ptr(), n, out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    rbuf, rt = guarded(4 * n)
    roundtrip_async(x, codec, rt.view(torch.float32), CodecStatus(x.device))
    wbuf, wv = guarded(4 * n)
    wv.view(torch.float32).copy_(x)
    _lib.call("gp_consume_update", wv.data_ptr(), codec, pay.data_ptr(), st.scale_view.data_ptr(), n, 0.01, 2,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for buf, nb, what in ((pbuf, n * w, "encode"), (obuf, 4 * n, "decode"), (rbuf, 4 * n, "roundtrip"),
                          (wbuf, 4 * n, "consume_update")):
        assert_guards(buf, nb, what)
    assert torch.equal(rt.view(torch.int32), out.view(torch.int32))


@pytest.mark.parametrize("n", [1, 17, 4099, 300_007])
@pytest.mark.parametrize("codec", [0, 1, 2])
def test_ring_writes_only_its_outputs(P, n, codec):
    """Per-rank launches (ranks share GPUs when the box has fewer): the fp32
    output and the fused slot output are written exactly, nothing around them."""
    from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait
    p, w = 4, P.Codec(codec).bytes_per_elem
    # the largest size takes the flag protocol, the others the LL slots
    tr = real_transport(P, p, timeout_s=60.0, max_elems=n, ll_max_bytes=0 if n >= 300_007 else None)

    def op(r, ep):
        dev = ep.device
        with torch.cuda.device(dev):
            x = torch.randn(n, device=dev)
            obuf, out = guarded(4 * n, dev)
            sbuf, slot = guarded(n * w, dev)
            cbuf, sc = guarded(4, dev)
            s = ep.stream
            s.wait_stream(torch.cuda.current_stream(dev))
            allreduce_into(x, out.view(torch.float32), ep, codec, 1, s)
            endpoint_wait(ep, n, s)
            o2buf, out2 = guarded(4 * n, dev)
            allreduce_into(x, out2.view(torch.float32), ep, codec, 2, s, precompress=True, slot=slot,
                           slot_scale=sc.view(torch.float32))
            endpoint_wait(ep, n, s)
            for buf, nb, what in ((obuf, 4 * n, "out"), (sbuf, n * w, "slot"), (cbuf, 4, "slot scale"),
                                  (o2buf, 4 * n, "quant8 scratch")):
                assert_guards(buf, nb, f"rank {r} {what}")

    try:
        run_ranks(tr, op)
    finally:
        tr.close()
