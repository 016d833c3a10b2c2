"""Workload for the bounds-checked library (libpipesgd_checked.so, selected
with PIPESGD_LIB): run by tests/test_gpu_bounds.py in a subprocess. Every
ring variant (emulated and per-rank launches; LL, flag and direct
reduce-scatter paths; plain and fused; unaligned block offsets) must finish
without a bounds violation and still equal the oracle. With
PIPESGD_CHECKED_SELFTEST=1 the kernel makes one deliberate out-of-bounds
store and the call must fail with the bounds error (negative control)."""

import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1811_03619_b200 as P  # noqa: E402
from helpers import assert_bits_equal, run_ranks  # noqa: E402
from oracle import codec as OC  # noqa: E402
from oracle import ring as OR  # noqa: E402
from paper_1811_03619_b200 import _lib  # noqa: E402
from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait  # noqa: E402

assert os.path.basename(_lib.LIB_PATH) == "libpipesgd_checked.so", _lib.LIB_PATH


def wire_bytes(ep, reset=True):
    import ctypes
    v = ctypes.c_uint64()
    _lib.call("gp_comm_wire_bytes", ep._comm, ep.rank, int(reset), ctypes.byref(v))
    return int(v.value)


WIRE = []  # (p, n, codec, protocol, kernel-counted bytes, reference payload bytes), summed over ranks
LL_MAX = 256 << 10  # transports cap LL blocks here, so the larger sizes exercise the flag protocol


def run_case(tr, p, n, codec, fused, seed):
    import ctypes
    g = np.random.default_rng(seed)
    ins = [g.normal(0, 1, n).astype(np.float32) for _ in range(p)]
    w = P.Codec(codec).bytes_per_elem
    for r in range(p):
        wire_bytes(tr.endpoint(r))
        tr.endpoint(r).reset_stats()

    def op(r, ep):
        dev = ep.device
        with torch.cuda.device(dev):
            x = torch.from_numpy(ins[r]).to(dev)
            out = torch.empty_like(x)
            s = ep.stream
            s.wait_stream(torch.cuda.current_stream(dev))
            if fused:
                slot = torch.empty(max(n * w, 16), dtype=torch.uint8, device=dev)
                sc = torch.empty(1, device=dev)
                allreduce_into(x, out, ep, codec, 3, s, precompress=True, slot=slot, slot_scale=sc)
                endpoint_wait(ep, n, s)
                return slot[:n * w].cpu().numpy(), sc.cpu().numpy()
            allreduce_into(x, out, ep, codec, 3, s)
            endpoint_wait(ep, n, s)
            return out.cpu().numpy()

    res = run_ranks(tr, op)
    got = sum(wire_bytes(tr.endpoint(r)) for r in range(p))
    want = sum(tr.endpoint(r).stats.payload_bytes for r in range(p))
    o = (ctypes.c_int64 * 5)()
    _lib.call("gp_ring_plan", n, p, tr.endpoint(0).info()["ctas"], codec, 1 if fused else 0, n, o)
    ll = bool(o[2]) and ((n + p - 1) // p + 16) * w <= LL_MAX  # plan_ring's rule under the cap
    WIRE.append((p, n, codec, "LL" if ll else "flag", got, want))
    if not ll:  # every payload byte the reference hands its transport, stored exactly once into a peer
        assert got == want, (p, n, codec, fused, got, want)
    else:  # LL: every 4 payload bytes travel in an 8-byte word, plus header lines and group padding
        assert 2 * want <= got <= 2 * want + 256 * p * p, (p, n, codec, got, want)  # edge groups, header lines
    if fused:
        summed = OR.ring_allreduce_all([OC.roundtrip(v, codec) for v in ins], codec).outputs[0]
        s_want, pl_want = OC.encode(summed, codec)
        for r, (pl, sc) in enumerate(res):
            assert pl.tobytes() == np.asarray(pl_want).tobytes(), (p, n, codec, r)
            assert np.float32(sc[0]).tobytes() == np.float32(s_want).tobytes(), (p, n, codec, r)
    else:
        want = OR.ring_allreduce_all(ins, codec).outputs[0]
        for r, y in enumerate(res):
            assert_bits_equal(y, want, f"p={p} n={n} codec={codec} rank {r}")


def main():
    if os.environ.get("PIPESGD_CHECKED_SELFTEST"):
        tr = P.EmulatedTransport(2, timeout_s=10.0, max_elems=4096)
        try:
            run_case(tr, 2, 1000, 0, False, 1)
        except P.CollectiveError as e:
            assert "bounds-checked build" in str(e), e
            print("SELFTEST CAUGHT", e)
            return
        raise SystemExit("the deliberate out-of-bounds store was not caught")
    cases = {2: [1, 17, 4099, 300_007, 1_200_007], 3: [5, 2_000_003], 4: [4099, 1_000_003], 8: [777, 250_007]}
    for p, sizes in cases.items():
        tr = P.EmulatedTransport(p, timeout_s=60.0, max_elems=max(sizes), ll_max_bytes=LL_MAX)
        for n in sizes:
            for codec in (0, 1, 2):
                for fused in (False, True):
                    run_case(tr, p, n, codec, fused, n + codec)
        tr.close()
        print(f"emulated p={p} ok", flush=True)
    for p, sizes in {2: [4099, 1_200_007], 4: [4099, 2_000_003]}.items():
        tr = P.GpuTransport(p, devices=[r % torch.cuda.device_count() for r in range(p)], timeout_s=60.0,
                            max_elems=max(sizes), ll_max_bytes=LL_MAX)
        for n in sizes:
            for codec in (0, 1, 2):
                for fused in (False, True):
                    run_case(tr, p, n, codec, fused, 7 * n + codec)
        tr.close()
        print(f"per-rank p={p} ok", flush=True)
    import json
    print("WIRE " + json.dumps(WIRE))
    print("CHECKED OK")


if __name__ == "__main__":
    main()
