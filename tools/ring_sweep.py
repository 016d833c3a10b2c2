"""Ring AllReduce sweep under torchrun: fused compressed ring vs NCCL.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/ring_sweep.py [--sizes ...]

One process per GPU, inboxes shared over CUDA IPC (ProcessGroupTransport).
Prints one JSON line per (size, codec) on rank 0: device time per call
(CUDA events on the launching stream, max over ranks), fp32-equivalent bus
bandwidth 2(p-1)/p*4n/t (nccl-tests convention), wire bus bandwidth
2(p-1)/p*w*n/t, and NCCL all_reduce on the same buffer for comparison.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1811_03619_b200 import Codec, ProcessGroupTransport  # noqa: E402
from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait  # noqa: E402


def clock_ctx(enabled, device):
    if not enabled:
        import contextlib
        return contextlib.nullcontext(None)
    from bench import ClockSampler
    return ClockSampler(device)


def cpu_reference_ms(n, p, cname, reps=2):
    """The unmodified reference ring (collective.ring_allreduce over
    transport.InProcTransport, p rank threads in one process, engine.py-style)
    on this host: ms per call, or None when baseline/_ref is absent."""
    import threading
    import time
    from bench import load_reference
    ref = load_reference()
    if ref is None:
        return None
    from gradpipe import collective as RC
    from gradpipe import compression as RZ
    from gradpipe import transport as RT
    codec = RZ.Codec.parse(cname)
    g = np.random.default_rng(n)
    ins = [g.normal(0, 1, n).astype(np.float32) for _ in range(p)]
    best = None
    for _ in range(reps):
        tr = RT.InProcTransport(p)
        th = [threading.Thread(target=RC.ring_allreduce, args=(ins[r], r, p, tr.endpoint(r), codec)) for r in range(p)]
        t0 = time.perf_counter()
        [t.start() for t in th]
        [t.join() for t in th]
        dt = (time.perf_counter() - t0) * 1e3
        best = dt if best is None else min(best, dt)
    return best


def timed(fn, iters, warmup, stream):
    for _ in range(warmup):
        fn()
    stream.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(2_000_000)  # host enqueues the whole series before the clock starts
    a.record(stream)
    for _ in range(iters):
        fn()
    b.record(stream)
    b.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) / 1e3


def max_all(v):
    t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def cpu_name():
    try:
        return [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:  # noqa: BLE001
        return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=str, default="256,4096,65536,1048576,4194304,16777216,67108864,268435456")
    ap.add_argument("--codecs", type=str, default="none,trunc16,quant8")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--nccl", action="store_true")
    ap.add_argument("--clocks", action="store_true", help="NVML SM clocks + throttle reasons during each series")
    ap.add_argument("--eq5", action="store_true",
                    help="Eq. 5 prediction per row from GPU-calibrated alpha/beta (rank 0: GPUs 0-1), gamma "
                         "(one fused hop on one GPU, per size and codec) and S (all-rank GPU barrier)")
    ap.add_argument("--cpu-ref-max", type=int, default=0,
                    help="also time the reference's ring_allreduce (baseline/_ref, InProcTransport, p threads) "
                         "on rank 0's host for sizes up to this many elements")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, p = dist.get_rank(), dist.get_world_size()
    sizes = [int(s) for s in args.sizes.split(",")]
    ep = ProcessGroupTransport.endpoint(local, max_elems=max(sizes), timeout_s=20.0, ctas=args.ctas)
    stream = torch.cuda.current_stream()
    sym = None
    if args.eq5:
        from paper_1811_03619_b200 import timing as T
        S = T.barrier_time(ep)
        S = float(max_all(S))
        ab = {}
        store = dist.distributed_c10d._get_default_store()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            try:
                ab = T.calibrate_nvlink(devices=(0, 1), nbytes=256 << 20, ctas=148, iters=4000)
            finally:
                store.set("sweep_eq5_calib", "done")
        else:
            store.wait(["sweep_eq5_calib"])
        sym = {"S_s": S, **ab}
        # per-call fixed cost: Eq. 5's residual on the smallest real call
        # (16 elements per rank, codec none), used by eq5_ext at every size
        xs = torch.randn(16 * p, device="cuda")
        ys = torch.empty_like(xs)
        t_small = timed(lambda: allreduce_into(xs, ys, ep, Codec.NONE, 0, stream), 50, 5, stream)
        endpoint_wait(ep, 16 * p, stream)
        if rank == 0 and "alpha_s" in sym:
            g_small = T.gamma_hop(Codec.NONE, 16, torch.device("cuda", local), ring_ctas=ep.info()["ctas"])
            sym["fixed_s"] = T.ring_fixed_overhead(t_small, p, 16 * p, sym["alpha_s"], sym["beta_s_per_byte"],
                                                   g_small, S)
            sym["small_call_s"] = t_small
        if rank == 0:
            print(json.dumps({"eq5_symbols": sym, "cpu": cpu_name(), "cpu_count": os.cpu_count()}), flush=True)
    for n in sizes:
        g = torch.Generator(device="cuda").manual_seed(1000 * rank + n % 997)
        x = torch.randn(n, device="cuda", generator=g)
        out = torch.empty_like(x)
        for cname in args.codecs.split(","):
            codec = Codec.parse(cname)
            it = max(3, min(args.iters, int(4e9 // max(1, 8 * n))))

            def run():
                allreduce_into(x, out, ep, codec, 0, stream)

            with clock_ctx(args.clocks, local) as clk:
                t = timed(run, it, args.warmup, stream)
            endpoint_wait(ep, n, stream)
            clk = clk if args.clocks else None
            rec = {"p": p, "n": n, "bytes": 4 * n, "codec": cname, "ms": t * 1e3,
                   "busbw_gbs": 2 * (p - 1) / p * 4 * n / t / 1e9,
                   "wire_busbw_gbs": 2 * (p - 1) / p * codec.bytes_per_elem * n / t / 1e9,
                   "ctas": ep.info()["ctas"]}
            if args.check:  # every rank holds the same bits (oracle parity: tests/test_gpu_ring.py)
                allreduce_into(x, out, ep, codec, 0, stream)
                endpoint_wait(ep, n, stream)
                ref = out.clone()
                dist.broadcast(ref, 0)
                same = torch.tensor([int(torch.equal(ref.view(torch.int32), out.view(torch.int32)))], device="cuda")
                dist.all_reduce(same, op=dist.ReduceOp.MIN)
                rec["replicas_bit_identical"] = bool(same.item())
            if clk is not None:
                rec["clocks"] = clk.summary()
            if sym is not None and rank == 0:
                from paper_1811_03619_b200 import timing as T
                dv = torch.device("cuda", local)
                gam = T.gamma_hop(codec, max(1, n // p), dv, ring_ctas=ep.info()["ctas"])
                dlt = T.delta_decode(codec, max(1, n // p), dv)
                rec["eq5"] = T.compare_ring(t, p, codec, n, sym["alpha_s"], sym["beta_s_per_byte"], gam, sym["S_s"],
                                            dlt, fixed_s=sym.get("fixed_s", 0.0), fence_s=sym.get("phi_s", 0.0),
                                            fenced_phases=T.ring_fenced_phases(n, p, ep.info()["ctas"], codec))
                rec["eq5"]["gamma_gbs"] = 1 / gam / 1e9 if gam > 0 else None
            if args.cpu_ref_max and n <= args.cpu_ref_max:
                dist.barrier()
                if rank == 0:
                    ms = cpu_reference_ms(n, p, cname)
                    if ms is not None:
                        rec["cpu_reference"] = {"ms": ms, "speedup": ms / (t * 1e3), "threads": p,
                                                "what": "baseline/_ref gradpipe.collective.ring_allreduce over "
                                                        "InProcTransport, one thread per rank, best of 2"}
                dist.barrier()
            if rank == 0:
                print(json.dumps(rec), flush=True)
        if args.nccl:
            y = x.clone()
            t = timed(lambda: dist.all_reduce(y), max(3, min(args.iters, int(4e9 // max(1, 8 * n)))), args.warmup, stream)
            if rank == 0:
                print(json.dumps({"p": p, "n": n, "bytes": 4 * n, "codec": "nccl", "ms": t * 1e3,
                                  "busbw_gbs": 2 * (p - 1) / p * 4 * n / t / 1e9}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
