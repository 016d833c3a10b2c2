"""Pipe-SGD benchmark: width-2 Pipe-SGD iterations/s with the fused compressed
ring AllReduce on B200, plus ring bus bandwidth, roofline and CPU baselines.

    python bench.py [--gpus 1] [--steps 30] [--warmup 5]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P bench.py --gpus N --steps K --warmup W
    python bench.py --impl reference ...     # the reference's CPU path (baseline/_ref)

Workload (BASELINE.json configs[2], "C3", the largest configuration that
fits one GPU): AlexNet-shaped (torchvision AlexNet, 61,100,840 fp32 params,
ImageNet-shaped 3x224x224 synthetic batch, global batch 256 as in the paper,
PAPER.md:250) trained with Pipe-SGD width 2 and 8-bit quantized ring
compression; the fixed global batch is split over N GPUs (strong scaling,
as in the paper's setup). One step = one Pipe-SGD iteration on every rank:
consume the aggregated gradient of t-2 (decode, /p, SGD), forward+backward
on the rank's batch, whole-vector D(C(grad)), fused compressed ring
AllReduce on the comm stream, whole-vector re-compress of the sum into
slot t. Prints ONE JSON line (rank 0). `--model c1|c2|c4` selects the other
BASELINE configs (each with its codec and global batch by default).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Pipe-SGD iters/sec & compressed ring-allreduce bus GB/s at 1/2/4/8 B200"
NVLINK_PEAK_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction (MEASURED_PEAKS has no NVLink)
L2_BYTES = 126.5 * 2**20
FULL_CTAS = 592  # 128-thread ring CTAs filling every SM (16 warps per SM)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="c3")
    ap.add_argument("--codec", default=None, help="default: the config's codec (BASELINE.json configs)")
    ap.add_argument("--mode", default="pipe_sgd")
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--global-batch", type=int, default=None,
                    help="default: the paper's global batch for the config (100 MNIST, 512 CIFAR, 256 ImageNet)")
    ap.add_argument("--ctas", type=int, default=-1,
                    help="128-thread CTAs the ring kernel may occupy per GPU (-1: engine.default_comm_partition "
                         "-- Pipe-SGD 64 on gradients <= 8 MB else 4 per partition SM, D-Sync every SM; "
                         "0: every SM)")
    ap.add_argument("--comm-sms", type=int, default=-1,
                    help="SMs of the green-context partition the comm stream runs in (-1: "
                         "engine.default_comm_partition -- Pipe-SGD at N > 1: 32 on gradients of 8-32 MB, 48 above; "
                         "0: no partition)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--graphs", type=int, default=1,
                    help="replay the steady-state step as CUDA graphs (pipe_sgd / d_sync / ps_sync, fused)")
    ap.add_argument("--fused", type=int, default=1,
                    help="one comm kernel per step (pre-compress + ring + re-compress fused)")
    ap.add_argument("--channels-last", type=int, default=0,
                    help="feed NHWC activations to cuDNN (no NCHW<->NHWC transposes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-allreduce-sweep", action="store_true")
    a = ap.parse_args()
    dflt = CONFIG_DEFAULTS.get(a.model, ("none", 256))
    if a.codec is None:
        a.codec = dflt[0]
    if a.global_batch is None:
        a.global_batch = dflt[1]
    return a


# BASELINE.json configs: codec and global batch per model
CONFIG_DEFAULTS = {"c1": ("none", 100), "c2": ("trunc16", 512), "c3": ("quant8", 256), "c4": ("none", 256)}


# ------------------------------------------------------------------ helpers

class ClockSampler:
    """SM clocks + throttle reasons sampled every few ms while the timed region
    runs (NVML in a thread: nvidia-smi's own start-up is longer than a
    150 ms timed region). Falls back to `nvidia-smi -lms 100`."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int, period_s: float = 0.005):
        self.device = device
        self.period = period_s
        self.proc = None
        self.nvml = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, float, set]] = []
        self._stop = threading.Event()

    def _nvml_sample(self):
        m = self.nvml
        sm = m.nvmlDeviceGetClockInfo(self.h, m.NVML_CLOCK_SM)
        r = m.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        bits = [m.nvmlClocksEventReasonHwSlowdown, m.nvmlClocksEventReasonHwThermalSlowdown,
                m.nvmlClocksEventReasonSwThermalSlowdown, m.nvmlClocksEventReasonSwPowerCap]
        self.samples.append((float(sm), self.max_sm, {nm for nm, b in zip(self.NAMES, bits) if r & b}))

    def _poll(self):
        while not self._stop.is_set():
            try:
                self._nvml_sample()
            except Exception:  # noqa: BLE001 - a failed sample is just skipped
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml:
            self._stop.set()
            self._t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for s_mhz, m_mhz, rs in self.samples:
            sm.append(s_mhz)
            mx = max(mx, m_mhz)
            reasons |= rs
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float over the default process group (CPU tensor for
    gloo, device tensor for nccl); the value itself when not distributed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = device if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_model():
    try:
        return [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:  # noqa: BLE001
        return "unknown"


# ------------------------------------------------- the reference's CPU path

def load_reference():
    """The unmodified reference package, installed into baseline/_ref
    (git-ignored; it travels to the GPU box with the repo snapshot):
    `pip install --no-index --no-deps --target baseline/_ref <copy of
    /root/reference/pkg>`. None when absent (then the oracle port stands in)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "gradpipe")):
        return None
    if path not in sys.path:
        sys.path.append(path)
    try:
        import gradpipe  # noqa: F401
        from gradpipe import collective, compression, engine, models, transport  # noqa: F401
    except Exception:  # noqa: BLE001 - a broken install is reported as absent
        return None
    import gradpipe
    return gradpipe


class RefPath:
    """The reference's per-iteration Pipe-SGD hot path on this host's CPU,
    p ranks as threads of one process exactly like run_inproc_cluster
    (engine.py:563-618), for an n-element gradient. Per rank and step:
      decompress(slot[t-K]) -> aggregate_mean -> sgd_update   (engine.py:420-426, :302-307)
      compress(grad)                                          (engine.py:333)
      ring_allreduce(decompress(block)) over InProcTransport  (engine.py:399-406)
      compress(summed) into slot t                            (engine.py:407)
    The model's forward/backward is not part of it: the reference has no
    CNN (models.py has logistic / MLP only), so this flatters the reference.
    Uses the real reference package when baseline/_ref holds it (kind
    "reference"), else the oracle's restatement of it (kind "port")."""

    def __init__(self, n, p, codec_name, depth=2, seed=0):
        from concurrent.futures import ThreadPoolExecutor
        self.ref = load_reference()
        self.kind = "reference" if self.ref is not None else "port"
        self.n, self.p, self.depth = n, p, depth
        g = np.random.default_rng(seed)
        self.grads = [g.normal(0, 1e-2, n).astype(np.float32) for _ in range(p)]
        w0 = g.normal(0, 0.05, n).astype(np.float32)
        self.w = [w0.copy() for _ in range(p)]
        self.t = 1
        if self.ref is not None:
            from gradpipe import compression as RC
            from gradpipe import transport as RT
            self.codec = RC.Codec.parse(codec_name)
            zero = RC.compress(np.zeros(n, np.float32), self.codec)
            self.tr = RT.InProcTransport(p)
        else:
            from oracle import codec as OC
            self.codec = {"none": OC.NONE, "trunc16": OC.TRUNC16, "quant8": OC.QUANT8}[codec_name]
            zero = OC.encode(np.zeros(n, np.float32), self.codec)
            self.tr = None
        self.slots = [[zero] * depth for _ in range(p)]
        self.threads = p
        self.pool = ThreadPoolExecutor(p) if p > 1 else None

    def _rank_step_ref(self, r):
        from gradpipe import collective as RCo
        from gradpipe import compression as RC
        from gradpipe import engine as RE
        from gradpipe import models as RM
        t, p = self.t, self.p
        total = RC.decompress(self.slots[r].pop(0))
        self.w[r] = RM.sgd_update(self.w[r], RE.aggregate_mean(total, p), 0.05)
        block = RC.compress(self.grads[r], self.codec)
        summed = RCo.ring_allreduce(RC.decompress(block), r, p, self.tr.endpoint(r), self.codec, iteration=t)
        self.slots[r].append(RC.compress(summed, self.codec))

    def _step_port(self):
        from oracle import codec as OC
        from oracle import engine as OE
        from oracle import ring as OR
        p = self.p
        for r in range(p):
            total = OC.decode(self.codec, *self.slots[r].pop(0))
            self.w[r] = OE.sgd_update(self.w[r], OE.aggregate_mean(total, p), 0.05)
        if self.pool is not None:
            local = list(self.pool.map(lambda g: OC.roundtrip(g, self.codec), self.grads))
        else:
            local = [OC.roundtrip(g, self.codec) for g in self.grads]
        summed = OR.ring_allreduce_all(local, self.codec).outputs[0] if p > 1 else local[0].copy()
        for r in range(p):
            self.slots[r].append(OC.encode(summed, self.codec))

    def step(self):
        if self.ref is None:
            self._step_port()
        elif self.pool is not None:
            list(self.pool.map(self._rank_step_ref, range(self.p)))
        else:
            self._rank_step_ref(0)
        self.t += 1


def ref_sample_size(n, p, codec_name, seconds_per_step):
    """Elements per reference step so one step takes about `seconds_per_step`:
    the per-element cost measured on a 2^20-element probe of the same path.
    The bounded sample is a contiguous slice of the gradient; the path is
    elementwise (its cost is linear in n), so iters/s = (n_s / n) / t_step."""
    m = min(n, 1 << 20)
    probe = RefPath(m, p, codec_name)
    probe.step()
    t0 = time.perf_counter()
    probe.step()
    per_elem = (time.perf_counter() - t0) / m
    ns = int(min(n, max(m, seconds_per_step / max(per_elem, 1e-12))))
    return max(p * 16, ns - ns % (p * 16)) if ns < n else n


def reference_rate(n, p, codec_name, steps, warmup, seconds_per_step=2.0):
    """iters/s of the reference path (scaled from the bounded sample), and the sample."""
    ns = ref_sample_size(n, p, codec_name, seconds_per_step)
    rp = RefPath(ns, p, codec_name)
    for _ in range(warmup):
        rp.step()
    per = []
    for _ in range(steps):
        t0 = time.perf_counter()
        rp.step()
        per.append(time.perf_counter() - t0)
    t = float(np.mean(per))
    return (ns / n) / t, rp, ns, t


def ref_sample_text(rp, n, ns, t, steps, codec_name):
    who = ("the unmodified reference package (baseline/_ref/gradpipe: compression.compress/decompress, "
           "collective.ring_allreduce over transport.InProcTransport, engine.aggregate_mean, "
           "models.sgd_update)" if rp.kind == "reference" else "the oracle's restatement of the reference path")
    frac = "the full gradient" if ns == n else f"a {ns}-element slice ({ns / n:.3f}) of the {n}-element gradient, " \
                                              f"iters/s scaled by that fraction (the path is elementwise)"
    return (f"{who}: per step and rank decompress(slot t-2) -> mean -> SGD, compress({codec_name}) of the local "
            f"gradient, ring_allreduce over p={rp.p} ranks as threads, compress of the sum; {frac}; {steps} steps "
            f"of {t:.2f} s; no forward/backward (the reference has no CNN: flatters the reference); "
            f"host {cpu_model()}, {os.cpu_count()} cpus")


def reference_arm(args, ws, rank):
    if rank != 0:
        return None
    from paper_1811_03619_b200.models import build_torch_model
    mod, _, _ = build_torch_model(args.model)
    n = sum(p.numel() for p in mod.parameters())
    p = max(1, args.gpus)
    v, rp, ns, t = reference_rate(n, p, args.codec, args.steps, args.warmup)
    sample = ref_sample_text(rp, n, ns, t, args.steps, args.codec)
    return {"metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": workload_config(args, n, args.gpus),
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": rp.threads, "kind": rp.kind,
                             "sample": sample},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


MODEL_NAMES = {"c1": ("C1 (configs[0]): MNIST-shaped MLP 784-500-500-10", "MLP 784-500-500-10"),
               "c2": ("C2 (BASELINE.json configs[1]): CIFAR-10-shaped small CNN", "SmallCNN 3conv+2fc"),
               "c3": ("C3 (configs[2]): AlexNet ImageNet-shaped", "torchvision AlexNet"),
               "c4": ("C4 (configs[3]): ResNet-50 ImageNet-shaped", "torchvision ResNet-50")}


def workload_config(args, n, N):
    title, model = MODEL_NAMES.get(args.model, (args.model, args.model))
    width = args.depth if args.mode == "pipe_sgd" else 1
    scheme = {"pipe_sgd": "Pipe-SGD", "d_sync": "D-Sync", "ps_sync": "PS-Sync"}[args.mode]
    return {"workload": f"{title}, {scheme} width {width}, "
                        f"{args.codec} ring compression",
            "model": model, "params": n, "global_batch": args.global_batch,
            "per_gpu_batch": args.global_batch // max(N, 1), "codec": args.codec,
            "mode": args.mode, "depth": width, "parallelism": f"dp{N}",
            "cuda_graphs": bool(args.graphs) and args.mode in ("pipe_sgd", "d_sync", "ps_sync") and bool(args.fused),
            "ring_ctas": args.ctas if args.ctas > 0 else None,
            "comm_partition_sms": args.comm_sms or None,
            "model_math": "fp32 (TF32 disabled for cuDNN convolutions and cuBLAS matmuls)",
            "l2": "not flushed: each step streams the model's activations for the per-GPU batch plus the "
                  "gradient, weights and slots through HBM"}


# ------------------------------------------------------------------ our arm

def our_arm(args, ws, rank, local):
    import torch
    import torch.distributed as dist

    from paper_1811_03619_b200 import GpuTransport, ProcessGroupTransport
    from paper_1811_03619_b200.engine import RankEngine, RunConfig
    from paper_1811_03619_b200.models import FlatModel, build_torch_model

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    N = ws
    torch.backends.cudnn.benchmark = True
    torch.manual_seed(0)  # identical replicas on every rank
    mod, in_shape, classes = build_torch_model(args.model)
    fm = FlatModel(mod, dev)
    n = fm.num_params
    cap = max(n, 1 << 26) if N > 1 else (n if args.mode == "ps_sync" else 1 << 10)
    from paper_1811_03619_b200.engine import default_comm_ctas, default_comm_partition
    part_sms, part_ctas = default_comm_partition(args.mode, n, N)
    if args.comm_sms < 0:
        args.comm_sms = part_sms
    if args.ctas < 0:
        args.ctas = part_ctas if args.comm_sms else default_comm_ctas(args.mode, n)
    if N > 1:
        ep = ProcessGroupTransport.endpoint(local, max_elems=cap, ctas=args.ctas, timeout_s=60.0)
    else:
        tr = GpuTransport(1, max_elems=cap, ctas=args.ctas)
        ep = tr.endpoint(0)
    args.ctas = ep.info()["ctas"]  # the budget the ring actually runs with (reported in config)
    B = args.global_batch // N
    total_steps = 2 * (args.warmup + args.steps) + 8
    cfg = RunConfig(mode=args.mode, iterations=total_steps, learning_rate=0.01, codec=args.codec,
                    depth=args.depth, batch_size=B, seed=0)
    g = torch.Generator(device="cpu").manual_seed(1000 + rank)
    x_host = torch.randn((B, *in_shape), generator=g).pin_memory()
    y_host = torch.randint(0, classes, (B,), generator=g).pin_memory()
    if args.channels_last and len(in_shape) == 3:
        x_host = x_host.contiguous(memory_format=torch.channels_last).pin_memory()
    x_dev, y_dev = x_host.to(dev), y_host.to(dev)
    mode = {"e2e": False, "end": 0}
    use_graphs = bool(args.graphs) and args.mode in ("pipe_sgd", "d_sync", "ps_sync") and bool(args.fused)
    # Inputs: one buffer per pipeline parity. In e2e mode step t's batch is
    # copied from pinned host memory into buffer t % NB on a copy stream while
    # step t-1 computes (every step's copy stays inside the timed region);
    # resident mode leaves the buffers alone.
    bufs = {}
    copy_stream = torch.cuda.Stream(dev)
    d2h_stream = torch.cuda.Stream(dev)

    def batch_fn(r, tt):
        b = tt % bufs["nb"]
        if mode["e2e"]:
            eng.cs.wait_event(bufs["copied"][b])
        return bufs["x"][b], bufs["y"][b]

    eng = RankEngine(rank, N, ep, fm, cfg, batch_fn, trace=True, fused=bool(args.fused), comm_sms=args.comm_sms)
    args.comm_sms = eng.comm_sms  # the partition actually made (0 = none / unavailable)
    loss_host = torch.zeros(total_steps + 2, dtype=torch.float32).pin_memory()
    nb = eng.K if eng.K >= 2 else 1  # buffer index == graph parity
    bufs.update(nb=nb, x=[x_dev.clone() for _ in range(nb)], y=[y_dev.clone() for _ in range(nb)],
                copied=[torch.cuda.Event() for _ in range(nb)], free=[torch.cuda.Event() for _ in range(nb)])

    copy_events = []

    copy_after_ring = os.environ.get("BENCH_COPY_AFTER_RING", "1") == "1"

    def prefetch(tt):
        """H2D copy of step tt's batch into its buffer, once the step that read it last is done.
        Pipe-SGD under graphs: also after the ring of step tt-2 -- it overlaps the start of step
        tt-1's compute, and a PCIe copy landing beside both slowed that compute (C3, N=4: compute
        4.90 -> 5.12 ms per step); the copy still has the rest of step tt-1 (~4 ms) to finish."""
        b = tt % nb
        copy_stream.wait_event(bufs["free"][b])
        if copy_after_ring and pipe and "graphs" in bufs and tt - 2 in eng.graph_ready_tag.values():
            copy_stream.wait_event(eng.ev_agg[(tt - 2) % eng.K])
        c0 = pool.pop() if pool else torch.cuda.Event(enable_timing=True)
        c0.record(copy_stream)
        with torch.cuda.stream(copy_stream):
            bufs["x"][b].copy_(x_host, non_blocking=True)
            bufs["y"][b].copy_(y_host, non_blocking=True)
        bufs["copied"][b].record(copy_stream)
        c1 = pool.pop() if pool else torch.cuda.Event(enable_timing=True)
        c1.record(copy_stream)
        copy_events.append((c0, c1))

    def barrier():
        if N > 1:
            dist.barrier()

    host_ms = {}  # host enqueue time per step (ms), resident / e2e
    pool = []  # timing events made before the timed region (host time inside it is the step's budget)

    def timed_region(t0, steps, e2e):
        mode["e2e"] = e2e
        eng.reserve_events(8 * steps + 16)
        pool[:] = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps + 4)]
        done_evs = [torch.cuda.Event() for _ in range(steps)]
        torch.cuda.synchronize(dev)
        barrier()
        eng.events.clear()
        start = torch.cuda.Event(enable_timing=True)
        start.record(eng.cs)
        eng.ms.wait_stream(eng.cs)
        mode["end"] = t0 + steps
        if e2e:
            copy_stream.wait_stream(eng.cs)
            prefetch(t0)
        h0 = time.perf_counter()
        for t in range(t0, t0 + steps):
            step(t)
            if e2e:  # device->host read of the step's loss (async into pinned memory), on its own
                # stream after the step so the next step's kernels do not queue behind the PCIe read
                done = done_evs[t - t0]
                done.record(eng.cs)
                d2h_stream.wait_event(done)
                with torch.cuda.stream(d2h_stream):
                    loss_host[t:t + 1].copy_(eng.losses[t:t + 1], non_blocking=True)
        host_ms[e2e] = (time.perf_counter() - h0) * 1e3 / steps
        ends = []
        for st in (eng.cs, eng.ms, d2h_stream):
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            ends.append(e)
        torch.cuda.synchronize(dev)
        barrier()
        ms = max(start.elapsed_time(e) for e in ends)
        return max_over_ranks(ms, dev), list(eng.events)

    pipe = args.mode == "pipe_sgd"
    inner = eng.step if pipe else (eng.ps_step if args.mode == "ps_sync" else eng.step_sync)

    def step(tt):
        if use_graphs and "graphs" in bufs:
            if mode["e2e"]:
                eng.cs.wait_event(bufs["copied"][tt % nb])
            eng.step_graph(tt)
        else:
            inner(tt)  # batch_fn waits for the copy
        bufs["free"][tt % nb].record(eng.cs)
        if mode["e2e"] and tt + 1 < mode["end"]:
            prefetch(tt + 1)

    with torch.cuda.device(dev), torch.cuda.stream(eng.cs):
        if pipe:
            eng.prime(1)
        t = 1
        for _ in range(args.warmup):
            step(t)
            t += 1
        if use_graphs:
            # compute graph i reads input buffer i (per-parity buffers)
            eng.capture_graphs([(bufs["x"][i % nb], bufs["y"][i % nb]) for i in range(eng.K)])
            bufs["graphs"] = True

            for _ in range(max(2, eng.K)):
                step(t)
                t += 1
        prof = bool(os.environ.get("BENCH_PROFILE_RANGE"))
        if prof:  # ncu --profile-from-start off: capture the timed region only
            torch.cuda.profiler.start()
        with ClockSampler(local) as clk:
            ms_total, events = timed_region(t, args.steps, e2e=False)
        if prof:
            torch.cuda.profiler.stop()
        t += args.steps
        for _ in range(2):
            step(t)
            t += 1
        copy_events.clear()
        e2e_ms, e2e_events = timed_region(t, args.steps, e2e=True)
        copy_ms = [a.elapsed_time(b) for a, b in copy_events]
        streams = stream_timeline(e2e_events, copy_events)
        t += args.steps
        if use_graphs:
            eng.drain_graph(t - 1)
        elif pipe:
            eng.drain(t - 1)
        elif args.mode == "d_sync":
            eng.drain_sync()
        torch.cuda.synchronize(dev)
    ep._check_errors(n)
    if any(int(s.t[1].item()) for s in eng.local_status):
        raise RuntimeError("non-finite gradient in the benchmark run")

    per_step_ms = ms_total / args.steps
    value = 1e3 / per_step_ms
    e2e_value = 1e3 / (e2e_ms / args.steps)

    # per-kernel device durations over the timed region (CUDA events on the
    # launching stream; kernels overlap the other stream there)
    durs: dict[str, list[float]] = {}
    for (_, stage, e0, e1, _) in events:
        durs.setdefault(stage, []).append(e0.elapsed_time(e1))
    avg = {k: float(np.mean(v)) for k, v in durs.items()}
    w = {"none": 4, "trunc16": 2, "quant8": 1}[args.codec]
    q8 = args.codec == "quant8"
    algo = {  # algorithmic HBM bytes per launch
        "update": (8 + w) * n,                     # slot read + w read + w write
        "compress": (12 if q8 else 8) * n,         # (absmax read) + read g + write D(C(g))
        "recompress": (9 if q8 else 4 + w) * n,    # (absmax read) + read sum + write payload
    }
    from paper_1811_03619_b200.collective import partition_blocks
    blocks = partition_blocks(n, N)
    wire = (sum(blocks[(rank - s) % N][1] for s in range(N - 1)) +
            sum(blocks[(rank + 1 - s) % N][1] for s in range(N - 1))) * w if N > 1 else 0
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    iso = isolated_kernels(eng, args.codec, N, dev)
    kernels = {}
    for k in ("update", "compress", "recompress", "ring"):
        if k not in avg and k not in iso:
            continue
        kernels[k] = {"in_pipeline_avg_ms": avg.get(k), "isolated_avg_ms": iso.get(k)}
        if k in algo:
            kernels[k]["algorithmic_bytes"] = algo[k]
            if iso.get(k):
                kernels[k]["isolated_hbm_gbs"] = algo[k] / (iso[k] * 1e-3) / 1e9
            if k in avg:
                kernels[k]["in_pipeline_hbm_gbs"] = algo[k] / (avg[k] * 1e-3) / 1e9
    traffic = ncu_traffic()
    if N > 1:
        kr = kernels["ring"]
        kr["wire_bytes"] = wire
        kr["isolated_nvlink_gbs"] = wire / (iso["ring"] * 1e-3) / 1e9
        kr["in_pipeline_nvlink_gbs"] = wire / (avg["ring"] * 1e-3) / 1e9 if avg.get("ring") else None
        live = kr["in_pipeline_nvlink_gbs"] or kr["isolated_nvlink_gbs"]
        roof = {"kernel": "ring_allreduce_kernel<%s> (fused decode+add+encode+NVLink push)" % args.codec,
                "bound": "nvlink", "achieved": live, "peak": NVLINK_PEAK_GBS,
                "unit": "GB/s", "frac": live / NVLINK_PEAK_GBS,
                "traffic": traffic.get(f"ring_{args.codec}_fused_p{N}_n{n}"),
                "traffic_note": "ncu cannot replay the multi-process ring (its ranks wait on each other); traffic "
                                "is the DRAM bytes per rank of the same fused ring with all ranks emulated in one "
                                "launch (profiles/ncu_traffic.json), null when no capture exists for this "
                                "(codec, p, n)",
                "measured": "CUDA events on the comm stream around every ring launch of the timed region "
                            "(the launch shares the SMs with the CNN and waits for the slower rank); the same "
                            "kernel alone (20 back-to-back launches after L2-evicting reads, minus the reads): "
                            f"{kr['isolated_nvlink_gbs']:.1f} GB/s",
                "achieved_isolated": kr["isolated_nvlink_gbs"],
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction (MEASURED_PEAKS.json has "
                               "no NVLink entry); this pool's bidirectional push ceiling measured by "
                               "gp_calib_p2p_copy is ~690-707 GB/s",
                "algorithmic_bytes_per_launch": wire}
    else:
        copy_gbs = 8 * n / (iso["copy_4n"] * 1e-3) / 1e9
        # dominant = the kernel with the longest duration of its own (isolated):
        # at N = 1 the update and the encode overlap each other inside the
        # step, so their in-step times swap order from run to run
        dom = max([k for k in ("update", "compress", "recompress") if k in kernels and avg.get(k)],
                  key=lambda k: iso.get(k) or avg[k])
        name = {"update": "consume_update_kernel", "compress": "roundtrip_kernel",
                "recompress": "encode_kernel"}[dom]
        kd = kernels[dom]
        live = kd["in_pipeline_hbm_gbs"]
        tr = traffic.get(name)
        if q8 and dom in ("recompress", "compress") and tr is not None and traffic.get("absmax_kernel"):
            tr += traffic["absmax_kernel"]  # quant8: the absmax pass belongs to the same encode
        roof = {"kernel": name + (" (+ absmax_kernel)" if q8 and dom != "update" else ""), "bound": "hbm",
                "achieved": live, "peak": hbm_peak, "unit": "GB/s", "frac": live / hbm_peak,
                "traffic": tr,
                "measured": "CUDA events on the launching stream around every launch of the timed region "
                            "(sharing HBM and SMs with the other stream); the same kernel alone, L2 flushed "
                            f"before each launch: {kd.get('isolated_hbm_gbs', 0):.1f} GB/s",
                "achieved_isolated": kd.get("isolated_hbm_gbs"),
                "peak_source": ("MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks else
                                "of fallback: B200_PROFILING.md 6.65 TB/s (MEASURED_PEAKS.json absent)"),
                "same_size_torch_copy_gbs": copy_gbs,
                "note": "at this vector size (%d fp32) launch/ramp latency bounds every kernel: torch's own "
                        "copy of 8n bytes reaches %.0f GB/s by the same method" % (n, copy_gbs),
                "algorithmic_bytes_per_launch": algo[dom]}
    # our kernels per step: consume_update + (fused) one ring kernel, or at p=1
    # the encode (absmax+encode for quant8); unfused adds pre-compress/re-compress
    if eng.fused:
        per_iter_launches = 1 + (1 if N > 1 else (2 if q8 else 1))
    else:
        per_iter_launches = 1 + (2 if q8 else 1) + (1 if N > 1 else 0) + (2 if q8 else 1)

    allreduce = None
    if N > 1 and not args.no_allreduce_sweep:
        allreduce = ring_vs_nccl(ep, args.codec, N, dev, [1024, n, 1 << 26], ctas_list=(0, FULL_CTAS))

    # Eq. 5 symbols calibrated on this box in this run: rank 0
    # drives GPUs 0 and 1 with the flag ping-pong and peer-push kernels while
    # the other ranks wait
    calib = None
    if N > 1 and not args.no_allreduce_sweep:
        # GPU 1 must be idle while rank 0 runs the ping-pong on it (kernels of
        # two processes are time-sliced, not concurrent): the other ranks wait
        # on the TCP store, not in an NCCL barrier kernel
        torch.cuda.synchronize(dev)
        dist.barrier()
        torch.cuda.synchronize(dev)
        store = dist.distributed_c10d._get_default_store()
        if rank == 0:
            from paper_1811_03619_b200.timing import calibrate_nvlink
            try:
                calib = calibrate_nvlink(devices=(0, 1), nbytes=256 << 20, ctas=148, iters=4000)
            except RuntimeError as e:
                print(f"Eq. 5 calibration skipped: {e}", file=sys.stderr)
            finally:
                store.set("pipesgd_eq5_calibration", "done")
        else:
            store.wait(["pipesgd_eq5_calibration"])
        torch.cuda.synchronize(dev)

    # Eq. 5's gamma (one fused hop on this GPU over a block of n/p) and S
    # (all-rank GPU barrier), measured directly rather than fitted from the ring
    probes = None
    if N > 1 and not args.no_allreduce_sweep:
        from paper_1811_03619_b200 import timing as T
        S = max_over_ranks(T.barrier_time(ep), dev)
        g = ep.info()["ctas"]  # the probes run on the ring's own thread budget
        # the smallest real call (16 elements per rank, codec none): calibrates
        # the per-call cost Eq. 5 has no term for (timing.ring_fixed_overhead)
        small = ring_vs_nccl(ep, "none", N, dev, [16 * N])[0]
        probes = {"S_s": S, "small_call_s": small["none"]["ms"] * 1e-3, "small_n": 16 * N, "ctas": g}
        if rank == 0:
            probes["gamma_small"] = T.gamma_hop("none", 16, dev, ring_ctas=g)
            for key, m in (("1k", 1024), ("mid", n), ("big", 1 << 26)):
                probes["gamma_" + key] = T.gamma_hop(args.codec, max(1, m // N), dev, ring_ctas=g)
                probes["delta_" + key] = T.delta_decode(args.codec, max(1, m // N), dev)

    line = None
    if rank == 0:
        h2d = x_host.numel() * x_host.element_size() + y_host.numel() * y_host.element_size()
        line = {"metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": N, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": per_step_ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": f"synthetic (random {'x'.join(map(str, in_shape))} inputs and labels, random-init weights)",
                "config": workload_config(args, n, N),
                "e2e": {"value": e2e_value, "unit": "iters/s", "h2d_bytes_per_step": h2d * N,
                        "d2h_bytes_per_step": 4 * N,
                        "h2d_copy_ms_avg": float(np.mean(copy_ms)) if copy_ms else None,
                        "host_enqueue_ms_per_step": host_ms.get(True),
                        "streams": streams,
                        "how": "same engine; every step copies the rank's batch from pinned host memory (on a "
                               "copy stream into a per-parity buffer, overlapping the previous step's compute) "
                               "and reads its loss back into pinned memory (on a D2H stream after the step)"},
                "gpu_launches": per_iter_launches * args.steps,
                "host_enqueue_ms_per_step": host_ms.get(False),
                "roofline": roof, "kernels": kernels, "clocks": clk.summary(),
                "samples_per_s": value * args.global_batch}
        if allreduce:
            line["allreduce"] = allreduce
            big = allreduce[-1]
            wire_big = 2 * (N - 1) / N * big["n"] * w
            key = f"{args.codec}@{FULL_CTAS}ctas"
            ach = wire_big / (big[key]["ms"] * 1e-3) / 1e9
            none_key = f"none@{FULL_CTAS}ctas"
            none_gbs = (2 * (N - 1) / N * 4 * big["n"] / (big[none_key]["ms"] * 1e-3) / 1e9
                        if none_key in big else None)
            line["roofline_large_bucket"] = {
                "kernel": roof["kernel"], "n": big["n"], "bound": "nvlink", "achieved": ach,
                "peak": NVLINK_PEAK_GBS, "unit": "GB/s", "frac": ach / NVLINK_PEAK_GBS, "ctas": FULL_CTAS,
                "codec_none_busbw_gbs": none_gbs,
                "codec_none_frac": none_gbs / NVLINK_PEAK_GBS if none_gbs else None,
                "note": "the same ring kernel alone on a 256 MiB fp32 bucket with every SM (standalone "
                        "allreduce configuration); the engine runs it on %d CTAs beside the CNN" % args.ctas}
        line["timing_model"] = timing_model(avg, iso, n, N, w, allreduce, args.codec, per_step_ms, calib, probes,
                                            args.mode, args.depth, args.steps)
    return line


def stream_timeline(events, copies):
    """Per-step stream timeline of the end-to-end region from the engine's
    CUDA events: gaps on the compute stream between consecutive steps, the
    comm kernel's start relative to its step's compute end, and whether the
    batch copy was still running when the step that reads it started."""
    if not events:
        return None
    t0 = events[0][2]
    by = {}
    for (t, stage, e0, e1, _) in events:
        by.setdefault(t, {})[stage] = (t0.elapsed_time(e0), t0.elapsed_time(e1))
    steps = sorted(by)
    gaps, comm_lag, comm_ms, compute_ms = [], [], [], []
    for a_, b_ in zip(steps, steps[1:]):
        if "backward" in by[a_] and "update" in by[b_]:
            gaps.append(by[b_]["update"][0] - by[a_]["backward"][1])
    for t in steps:
        st = by[t]
        if "backward" in st:
            compute_ms.append(st["backward"][1] - st["backward"][0])
        if "allreduce" in st and "backward" in st:
            comm_lag.append(st["allreduce"][0] - st["backward"][1])
            comm_ms.append(st["allreduce"][1] - st["allreduce"][0])
    late = []
    for i, (c0, c1) in enumerate(copies[1:], start=1):  # copy i feeds step steps[i]
        if i < len(steps) and "update" in by[steps[i]]:
            late.append(t0.elapsed_time(c1) - by[steps[i]]["update"][0])
    f = lambda v: float(np.mean(v)) if v else None  # noqa: E731
    return {"compute_gap_ms_avg": f(gaps), "compute_ms_avg": f(compute_ms), "comm_ms_avg": f(comm_ms),
            "comm_start_after_compute_ms_avg": f(comm_lag),
            "copy_end_minus_step_start_ms_avg": f(late),
            "note": "events on the compute / comm streams (engine trace) and the copy stream; a positive "
                    "copy_end_minus_step_start means the copy ended after the step that reads it started "
                    "(the compute graph then waits on it)"}


def ncu_traffic():
    """dram read+write bytes per launch from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    return {k: v.get("dram_bytes_per_launch") for k, v in json.load(open(p)).items()}


def isolated_kernels(eng, codec, N, dev, reps=20):
    """Each of our kernels alone on the engine's own buffers: CUDA events on
    the launching stream around every launch, a 256 MiB read (> 126 MB L2)
    read between launches so nothing is served from L2. Returns avg ms."""
    import torch
    import torch.distributed as dist

    from paper_1811_03619_b200 import _lib
    from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait
    from paper_1811_03619_b200.compression import CodecStatus, as_codec, encode_async, roundtrip_async
    codec = as_codec(codec)
    s = torch.cuda.Stream(dev)
    flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)  # 256 MiB, read to evict L2
    n = eng.n
    w_scratch = eng.fm.params.clone()
    loc = torch.empty_like(eng.local[0])
    st = CodecStatus(dev)
    slot = eng.slots[0]
    lr = float(np.float32(1e-3))

    def timeit(fn, sync_ranks=False):
        # R x (flush) and R x (flush + kernel) back to back, so the stream
        # never idles between launches; the difference / R is the kernel's
        # own cold-L2 time without launch gaps. A ~2 ms GPU sleep ahead of
        # the first event lets the host enqueue the whole series before the
        # clock starts (a Python-side launch is slower than these kernels).
        # Cross-GPU kernels: one barrier before each series; the ring's flag
        # waits keep the ranks in lockstep from there on.
        def series(with_kernel):
            s.synchronize()
            if sync_ranks:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                flush.sum()
                torch.cuda._sleep(4_000_000)
                e0.record(s)
                for _ in range(reps):
                    flush.sum()
                    if with_kernel:
                        fn()
                e1.record(s)
            e1.synchronize()
            return e0.elapsed_time(e1)
        series(True)
        return max(0.0, (series(True) - series(False)) / reps)

    torch.cuda.synchronize(dev)
    cp_src = torch.empty(n, dtype=torch.float32, device=dev)
    cp_dst = torch.empty_like(cp_src)
    g = eng.fm.grads
    out = {
        "copy_4n": timeit(lambda: cp_dst.copy_(cp_src)),  # torch copy: 4n read + 4n write, same method
        "update": timeit(lambda: _lib.call("gp_consume_update", w_scratch.data_ptr(), int(slot.codec),
                                           slot.payload.data_ptr(), slot.status.scale_view.data_ptr(), n, lr,
                                           N, s.cuda_stream)),
    }
    if not eng.fused:
        out["compress"] = timeit(lambda: roundtrip_async(g, codec, loc, st, s.cuda_stream))
    if N == 1 or not eng.fused:
        out["recompress"] = timeit(lambda: encode_async(g, codec, slot.payload, st, s.cuda_stream))
    if N > 1:  # Eq. 5's gamma: the codec's D(C(.)) pass over the step's gradient on one GPU
        out["roundtrip"] = timeit(lambda: roundtrip_async(g, codec, loc, st, s.cuda_stream))
    if N > 1:
        if eng.fused:  # the comm stream's single kernel: D(C(g)) -> ring -> C(sum) into the slot
            out["ring"] = timeit(lambda: allreduce_into(g, eng.summed, eng.ep, codec, 0, s, precompress=True,
                                                        slot=slot.payload, slot_scale=slot.status.scale_view),
                                 sync_ranks=True)
        else:
            out["ring"] = timeit(lambda: allreduce_into(loc, eng.summed, eng.ep, codec, 0, s), sync_ranks=True)
        endpoint_wait(eng.ep, n, s)
    return out


def ring_vs_nccl(ep, codec, N, dev, sizes, ctas_list=(0,)):
    """Back-to-back allreduce of each size (device time, max over ranks):
    our ring with `codec` and with none at each CTA budget (0 = the
    engine's), and NCCL all_reduce on the same buffer."""
    import torch
    import torch.distributed as dist
    from paper_1811_03619_b200 import _lib
    from paper_1811_03619_b200.collective import allreduce_into, endpoint_wait
    out = []
    s = torch.cuda.Stream(dev)
    base = ep.info()["ctas"]
    for n in sizes:
        x = torch.randn(n, device=dev)
        y = torch.empty_like(x)
        res = {"n": n, "bytes_fp32": 4 * n}
        runs = [(c, g) for g in ctas_list for c in dict.fromkeys((codec, "none"))] + [("nccl", 0)]
        for name, g in runs:
            it = 20 if n < (1 << 24) else 8
            key = name if (g == 0 or name == "nccl") else f"{name}@{g}ctas"
            if name != "nccl":
                _lib.call("gp_comm_set_tuning", ep._comm, int(g or base), 0.0)

            def run():
                if name == "nccl":
                    with torch.cuda.stream(s):
                        dist.all_reduce(y)
                else:
                    allreduce_into(x, y, ep, name, 0, s)

            for _ in range(3):
                run()
            s.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                torch.cuda._sleep(2_000_000)  # host enqueues the series before the clock starts
            a.record(s)
            for _ in range(it):
                run()
            b.record(s)
            b.synchronize()
            ms = max_over_ranks(a.elapsed_time(b) / it, dev)
            if name != "nccl":
                endpoint_wait(ep, n, s)
            rec = {"ms": ms, "busbw_gbs": 2 * (N - 1) / N * 4 * n / (ms * 1e-3) / 1e9}
            if name != "nccl":  # wire bytes actually moved, as a fraction of the NVLink peak
                wb = {"none": 4, "trunc16": 2, "quant8": 1}[name]
                rec["wire_busbw_gbs"] = 2 * (N - 1) / N * wb * n / (ms * 1e-3) / 1e9
                rec["nvlink_frac"] = rec["wire_busbw_gbs"] / NVLINK_PEAK_GBS
            res[key] = rec
        _lib.call("gp_comm_set_tuning", ep._comm, int(base), 0.0)
        out.append(res)
    return out


def timing_model(avg, iso, n, N, w, allreduce, codec, step_ms, calib=None, probes=None, mode="pipe_sgd",
                 depth=2, steps=30):
    """The paper's timing model with GPU-measured symbols (timing.py:97-132,
    harness.py:513-720).

    * Eq. 4 (pipe) / Eq. 2 (sync) from the stage times measured inside the
      step (update, compute, in-pipeline comm) vs the measured step.
    * Eq. 5 for the ring: alpha = one-way flag latency (gp_calib_pingpong),
      beta = bidirectional peer push per byte (gp_calib_p2p_copy), gamma =
      one fused hop C(x + D(in)) on one GPU per payload byte (gp_calib_hop,
      the reference's reduce_hop), S = an all-rank GPU barrier
      (gp_comm_barrier, the reference's barrier probe); each ring size of the
      allreduce rows is compared with its Eq. 5 prediction (25 % flag).
    * compare_prediction (harness.py:687-720): the iteration predicted with
      Eq. 5's comm (predict_iteration_time, harness.py:667-684) vs measured."""
    from paper_1811_03619_b200 import timing as T
    upd = avg.get("update", 0.0) + avg.get("compress", 0.0)
    comp = avg.get("backward", 0.0)
    comm = avg.get("allreduce", 0.0)
    out = {"update_ms": upd, "compute_ms": comp, "comm_ms_in_pipeline": comm}
    stages = T.StageTimes(update=upd / 1e3, forward=0.0, backward=comp / 1e3, comm=comm / 1e3)
    out["eq4_pipe_ms"] = T.t_pipe_limited(1, stages) * 1e3
    out["eq2_sync_ms"] = T.t_sync_total(1, stages) * 1e3
    out["measured_step_ms"] = step_ms
    out["eq4_over_measured"] = out["eq4_pipe_ms"] / step_ms
    out["bound"] = "compute" if upd + comp >= comm else "communication"
    if upd + comp > 0:
        out["eq7_scaling_efficiency"] = T.scaling_efficiency(stages)  # busy / max(busy, comm), timing.py:191-200
    if not (allreduce and N > 1 and calib and probes):
        return out
    a, b, S = max(0.0, calib["alpha_s"]), calib["beta_s_per_byte"], probes["S_s"]
    fixed = T.ring_fixed_overhead(probes["small_call_s"], N, probes["small_n"], a, b, probes["gamma_small"], S)
    rows = []
    for row, key in zip(allreduce, ("1k", "mid", "big")):
        rows.append(T.compare_ring(row[codec]["ms"] * 1e-3, N, codec, row["n"], a, b, probes["gamma_" + key], S,
                                   probes["delta_" + key], fixed_s=fixed, fence_s=calib.get("phi_s", 0.0),
                                   fenced_phases=T.ring_fenced_phases(row["n"], N, probes["ctas"], codec)))
    mid = rows[1]
    gam = probes["gamma_mid"]
    cluster = T.ClusterParams(workers=N, latency_s=a, byte_time_s=b, reduce_time_s=gam, sync_time_s=S,
                              model_bytes=float(n * w))
    pred_it = T.predict_iteration_time(T.StageTimes(update=upd / 1e3, forward=0.0, backward=comp / 1e3,
                                                    comm=T.ring_comm_time(cluster)),
                                       cluster, "d_sync" if mode == "d_sync" else "pipe_sgd", steps, depth)
    rel = (step_ms * 1e-3 - pred_it) / pred_it
    out["eq5"] = {
        "symbols": {"alpha_us": a * 1e6, "beta_push_gbs": calib["push_gbs"],
                    "phi_fence_us": calib.get("phi_s", 0.0) * 1e6,
                    "gamma_gbs": 1 / gam / 1e9 if gam else None, "S_us": S * 1e6},
        "rings": rows, "step_gradient_ring": mid,
        "note": "measured = the same ring alone, back-to-back, at the engine's CTA budget (the allreduce rows); "
                "gamma is one fused hop on one GPU on that same budget; eq5_ext adds the step-0 encode, the "
                "allgather decode, the per-call fixed cost (launch, call open / close: Eq. 5's residual on a "
                "16-element-per-rank call) and the release drain of each flag-protocol phase (phi, measured by "
                "timing.calibrate_nvlink) the paper's model leaves out (timing.compare_ring)",
        "fixed_per_call_us": fixed * 1e6}
    out["compare_prediction"] = [{"mode": mode, "measured_ms": step_ms, "predicted_ms": pred_it * 1e3,
                                  "rel_error": rel, "flagged": abs(rel) > 0.25,
                                  "bound": "communication" if T.ring_comm_time(cluster) > (upd + comp) / 1e3
                                  else "compute"}]
    return out


def main():
    args = parse()
    ws, rank, local = dist_info()
    if ws != args.gpus and ws > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
    if args.impl == "reference":
        line = reference_arm(args, ws, rank)
        if line:
            print(json.dumps(line), flush=True)
        return
    import torch
    import torch.distributed as dist
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    line = our_arm(args, ws, rank, local)
    if line is not None and not args.no_cpu_baseline and ws == 1:
        n = line["config"]["params"]
        steps = 5
        v, rp, ns, t = reference_rate(n, 1, args.codec, steps, 1, seconds_per_step=args.cpu_seconds / steps)
        line["cpu_baseline"] = {"value": v, "unit": "iters/s", "cores": rp.threads, "kind": rp.kind,
                                "sample": ref_sample_text(rp, n, ns, t, steps, args.codec)}
        # the same work on both sides: our kernels' device time per step (the
        # update + the comm stream's codec / ring kernels) vs the reference's
        # CPU time per step for the identical path
        ours_ms = sum(line["kernels"][k]["in_pipeline_avg_ms"] or 0.0 for k in line["kernels"]
                      if k in ("update", "compress", "recompress", "ring"))
        line["hot_path_per_step"] = {
            "gpu_ms": ours_ms, "cpu_reference_ms": 1e3 / v, "speedup": (1e3 / v) / ours_ms if ours_ms else None,
            "what": "decode(slot t-2) + mean + SGD, whole-vector compress of the gradient, ring (identity at "
                    "p = 1), compress of the sum: our kernels' in-step device time vs the reference's CPU time"}
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
