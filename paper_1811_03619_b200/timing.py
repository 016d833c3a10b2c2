"""The paper's analytic timing model (Eqs. 2-7), plus GPU calibration.

Same names and float64 formulas as /root/reference/pkg/src/gradpipe/timing.py
(StageTimes :21-47, ClusterParams :50-85, t_sync_total Eq. 2 :97-99,
t_pipe_ideal Eq. 3 :102-106, t_pipe_limited Eq. 4 :109-116, ring_comm_time
Eq. 5 :119-132, segmented_comm_time / t_pipe_seq / t_pipe_segmented Eq. 6
:135-188, star_comm_time :155-170, scaling_efficiency Eq. 7 :191-200,
recommend_config :210-232). `calibrate_nvlink` measures the symbols on the
B200s instead of on sockets (reference calibrate(): harness.py:513-586):
alpha from a flag ping-pong, beta from a peer push copy, gamma from the
fused hop's measured time per byte.
"""

from __future__ import annotations

from dataclasses import dataclass, fields

from .errors import ConfigError

SEQUENTIAL, SEGMENTED = "sequential", "segmented"
COMPUTE_BOUND, COMM_BOUND = "compute", "communication"


def _nonneg(obj, names):
    for nm in names:
        if getattr(obj, nm) < 0:
            raise ConfigError(f"{nm} must be >= 0")


@dataclass(frozen=True)
class StageTimes:
    """Per-iteration stage durations (s); first_segment_backward <= backward."""

    update: float = 0.0
    forward: float = 0.0
    backward: float = 0.0
    first_segment_backward: float = 0.0
    comm: float = 0.0

    def __post_init__(self):
        for f in fields(self):
            if getattr(self, f.name) < 0:
                raise ConfigError(f"stage time {f.name} must be >= 0")
        if self.first_segment_backward > self.backward:
            raise ConfigError("first-segment backward time cannot exceed the full backward time")

    @property
    def compute(self) -> float:
        return self.forward + self.backward

    @property
    def busy(self) -> float:
        return self.update + self.compute


@dataclass(frozen=True)
class ClusterParams:
    """p workers; alpha (s/msg), beta (s/B), gamma_red (s/B), S (s), n (B), L segments."""

    workers: int
    latency_s: float = 0.0
    byte_time_s: float = 0.0
    reduce_time_s: float = 0.0
    sync_time_s: float = 0.0
    model_bytes: float = 0.0
    segments: int = 1

    def __post_init__(self):
        if self.workers < 1:
            raise ConfigError("need at least one worker")
        if self.segments < 1:
            raise ConfigError("need at least one gradient segment")
        _nonneg(self, ("latency_s", "byte_time_s", "reduce_time_s", "sync_time_s", "model_bytes"))


@dataclass(frozen=True)
class PipelineConfig:
    depth: int = 2
    iterations: int = 1

    def __post_init__(self):
        if self.depth < 1 or self.iterations < 1:
            raise ConfigError("pipeline depth and iteration count must be >= 1")


def t_sync_total(iterations: int, stages: StageTimes) -> float:
    """Eq. 2: every stage on the critical path each iteration."""
    return iterations * (stages.busy + stages.comm)


def t_pipe_ideal(iterations: int, depth: int, stages: StageTimes) -> float:
    """Eq. 3: unlimited resources shorten the run depth-fold."""
    if depth < 1:
        raise ConfigError("pipeline depth must be >= 1")
    return iterations / depth * (stages.busy + stages.comm)


def t_pipe_limited(iterations: int, stages: StageTimes) -> float:
    """Eq. 4: limited resources — the slower of compute and comm dominates."""
    return iterations * max(stages.busy, stages.comm)


def _ring_terms(c: ClusterParams, rounds: int):
    p = c.workers
    share = (p - 1) / p
    return (2 * (p - 1) * rounds * c.latency_s,
            2 * share * c.model_bytes * c.byte_time_s,
            share * c.model_bytes * c.reduce_time_s,
            rounds * c.sync_time_s)


def ring_comm_time(params: ClusterParams) -> float:
    """Eq. 5: 2(p-1)a + 2(p-1)/p n b + (p-1)/p n g + S."""
    if params.workers == 1:
        return params.sync_time_s
    return sum(_ring_terms(params, 1))


def segmented_comm_time(params: ClusterParams) -> float:
    """Eq. 6 comm: latency and sync terms scale with L, byte terms do not."""
    if params.workers == 1:
        return params.segments * params.sync_time_s
    return sum(_ring_terms(params, params.segments))


def star_comm_time(params: ClusterParams) -> float:
    """Parameter-server exchange: (p+1)(a + n b) + p n g + S."""
    p, n = params.workers, params.model_bytes
    if p == 1:
        return params.sync_time_s
    return (p + 1) * (params.latency_s + n * params.byte_time_s) + p * n * params.reduce_time_s + \
        params.sync_time_s


def t_pipe_seq(iterations: int, stages: StageTimes, params: ClusterParams) -> float:
    return iterations * max(stages.busy, ring_comm_time(params))


def t_pipe_segmented(iterations: int, stages: StageTimes, params: ClusterParams) -> float:
    head = stages.update + stages.forward + stages.first_segment_backward
    return iterations * max(head, segmented_comm_time(params))


def scaling_efficiency(stages: StageTimes) -> float:
    """Eq. 7: busy / max(busy, comm); 1 when communication is fully masked."""
    if stages.busy <= 0:
        raise ConfigError("scaling efficiency undefined for zero compute time")
    return stages.busy / max(stages.busy, stages.comm)


@dataclass(frozen=True)
class Recommendation:
    depth: int
    comm_mode: str
    bound: str


def recommend_config(stages: StageTimes, params: ClusterParams) -> Recommendation:
    """Depth 2 always; segment only if compute-bound and it strictly helps."""
    comm = ring_comm_time(params)
    busy = stages.busy
    bound = COMM_BOUND if comm > busy else COMPUTE_BOUND
    if params.workers == 1 or bound == COMM_BOUND:
        return Recommendation(2, SEQUENTIAL, bound)
    seg = max(stages.update + stages.forward + stages.first_segment_backward, segmented_comm_time(params))
    return Recommendation(2, SEGMENTED if seg < max(busy, comm) else SEQUENTIAL, bound)


def predict_iteration_time(stages: StageTimes, params: ClusterParams, mode: str, iterations: int,
                           depth: int = 2) -> float:
    """harness.py:667-684: d_sync = busy + comm; pipe = max(busy, comm) with
    the pipeline fill correction (T + K - 1) / T."""
    comm = ring_comm_time(params)
    if mode == "d_sync":
        return stages.busy + comm
    return max(stages.busy, comm) * (iterations + depth - 1) / iterations


def calibrate_nvlink(devices=(0, 1), nbytes: int = 1 << 30, ctas: int = 148, iters: int = 20000) -> dict:
    """alpha (one-way flag latency, s) and beta (s/byte of a bidirectional
    peer push) between two GPUs of this process, with libpipesgd's
    calibration kernels. Requires two GPUs with peer access."""
    import torch

    from . import _lib
    from .transport import GpuTransport

    tr = GpuTransport(2, devices=list(devices), max_elems=1024)
    a = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    b = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    st = [torch.cuda.Stream(device=d) for d in devices]
    ev = []
    for rep in range(2):
        for i, d in enumerate(devices):
            with torch.cuda.device(d):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st[i])
                _lib.call("gp_calib_p2p_copy", b[1 - i].data_ptr(), a[i].data_ptr(), nbytes, ctas, 0,
                          st[i].cuda_stream)
                e1.record(st[i])
                if rep == 1:
                    ev.append((e0, e1))
        for s in st:
            s.synchronize()
    beta = max(e0.elapsed_time(e1) for e0, e1 in ev) / 1e3 / nbytes
    flags = [torch.zeros(4, dtype=torch.int64, device=f"cuda:{d}") for d in devices]
    ns = [torch.zeros(1, dtype=torch.int64, device=f"cuda:{d}") for d in devices]
    for i, d in enumerate(devices):
        with torch.cuda.device(d):
            _lib.call("gp_calib_pingpong", flags[i].data_ptr(), flags[1 - i].data_ptr(), iters, int(i == 0), 0,
                      ns[i].data_ptr(), st[i].cuda_stream)
    for s in st:
        s.synchronize()
    t = ns[0].item()
    if t < 0:  # the kernel's timeout sentinel (~0): the partner never answered
        tr.close()
        raise RuntimeError("flag ping-pong timed out (is the peer GPU busy with another process?)")
    alpha = t / iters / 2 / 1e9
    phi = _fence_tail(devices, a, b, st)
    tr.close()
    return {"alpha_s": alpha, "beta_s_per_byte": beta, "push_gbs": 1 / beta / 1e9, "phi_s": phi}


def _fence_tail(devices, a, b, st, nbytes: int = 8 << 20, chunk: int = 4096, ctas: int = 148, reps: int = 20) -> float:
    """phi: what a system-scope release per chunk adds to one phase of
    pushes (the flag protocol's publish, which Eq. 5's per-hop alpha does not
    cover): both GPUs push 8 MiB to each other in 4 KiB warp chunks, with and
    without a st.release.sys flag after every chunk (gp_calib_p2p_copy_ex
    modes 6 / 2); the difference of the two, per phase."""
    import torch

    from . import _lib

    ctr = [torch.zeros(reps, dtype=torch.int64, device=f"cuda:{d}") for d in devices]
    flags = [torch.zeros(nbytes // chunk + 1, dtype=torch.int64, device=f"cuda:{d}") for d in devices]
    times = {}
    for mode in (2, 6, 2, 6):
        for c in ctr:
            c.zero_()
        for d in devices:
            torch.cuda.synchronize(d)
        ev = []
        for i, d in enumerate(devices):
            with torch.cuda.device(d):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st[i])
                for k in range(reps):
                    _lib.call("gp_calib_p2p_copy_ex", b[1 - i].data_ptr(), a[i].data_ptr(), nbytes, ctas, mode, chunk,
                              ctr[i][k:k + 1].data_ptr(), flags[1 - i].data_ptr(), st[i].cuda_stream)
                e1.record(st[i])
                ev.append((e0, e1))
        for s in st:
            s.synchronize()
        times[mode] = max(e0.elapsed_time(e1) for e0, e1 in ev) / 1e3 / reps  # the second run of each mode wins
    return max(0.0, times[6] - times[2])


def ring_fenced_phases(n: int, p: int, ctas: int, codec) -> int:
    """How many phases of a ring call end in system-scope releases (the flag
    protocol; the LL protocol has none): p - 1 reduce-scatter hops plus the
    allgather publish, or 2 for codec none's direct reduce-scatter
    (gp_ring_plan decides, as the launch does)."""
    import ctypes

    from . import _lib
    from .compression import as_codec

    if p < 2:
        return 0
    out = (ctypes.c_int64 * 5)()
    _lib.call("gp_ring_plan", int(n), int(p), int(ctas), int(as_codec(codec)), 0, int(n), out)
    if out[2]:
        return 0
    return 2 if out[4] else p


def gamma_hop(codec, n: int, device, reps: int = 10, ring_ctas: int = 0) -> float:
    """Eq. 5's gamma on this GPU: seconds per payload byte of one fused
    reduce-scatter hop out = C(x + D(in)) over an n-element block (the
    reference calibrate()'s reduce_hop, harness.py:561-568), inputs cold in L2
    (a 256 MiB read between launches, subtracted). The probe's own launch
    cost (the same hop over 16 elements) is subtracted too: the ring runs the
    hop inside its one kernel, so only the per-byte rate belongs in Eq. 5."""
    import torch

    from . import _lib
    from .compression import CodecStatus, as_codec, encode_async

    codec = as_codec(codec)
    w = codec.bytes_per_elem
    with torch.cuda.device(device):
        s = torch.cuda.Stream(device)
        x = torch.randn(n, device=device) * 1e-2
        pay = torch.empty(max(16, n * w), dtype=torch.uint8, device=device)
        out = torch.empty_like(pay)
        st_in, st = CodecStatus(torch.device(device)), CodecStatus(torch.device(device))
        flush = torch.ones(64 << 20, dtype=torch.float32, device=device)
        with torch.cuda.stream(s):
            encode_async(x, codec, pay, st_in, s.cuda_stream)

        def series(hop: bool) -> float:
            s.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                flush.sum()
                torch.cuda._sleep(2_000_000)
                a.record(s)
                for _ in range(reps):
                    flush.sum()
                    if hop:
                        _lib.call("gp_calib_hop", int(codec), x.data_ptr(), pay.data_ptr(), st_in.scale_view.data_ptr(),
                                  out.data_ptr(), n, (ring_ctas + 1) // 2, st.ptr, s.cuda_stream)
                b.record(s)
            b.synchronize()
            return a.elapsed_time(b) / 1e3

        series(True)
        t = max(0.0, (series(True) - series(False)) / reps)
    if n > 16:
        t = max(0.0, t - gamma_hop(codec, 16, device, reps, ring_ctas) * 16 * w)
    return t / max(1, n * w)


def delta_decode(codec, n: int, device, reps: int = 10) -> float:
    """Seconds per element to decode a block into fp32 (the allgather's
    receive side, which Eq. 5 has no term for), cold L2, launch cost of a
    16-element decode subtracted."""
    import torch

    from . import _lib
    from .compression import CodecStatus, as_codec, encode_async

    codec = as_codec(codec)
    w = codec.bytes_per_elem
    with torch.cuda.device(device):
        s = torch.cuda.Stream(device)
        x = torch.randn(max(n, 16), device=device)
        pay = torch.empty(max(16, x.numel() * w), dtype=torch.uint8, device=device)
        st = CodecStatus(torch.device(device))
        out = torch.empty_like(x)
        flush = torch.ones(64 << 20, dtype=torch.float32, device=device)
        with torch.cuda.stream(s):
            encode_async(x, codec, pay, st, s.cuda_stream)

        def series(m: int, dec: bool) -> float:
            s.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                flush.sum()
                torch.cuda._sleep(2_000_000)
                a.record(s)
                for _ in range(reps):
                    flush.sum()
                    if dec:
                        _lib.call("gp_decode", int(codec), pay.data_ptr(), st.scale_view.data_ptr(), m,
                                  out.data_ptr(), s.cuda_stream)
                b.record(s)
            b.synchronize()
            return a.elapsed_time(b) / 1e3

        series(n, True)
        base = series(n, False)
        t = max(0.0, (series(n, True) - base) / reps - max(0.0, (series(16, True) - base) / reps))
    return t / max(1, n)


def barrier_time(endpoint, rounds: int = 200) -> float:
    """Eq. 5's S on the GPUs: one all-to-all flag barrier over the
    communicator (gp_comm_barrier; the reference's barrier probe,
    harness.py:589-609), seconds per barrier. Every rank must call it."""
    import torch

    from . import _lib

    dev = endpoint.device
    with torch.cuda.device(dev):
        s = torch.cuda.Stream(dev)
        ns = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.call("gp_comm_barrier", endpoint._comm, 8, ns.data_ptr(), s.cuda_stream)  # warm-up
        s.synchronize()
        _lib.call("gp_comm_barrier", endpoint._comm, int(rounds), ns.data_ptr(), s.cuda_stream)
        s.synchronize()
        t = int(ns.item())
    if t < 0 or t == (1 << 64) - 1:
        raise RuntimeError("GPU barrier probe timed out")
    return t / 1e9 / rounds


def ring_fixed_overhead(measured_small_s: float, p: int, n_small: int, alpha: float, beta: float, gamma: float,
                        sync: float) -> float:
    """The per-call cost Eq. 5 has no term for -- kernel launch, call open /
    close, the first chunk's ramp -- calibrated as Eq. 5's residual on the
    smallest real call (n_small = 16 elements per rank, codec none), >= 0.
    Used only by the extended model (compare_ring eq5_ext), on every larger
    size, so no row predicts itself."""
    params = ClusterParams(workers=p, latency_s=alpha, byte_time_s=beta, reduce_time_s=gamma, sync_time_s=sync,
                           model_bytes=float(4 * n_small))
    return max(0.0, measured_small_s - ring_comm_time(params))


def compare_ring(measured_s: float, p: int, codec, n: int, alpha: float, beta: float, gamma: float, sync: float,
                 delta: float = 0.0, flag_threshold: float = 0.25, fixed_s: float = 0.0, fence_s: float = 0.0,
                 fenced_phases: int = 0) -> dict:
    """One prediction-vs-measurement row for a ring call (compare_prediction,
    harness.py:687-720, applied to Eq. 5 itself): n is the element count,
    model bytes are the codec's payload (harness.py:562).

    `eq5_ext` (an extension, not the paper's), quant8 only: Eq. 5 plus the
    two passes of the quant8 ring that overlap no transfer -- the step-0 max
    and encode of the own block before the first hop, (1/p) n_b gamma, and
    the allgather's decode of the p-1 received blocks into the fp32 output,
    (p-1)/p n delta (delta = decode time per element). For none / trunc16 the
    step-0 encode streams straight onto the link and the decode overlaps the
    owners' pushes. Every codec's eq5_ext also adds `fixed_s`, the per-call
    cost calibrated on the smallest call (ring_fixed_overhead), and, for the
    flag protocol, `fenced_phases` x `fence_s` (ring_fenced_phases; phi from
    calibrate_nvlink): the release drain that ends each phase."""
    from .compression import as_codec

    nb = float(n * as_codec(codec).bytes_per_elem)
    params = ClusterParams(workers=p, latency_s=alpha, byte_time_s=beta, reduce_time_s=gamma, sync_time_s=sync,
                           model_bytes=nb)
    lat, bw, red, syn = _ring_terms(params, 1)
    pred = ring_comm_time(params)
    q8 = as_codec(codec).name.lower() == "quant8"
    step0 = nb / p * gamma if (p > 1 and q8) else 0.0
    ag = (p - 1) / p * n * delta if q8 else 0.0
    fence = fenced_phases * fence_s
    ext = pred + step0 + ag + fixed_s + fence
    rel = (measured_s - pred) / pred if pred > 0 else float("inf")
    rel_ext = (measured_s - ext) / ext if ext > 0 else float("inf")
    return {"n": n, "codec": as_codec(codec).name.lower(), "measured_ms": measured_s * 1e3, "eq5_ms": pred * 1e3,
            "terms_us": {"latency": lat * 1e6, "bandwidth": bw * 1e6, "reduction": red * 1e6, "sync": syn * 1e6,
                         "ext_step0_encode": step0 * 1e6, "ext_allgather_decode": ag * 1e6,
                         "ext_fixed_per_call": fixed_s * 1e6, "ext_fence_drain": fence * 1e6},
            "eq5_over_measured": pred / measured_s if measured_s > 0 else None, "rel_error": rel,
            "flagged": abs(rel) > flag_threshold,
            "eq5_ext_ms": ext * 1e3, "eq5_ext_over_measured": ext / measured_s if measured_s > 0 else None,
            "ext_flagged": abs(rel_ext) > flag_threshold}
