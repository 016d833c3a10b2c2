"""An SM partition for the comm stream (CUDA green contexts): the ring kernel
launched on this stream runs only on its `sms` SMs, so the pipelined ring
takes a fixed slice of the GPU instead of spreading its resident CTAs over
every SM beside the next iteration's compute (RankEngine comm_sms,
engine.default_comm_partition). Kernels of the primary context (the
forward/backward) still run on every SM. Driver API through cuda-python;
one green context + stream per (device, SM count) per process."""

from __future__ import annotations

import threading


def _check(res, what):
    """cuda-python returns (err,) or (err, value) or (err, v1, v2, ...)."""
    res = res if isinstance(res, tuple) else (res,)
    if int(res[0]) != 0:
        raise RuntimeError(f"{what} failed: {res[0]}")
    return None if len(res) == 1 else (res[1] if len(res) == 2 else res[1:])


_CONTEXTS: dict = {}
_LOCK = threading.Lock()


def green_stream(device_index: int, sms: int, priority: int = 0):
    """A new torch ExternalStream bound to a green context of `sms` SMs (the
    driver may round up to its SM granularity). Returns (stream, sm_count).
    The green context is made once per (device, SM count) and shared; every
    call gets its own stream (ranks sharing a GPU must not share one)."""
    import torch
    from cuda.bindings import driver as d

    key = (int(device_index), int(sms))
    with _LOCK:
        if key not in _CONTEXTS:
            _CONTEXTS[key] = _make_green_ctx(*key)
        gctx, count = _CONTEXTS[key]
    # out-of-range priorities are clamped by the driver, as for cuStreamCreateWithPriority
    st = _check(d.cuGreenCtxStreamCreate(gctx, d.CUstream_flags.CU_STREAM_NON_BLOCKING, int(priority)),
                "cuGreenCtxStreamCreate")
    stream = torch.cuda.ExternalStream(int(st), device=torch.device("cuda", device_index))
    return stream, count


def _make_green_ctx(device_index: int, sms: int):
    from cuda.bindings import driver as d

    _check(d.cuInit(0), "cuInit")
    dev = _check(d.cuDeviceGet(device_index), "cuDeviceGet")
    res = _check(d.cuDeviceGetDevResource(dev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource")
    out = d.cuDevSmResourceSplitByCount(1, res, 0, sms)
    if int(out[0]) != 0:
        raise RuntimeError(f"cuDevSmResourceSplitByCount failed: {out[0]}")
    groups = out[1]
    desc = _check(d.cuDevResourceGenerateDesc(groups, 1), "cuDevResourceGenerateDesc")
    gctx = _check(d.cuGreenCtxCreate(desc, dev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM),
                  "cuGreenCtxCreate")
    count = groups[0].sm.smCount if hasattr(groups[0], "sm") else sms
    return gctx, int(count)
