"""An SM partition for the comm stream (CUDA green contexts): the ring kernel
launched on this stream runs only on its `sms` SMs, so the pipelined ring
takes a fixed slice of the GPU instead of spreading its resident CTAs over
every SM beside the next iteration's compute. Experimental (bench knob
BENCH_COMM_SMS); driver API through cuda-python."""

from __future__ import annotations


def _check(res, what):
    err = res[0] if isinstance(res, tuple) else res
    if int(err) != 0:
        raise RuntimeError(f"{what} failed: {err}")
    return res[1:] if isinstance(res, tuple) and len(res) > 2 else (res[1] if isinstance(res, tuple) else None)


def green_stream(device_index: int, sms: int):
    """A torch ExternalStream bound to a green context of `sms` SMs (the
    driver may round up to its SM granularity). Returns (stream, sm_count)."""
    import torch
    from cuda.bindings import driver as d

    _check(d.cuInit(0), "cuInit")
    dev = _check(d.cuDeviceGet(device_index), "cuDeviceGet")
    res = _check(d.cuDeviceGetDevResource(dev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource")
    out = d.cuDevSmResourceSplitByCount(1, res, 0, sms)
    if int(out[0]) != 0:
        raise RuntimeError(f"cuDevSmResourceSplitByCount failed: {out[0]}")
    groups, n_groups = out[1], out[2]
    desc = _check(d.cuDevResourceGenerateDesc(groups, 1), "cuDevResourceGenerateDesc")
    gctx = _check(d.cuGreenCtxCreate(desc, dev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM),
                  "cuGreenCtxCreate")
    st = _check(d.cuGreenCtxStreamCreate(gctx, d.CUstream_flags.CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate")
    count = groups[0].sm.smCount if hasattr(groups[0], "sm") else sms
    stream = torch.cuda.ExternalStream(int(st), device=torch.device("cuda", device_index))
    stream._green_ctx = gctx  # keep alive
    return stream, int(count)
