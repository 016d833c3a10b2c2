"""ctypes binding of libpipesgd.so — the C ABI declared in include/pipesgd.h.

The library is built in-tree by `__graft_entry__.build()` (or
`python -m paper_1811_03619_b200.build`). There is no fallback: if the
shared object is missing every entry point raises NativeLibraryError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, NativeLibraryError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIPESGD_LIB") or os.path.join(HERE, "libpipesgd.so")

GP_OK = 0
GP_FAIL_NONFINITE, GP_FAIL_TIMEOUT, GP_FAIL_HEADER, GP_FAIL_BOUNDS = 1, 2, 3, 4
GP_PHASE_RS, GP_PHASE_AG, GP_PHASE_BARRIER = 0, 1, 2
GP_RING_PRECOMPRESS, GP_RING_SLOT_OUT = 1, 2

# Every symbol include/pipesgd.h declares (checked by tests/test_cabi.py).
EXPORTS = (
    "gp_comm_create", "gp_comm_create_emulated", "gp_comm_ipc_handle", "gp_comm_connect_ipc",
    "gp_comm_connect_local", "gp_comm_set_tuning", "gp_comm_set_trace", "gp_comm_set_iteration_source", "gp_comm_set_protocol", "gp_comm_info", "gp_comm_destroy",
    "gp_comm_set_call_counter", "gp_ring_plan",
    "gp_allreduce", "gp_allreduce_ex", "gp_allreduce_emulated", "gp_allreduce_emulated_ex",
    "gp_gather_sum", "gp_broadcast", "gp_gather_sum_emulated", "gp_broadcast_emulated",
    "gp_comm_poll_error", "gp_get_stats",
    "gp_reset_stats", "gp_encode", "gp_decode", "gp_roundtrip", "gp_consume_update", "gp_consume_update_dev",
    "gp_calib_p2p_copy", "gp_calib_p2p_copy_ex", "gp_calib_pingpong", "gp_calib_hop", "gp_comm_barrier", "gp_comm_wire_bytes", "gp_last_error_string", "gp_version",
)


class GpError(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("phase", ctypes.c_int32), ("step", ctypes.c_int32),
                ("block", ctypes.c_int32), ("rank", ctypes.c_int32), ("detail", ctypes.c_int32)]


class GpStats(ctypes.Structure):
    _fields_ = [("messages", ctypes.c_uint64), ("payload_bytes", ctypes.c_uint64),
                ("frame_bytes", ctypes.c_uint64)]


_vp, _u64, _i, _u32, _f, _d = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32,
                               ctypes.c_float, ctypes.c_double)

_SIGS = {
    "gp_comm_create": (_i, [_i, _i, _i, _u64, ctypes.POINTER(_vp)]),
    "gp_comm_create_emulated": (_i, [_i, _i, _u64, ctypes.POINTER(_vp)]),
    "gp_comm_ipc_handle": (_i, [_vp, ctypes.c_char_p]),
    "gp_comm_connect_ipc": (_i, [_vp, ctypes.c_char_p]),
    "gp_comm_connect_local": (_i, [ctypes.POINTER(_vp), _i]),
    "gp_comm_set_tuning": (_i, [_vp, _i, _d]),
    "gp_comm_set_trace": (_i, [_vp, _vp]),
    "gp_comm_set_iteration_source": (_i, [_vp, _vp]),
    "gp_comm_set_protocol": (_i, [_vp, ctypes.c_uint64]),
    "gp_comm_info": (_i, [_vp, ctypes.POINTER(ctypes.c_int64)]),
    "gp_comm_set_call_counter": (_i, [_vp, ctypes.c_uint64]),
    "gp_ring_plan": (_i, [_u64, _i, _i, _i, _i, _u64, ctypes.POINTER(ctypes.c_int64)]),
    "gp_comm_destroy": (_i, [_vp]),
    "gp_allreduce": (_i, [_vp, _vp, _vp, _u64, _i, _u32, _vp]),
    "gp_allreduce_emulated": (_i, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _u64, _i, _u32, _vp]),
    "gp_allreduce_ex": (_i, [_vp, _vp, _vp, _vp, _vp, _u64, _i, _i, _u32, _vp]),
    "gp_allreduce_emulated_ex": (_i, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                      ctypes.POINTER(_vp), _u64, _i, _i, _u32, _vp]),
    "gp_gather_sum": (_i, [_vp, _vp, _vp, _u64, _i, _i, _u32, _vp]),
    "gp_broadcast": (_i, [_vp, _vp, _vp, _u64, _i, _u32, _vp]),
    "gp_gather_sum_emulated": (_i, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _u64, _i, _i, _u32, _vp]),
    "gp_broadcast_emulated": (_i, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _u64, _i, _u32, _vp]),
    "gp_comm_poll_error": (_i, [_vp, ctypes.POINTER(GpError)]),
    "gp_get_stats": (_i, [_vp, _i, ctypes.POINTER(GpStats)]),
    "gp_reset_stats": (_i, [_vp]),
    "gp_encode": (_i, [_i, _vp, _u64, _vp, _vp, _vp]),
    "gp_decode": (_i, [_i, _vp, _vp, _u64, _vp, _vp]),
    "gp_roundtrip": (_i, [_i, _vp, _vp, _u64, _vp, _vp]),
    "gp_consume_update": (_i, [_vp, _i, _vp, _vp, _u64, _f, _i, _vp]),
    "gp_consume_update_dev": (_i, [_vp, _i, _vp, _vp, _u64, _vp, _i, _vp]),
    "gp_calib_p2p_copy": (_i, [_vp, _vp, _u64, _i, _i, _vp]),
    "gp_calib_p2p_copy_ex": (_i, [_vp, _vp, _u64, _i, _i, _u64, _vp, _vp, _vp]),
    "gp_calib_pingpong": (_i, [_vp, _vp, _i, _i, _u64, _vp, _vp]),
    "gp_calib_hop": (_i, [_i, _vp, _vp, _vp, _vp, _u64, _i, _vp, _vp]),
    "gp_comm_barrier": (_i, [_vp, _i, _vp, _vp]),
    "gp_comm_wire_bytes": (_i, [_vp, _i, _i, ctypes.POINTER(ctypes.c_uint64)]),
    "gp_last_error_string": (ctypes.c_char_p, []),
    "gp_version": (_i, []),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libpipesgd.so once (thread-safe); raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                    " (the CUDA path has no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    """GP_ERR_ARG / GP_ERR_STATE (a caller error: size over capacity, bad
    codec, misalignment, unconnected communicator) raise the reference's
    ConfigError; CUDA and platform failures raise NativeLibraryError."""
    if rc != GP_OK:
        msg = load().gp_last_error_string().decode(errors="replace")
        cls = ConfigError if rc in (1, 3) else NativeLibraryError  # GP_ERR_ARG, GP_ERR_STATE
        raise cls(f"{what} failed (code {rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
