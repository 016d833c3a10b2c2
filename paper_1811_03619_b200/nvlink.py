"""NVLink byte counters read through NVML, for measured (not computed) wire
bytes of the fused ring.

The reference counts the bytes its path hands to the transport
(/root/reference/pkg/src/gradpipe/transport.py:52-61, :85-91); on B200 the
ring's stores go straight onto NVLink, so the counterpart is the NIC-side
counter: NVML's per-GPU NVLink data throughput counters
(NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, cumulative KiB of user data
over all links; _RAW_* include protocol overhead). `NvlinkCounters` snapshots
them around a region of back-to-back calls; `delta()` returns bytes.

Measurement infrastructure only (bench.py, tools/): nothing on the hot path
reads it.
"""

from __future__ import annotations

FIELDS = {  # NVML field id -> name (nvml.h NVML_FI_DEV_NVLINK_THROUGHPUT_*), values in KiB
    138: "data_tx",
    139: "data_rx",
    140: "raw_tx",
    141: "raw_rx",
}
UINT_MAX = 0xFFFFFFFF


class NvlinkCounters:
    """Cumulative NVLink TX/RX counters of one GPU (NVML device index)."""

    def __init__(self, device: int):
        import pynvml
        pynvml.nvmlInit()
        self.m = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        self.device = device
        self._base = None

    def read(self) -> dict:
        vals = self.m.nvmlDeviceGetFieldValues(self.h, [(f, UINT_MAX) for f in FIELDS])
        out = {}
        for f, v in zip(FIELDS, vals):
            if v.nvmlReturn != 0:
                continue
            out[FIELDS[f]] = int(v.value.ullVal) * 1024  # KiB -> bytes
        return out

    def start(self) -> None:
        self._base = self.read()

    def delta(self) -> dict:
        now = self.read()
        return {k: now[k] - self._base.get(k, 0) for k in now if k in (self._base or {})}


def available(device: int = 0) -> bool:
    try:
        return bool(NvlinkCounters(device).read())
    except Exception:  # noqa: BLE001 - no NVML / no NVLink: counters unavailable
        return False
