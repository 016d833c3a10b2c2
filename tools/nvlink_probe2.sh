#!/bin/bash
# Other NVLink byte-counter sources than NVML field values (which answer
# NVML_ERROR_NOT_SUPPORTED on this pool, profiles/r02_nvlink/): the legacy
# utilization counters and nvidia-smi's own nvlink views.
cd "$(dirname "$0")/.."
python - <<'PY'
import pynvml as m
m.nvmlInit()
h = m.nvmlDeviceGetHandleByIndex(0)
for link in range(2):
    for fn in ("nvmlDeviceGetNvLinkState", "nvmlDeviceGetNvLinkVersion"):
        try:
            print(fn, link, getattr(m, fn)(h, link))
        except Exception as e:
            print(fn, link, "ERR", e)
    for c in range(2):
        try:
            print("util", link, c, m.nvmlDeviceGetNvLinkUtilizationCounter(h, link, c))
        except Exception as e:
            print("util", link, c, "ERR", e)
PY
nvidia-smi nvlink -s -i 0 2>&1 | head -8
nvidia-smi nvlink -gt d -i 0 2>&1 | head -8
nvidia-smi nvlink -gt r -i 0 2>&1 | head -4
