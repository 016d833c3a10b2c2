"""Print the box facts the design depends on (GPU count, SMs, P2P, host CPUs)."""
import json
import os
import subprocess

import torch

info = {"gpus": torch.cuda.device_count(), "cpu_count": os.cpu_count()}
try:
    info["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    pass
devs = []
for i in range(info["gpus"]):
    pr = torch.cuda.get_device_properties(i)
    devs.append({"name": pr.name, "sms": pr.multi_processor_count, "mem_gb": round(pr.total_memory / 2**30, 1),
                 "l2_mb": getattr(pr, "L2_cache_size", 0) / 2**20})
info["devices"] = devs
info["p2p"] = [[torch.cuda.can_device_access_peer(i, j) if i != j else None for j in range(info["gpus"])]
               for i in range(info["gpus"])]
print(json.dumps(info))
try:
    print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
except Exception as e:
    print(e)
