"""Is NVLS multicast available on this box? Device attribute, and torch's
symmetric memory multicast pointer under torchrun (2 ranks)."""
import os

import torch
import torch.distributed as dist

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
from cuda.bindings import driver as d  # noqa: E402
d.cuInit(0)
err, dev = d.cuDeviceGet(local)
err, mc = d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print(f"rank {dist.get_rank()}: CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED={mc} (err {err})", flush=True)
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1 << 20, device=f"cuda:{local}")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print(f"rank {dist.get_rank()}: symm mem multicast_ptr={getattr(h, 'multicast_ptr', None)} "
          f"buffer_ptrs={len(h.buffer_ptrs)}", flush=True)
except Exception as e:  # noqa: BLE001
    print(f"rank {dist.get_rank()}: symmetric memory failed: {e!r}", flush=True)
x = torch.ones(1 << 24, device="cuda")
dist.all_reduce(x)
torch.cuda.synchronize()
dist.destroy_process_group()
