"""torchrun helper for tests: run_process_worker (one rank per GPU) with
oracle gradients must reproduce the oracle trajectory bit for bit."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import engine as OE  # noqa: E402
from paper_1811_03619_b200.engine import RunConfig, run_process_worker  # noqa: E402
from paper_1811_03619_b200.models import ModelSpec  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, p = dist.get_rank(), dist.get_world_size()
data = OE.synthetic_blobs(dim=8, num_classes=3, num_samples=512, seed=1)
net = OE.Net("mlp", (8, 16, 12, 3))
out = {}
for codec in (0, 1, 2):
    for mode in ("d_sync", "pipe_sgd"):
        rng = np.random.default_rng([7, rank])
        shard = data.shard(rank, p)

        def grad_fn(r, t, params):
            b = OE.sample_from_shard(shard, 16, rng)
            return OE.loss_and_grad(params.cpu().numpy(), net, data, b)

        cfg = RunConfig(mode=mode, iterations=7, learning_rate=0.1, codec=codec, batch_size=16, seed=7)
        res = run_process_worker(cfg, data, ModelSpec("mlp", (8, 16, 12, 3)), grad_fn=grad_fn)
        want = OE.run_trajectory(p, OE.Config(mode=mode, iterations=7, learning_rate=0.1, codec=codec,
                                              batch_size=16, seed=7), data, net).params
        out[f"{mode}_{codec}"] = bool(res.params.tobytes() == want.tobytes())
        if mode == "pipe_sgd":  # the comm stream in a 16-SM green context (engine.default_comm_partition's path)
            rng = np.random.default_rng([7, rank])
            res = run_process_worker(cfg, data, ModelSpec("mlp", (8, 16, 12, 3)), grad_fn=grad_fn, comm_sms=16,
                                     comm_ctas=64)
            out[f"{mode}_{codec}_partition"] = bool(res.params.tobytes() == want.tobytes())
if rank == 0:
    print(json.dumps(out))
dist.barrier()
dist.destroy_process_group()
