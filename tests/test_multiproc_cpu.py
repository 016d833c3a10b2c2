"""World-size-2 host-side tests on CPU (gloo): the N>1 plumbing that does
not need a GPU — IPC-handle exchange/validation of ProcessGroupTransport,
bench.py's max-over-ranks timing, and the torchrun contract of
`bench.py --impl reference` (rank 0 prints one JSON line, others exit 0)."""

import json
import os
import socket
import subprocess
import sys

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, globals()[fn_name](rank, world)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _exchange_ok(rank, world):
    from paper_1811_03619_b200.transport import exchange_handles
    blob = exchange_handles(bytes([rank]) * 64, 1 << 20, device=rank)
    return blob == b"".join(bytes([r]) * 64 for r in range(world))


def _exchange_bad_capacity(rank, world):
    from paper_1811_03619_b200.transport import exchange_handles
    try:
        exchange_handles(bytes(64), 1000 + rank, device=rank)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__
    return "no error"


def _exchange_same_device(rank, world):
    from paper_1811_03619_b200.transport import exchange_handles
    try:
        exchange_handles(bytes(64), 10, device=0)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__
    return "no error"


def _exchange_bad_ctas(rank, world):
    from paper_1811_03619_b200.transport import exchange_handles
    try:
        exchange_handles(bytes(64), 10, device=rank, ctas=16 + rank)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__
    return "no error"


def _max_over_ranks(rank, world):
    import bench
    return bench.max_over_ranks(1.5 + rank)


def test_ipc_handle_exchange_gloo():
    assert _run("_exchange_ok") == {0: True, 1: True}


def test_ipc_handle_exchange_rejects_mismatched_geometry():
    assert _run("_exchange_bad_capacity") == {0: "ConfigError", 1: "ConfigError"}
    assert _run("_exchange_same_device") == {0: "ConfigError", 1: "ConfigError"}
    assert _run("_exchange_bad_ctas") == {0: "ConfigError", 1: "ConfigError"}


def test_bench_max_over_ranks_gloo():
    assert _run("_max_over_ranks") == {0: 2.5, 1: 2.5}


def test_reference_arm_under_torchrun_two_ranks():
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--model", "c1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    # the real reference when baseline/_ref holds it, else the oracle port
    want_kind = "reference" if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "gradpipe")) else "port"
    assert d["cpu_baseline"]["kind"] == want_kind and d["e2e"]["h2d_bytes_per_step"] == 0
    # the driver's JSON line contract (bench.py docstring / task contract)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert "workload" in d["config"]
    assert set(d["cpu_baseline"]) >= {"value", "unit", "cores", "kind", "sample"}
    assert d["cpu_baseline"]["cores"] == 2  # one thread per simulated rank
    assert set(d["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
