"""CPU checks of the drop-in boundary: libpipesgd.so loads without a GPU and
exports every symbol include/pipesgd.h declares; the Python mirror keeps
the reference's names and pure-host semantics."""

import ctypes
import os
import re
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pipesgd.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(gp_\w+)\s*\(", src, re.M)))


def test_header_and_binding_agree():
    from paper_1811_03619_b200 import _lib
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_everything():
    from paper_1811_03619_b200 import _lib
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.gp_version() == 1


def test_argument_errors_need_no_gpu():
    from paper_1811_03619_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.gp_comm_create(5, 4, 0, 16, ctypes.byref(h)) == 1  # rank outside world
    assert b"outside" in lib.gp_last_error_string()
    assert lib.gp_encode(7, None, 0, None, None, None) == 1        # unknown codec


def test_reference_names_present():
    import paper_1811_03619_b200 as pkg
    for name in ("Codec", "CompressedBlock", "compress", "decompress", "wire_size", "payload_size",
                 "serialize_block", "deserialize_block", "ring_allreduce", "pipelined_allreduce",
                 "partition_blocks", "CollectiveError", "CodecError", "ConfigError"):
        assert hasattr(pkg, name), name


def test_codec_host_semantics():
    from paper_1811_03619_b200 import Codec, CodecError, wire_size, payload_size
    assert Codec.parse(" NONE ") is Codec.NONE and Codec.parse("quant8") is Codec.QUANT8
    with pytest.raises(CodecError):
        Codec.parse("topk")
    assert wire_size(Codec.TRUNC16, 1024) == 2048 + 9
    assert payload_size(Codec.QUANT8, 7) == 7


def test_partition_blocks_matches_oracle():
    from oracle.ring import partition_blocks as ref
    from paper_1811_03619_b200 import partition_blocks
    for n in (0, 1, 7, 4099, 61_100_840):
        for p in (1, 2, 3, 4, 8):
            assert partition_blocks(n, p) == ref(n, p)


def test_argument_errors_are_reported_without_a_gpu():
    """Argument validation runs before any CUDA call: GP_ERR_ARG (1), the
    thread's last-error string, and the Python mapping to ConfigError."""
    from paper_1811_03619_b200 import _lib
    from paper_1811_03619_b200.errors import ConfigError
    lib = _lib.load()
    buf = (ctypes.c_float * 8)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    cases = [
        (lambda: lib.gp_encode(7, p, 8, p, p, None), "unknown codec"),
        (lambda: lib.gp_decode(-1, p, p, 8, p, None), "unknown codec"),
        (lambda: lib.gp_consume_update(p, 0, p, None, 8, ctypes.c_float(0.1), 0, None), "worker count"),
        (lambda: lib.gp_consume_update_dev(p, 0, p, None, 8, None, 1, None), "learning-rate pointer"),
        (lambda: lib.gp_comm_set_call_counter(None, ctypes.c_uint64(0)), "null communicator"),
        (lambda: lib.gp_comm_set_call_counter(None, ctypes.c_uint64(1 << 33)), "null communicator"),
    ]
    for fn, msg in cases:
        assert fn() == 1
        assert msg in lib.gp_last_error_string().decode()
    with pytest.raises(ConfigError, match="unknown codec"):
        _lib.call("gp_encode", 9, p, 8, p, p, None)


def _plan(n, world, ctas, codec, flags=0, max_elems=None):
    from paper_1811_03619_b200 import _lib
    out = (ctypes.c_int64 * 5)()
    _lib.call("gp_ring_plan", n, world, ctas, codec, flags, max_elems or n, out)
    return {"chunk": out[0], "ctas": out[1], "ll": out[2], "nch": out[3], "direct": out[4]}


@pytest.mark.parametrize("world,codec", [(2, 0), (2, 1), (2, 2), (4, 0), (4, 1), (8, 0), (8, 2)])
def test_ll_protocol_threshold(world, codec):
    """LL iff the block payload (incl. 16 elements of slack) fits 2 MiB at
    p = 2 and 1 MiB x (p - 1) from p = 3 on, capped at the 2 MiB LL slot
    (ring.cuh:ll_payload_limit)."""
    w = (4, 2, 1)[codec]
    limit = min((2 << 20) if world == 2 else (1 << 20) * (world - 1), 2 << 20)
    n_max = world * (limit // w - 16)  # largest n whose ceil(n/p) + 16 blocks fit
    assert _plan(n_max, world, 592, codec)["ll"] == 1
    assert _plan(n_max + world, world, 592, codec)["ll"] == 0
    assert _plan(1, world, 592, codec)["ll"] == 1


def test_launch_and_chunk_plan():
    # tiny calls launch one CTA; LL calls (no flags) use short chunks so more
    # warps share a block: 128 elements for none / trunc16, 256 for small quant8
    assert _plan(8, 2, 592, 1) == {"chunk": 128, "ctas": 1, "ll": 1, "nch": 1, "direct": 0}
    pl = _plan(648_010, 4, 592, 0)  # C1 gradient, codec none, LL
    assert pl["ll"] == 1 and pl["chunk"] == 128 and pl["nch"] == 1266 and pl["ctas"] == 317
    assert _plan(65_536, 4, 592, 2)["chunk"] == 256
    # larger quant8 LL blocks keep the flag-protocol chunk (barrier arrivals per warp)
    assert _plan(1 << 20, 4, 592, 2)["chunk"] == 1024
    # C2 gradient, standalone budget: 1024-element chunks, one per warp
    pl = _plan(4_710_538, 2, 592, 1)
    assert pl["chunk"] == 1024 and pl["nch"] == 2301 and pl["ctas"] == 576 and pl["ll"] == 0
    # the engine's 256-CTA budget: bigger chunks, fewer of them, still one per warp
    pl = _plan(4_710_538, 2, 256, 1)
    assert pl["chunk"] == 3072 and pl["ctas"] == 192
    # quant8 with the fused pre-compress scans the whole vector in chunk units
    a, b = _plan(1_000_000, 4, 592, 2), _plan(1_000_000, 4, 592, 2, flags=1)
    assert b["nch"] >= 4 * a["nch"] - 4


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_direct_reduce_scatter_plan(world):
    """codec none folds D(C(.)) = identity, so from 3 ranks on the owner folds
    every rank's block after one hop (bit-identical to the ring's fold);
    compressed codecs keep the ring (their partial sums travel compressed)."""
    for codec in (0, 1, 2):
        for n in (8, 1 << 20, 61_100_840):
            assert _plan(n, world, 592, codec)["direct"] == int(codec == 0 and world >= 3)


def test_plain_c_client_compiles_links_and_runs(tmp_path):
    """include/pipesgd.h is plain C: a C11 program using it compiles with gcc,
    links against libpipesgd.so and gets plans and error codes without a GPU."""
    import shutil
    import subprocess
    from paper_1811_03619_b200 import _lib
    lib = _lib.load()._name
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "c_abi_client"
    libdir = os.path.dirname(lib)
    subprocess.run([gcc, "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_abi_client.c"), "-L", libdir, "-l:" + os.path.basename(lib),
                    "-Wl,-rpath," + libdir, "-o", str(exe)], check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "chunk=1024 ctas=576 ll=0 nch=2301" in r.stdout
    assert "errors ok" in r.stdout


def test_reference_side_ctypes_shim_binds_without_a_gpu():
    """integration/gradpipe_b200.py (the module INTEGRATION.md has the
    reference add) binds its entry points against the built library."""
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import gradpipe_b200
    L = gradpipe_b200.lib()
    for name in ("gp_comm_create", "gp_comm_connect_local", "gp_allreduce", "gp_comm_poll_error", "gp_get_stats"):
        assert getattr(L, name).restype is ctypes.c_int
