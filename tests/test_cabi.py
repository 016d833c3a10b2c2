"""CPU checks of the drop-in boundary: libpipesgd.so loads without a GPU and
exports every symbol include/pipesgd.h declares; the Python mirror keeps
the reference's names and pure-host semantics."""

import ctypes
import os
import re

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
