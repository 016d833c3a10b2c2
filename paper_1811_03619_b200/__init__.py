"""B200-native Pipe-SGD communication hot path (arXiv 1811.03619).

Drop-in for the ring/codec/engine path of the reference package `gradpipe`
(/root/reference/pkg/src/gradpipe): the same public names, backed by
hand-written sm_100a CUDA kernels in libpipesgd.so (C ABI: include/pipesgd.h).
"""

import os as _os

for _var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    _os.environ.setdefault(_var, "1")

from .compression import (  # noqa: E402
    Codec,
    CompressedBlock,
    compress,
    decompress,
    deserialize_block,
    payload_size,
    serialize_block,
    wire_size,
)
from .collective import (  # noqa: E402
    broadcast_from_root,
    gather_to_root,
    partition_blocks,
    pipelined_allreduce,
    ring_allreduce,
)
from .errors import (  # noqa: E402
    CodecError,
    CollectiveError,
    ConfigError,
    CorruptBlockError,
    EngineError,
    GradPipeError,
    NativeLibraryError,
    TransportError,
)
from .transport import (  # noqa: E402
    EmulatedTransport,
    GpuEndpoint,
    GpuTransport,
    ProcessGroupTransport,
    TrafficStats,
)

__version__ = "0.1.0"
