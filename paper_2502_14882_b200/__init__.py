"""B200-native CalibQuant decode hot path (quantize+pack, calibrated post-scaled
decode attention, KV append) behind the reference `kvq` API.

The compute lives in libkvq_b200.so (CUDA, sm_100a) behind include/kvq_capi.h; this
package is the Python mirror of the reference interface (kvq.py) plus the in-tree build
(build.py) and the multi-GPU shard driver (shard.py).
"""
from . import kvq  # noqa: F401
from .kvq import (  # noqa: F401
    BatchedCache,
    CalibrationParams,
    ChannelStats,
    ConfigError,
    CudaError,
    DomainError,
    FormatError,
    HybridKVCache,
    KernelConfig,
    PackedBuffer,
    QuantizationConfig,
    QuantizedSegment,
    QuantMode,
    calibrated_softmax_concat,
    compute_stats,
    dequantize,
    pack,
    qk_scores,
    quantize,
    unpack,
    wv_output,
)
