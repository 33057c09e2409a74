"""emesh_b200 — B200-native DiLoCo outer-synchronisation hot path.

pseudo-gradient -> int8 (uint8-codebook) ring reduce-scatter/all-gather with
per-hop dequantize + fp32 accumulate + requantize -> Nesterov outer update
fused with the final dequantize, as sm_100a kernels behind a C ABI
(include/emesh_b200.h). `emesh` mirrors the reference's C++ API
(proj/include/emesh) for this path.
"""
from . import emesh  # noqa: F401
from .emesh import (  # noqa: F401
    ConfigError, DecodeError, Error, FatalError, HyperParams, ModelParams, NesterovState, NumericError,
    QuantChunk, ReduceJob, ReduceMode, ReduceOptions, RingEngine, RingFailureError, RingPlan, ShapeError,
    StalePlanError,
    compute_pseudo_gradient, decode_quant_chunk, dequantize, dequantize_into, encode_quant_chunk,
    nesterov_outer_step, quantize, quantize_segments, codec_check, ring_allreduce, segment_table,
    MeshState, RetryResult, allreduce_with_retry, plan_tensor_segments, AdamWState, adamw_step,
    Checkpoint, encode_checkpoint, decode_checkpoint, checkpoint_layout, write_checkpoint_file,
    read_checkpoint_file, sha256,
)

__all__ = [n for n in dir() if not n.startswith("_")]
