"""ctypes binding of the C ABI in include/emesh_b200.h (libemesh_b200.so).

The product path has no fallback: if the shared library is missing or the
CUDA driver is absent, every entry point raises. Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_2412_01152_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMESH_LIB") or os.path.join(HERE, "libemesh_b200.so")  # EMESH_LIB: build variants

# every symbol include/emesh_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = (
    "emesh_last_error", "emesh_abi_version",
    "emesh_quantize", "emesh_quantize_segments", "emesh_codec_check",
    "emesh_dequantize", "emesh_dequantize_segments",
    "emesh_encode_quant_chunk", "emesh_decode_quant_chunk",
    "emesh_pseudo_gradient", "emesh_nesterov_outer_step",
    "emesh_adamw_step", "emesh_plan_segments", "emesh_plan_tensor_segments", "emesh_ring_schedule",
    "emesh_nccl_unique_id", "emesh_engine_create", "emesh_engine_destroy",
    "emesh_engine_segments", "emesh_engine_ring_allreduce", "emesh_engine_outer_sync",
    "emesh_engine_outer_sync_host", "emesh_engine_check", "emesh_engine_payload", "emesh_engine_payload_host",
    "emesh_engine_launches", "emesh_engine_profile", "emesh_engine_profile_read", "emesh_engine_timeline", "emesh_engine_transport",
    "emesh_engine_failed_rank", "emesh_engine_set_job",
    "emesh_checkpoint_encoded_size", "emesh_checkpoint_encode", "emesh_checkpoint_decode",
    "emesh_checkpoint_probe", "emesh_checkpoint_layout", "emesh_checkpoint_write_file",
    "emesh_checkpoint_read_file", "emesh_sha256",
)

OK, ESHAPE, ENUMERIC, EDECODE, ECUDA, ENCCL, ERING, ECONFIG, EIO, ESTALE, EPROTO = range(11)


class EngineConfig(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("k", C.c_uint32),
        ("rank", C.c_uint32),
        ("pipeline_subchunks", C.c_uint32),
        ("virtual_workers", C.c_uint32),
        ("window_elems", C.c_uint64),
        ("nccl_id", C.c_void_p),
        ("device", C.c_int),
        ("transport", C.c_uint32),
        ("reduce_fp32", C.c_uint32),
        ("tensor_numel", C.c_void_p),
        ("ntensors", C.c_uint32),
        ("step_timeout_s", C.c_double),
        ("plan_epoch", C.c_uint32),
    ]


class RingOp(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("phase", C.c_int32), ("hop", C.c_int32), ("window", C.c_int32),
        ("send_chunk", C.c_int32), ("recv_chunk", C.c_int32),
        ("send_seg0", C.c_uint32), ("send_nseg", C.c_uint32), ("recv_seg0", C.c_uint32), ("recv_nseg", C.c_uint32),
        ("final_hop", C.c_int32), ("pad", C.c_int32),
    ]


class CheckpointView(C.Structure):
    """emesh_checkpoint (include/emesh_b200.h; checkpoint.hpp:19-29)."""
    _fields_ = [
        ("outer_step", C.c_uint64),
        ("ntensors", C.c_uint32),
        ("names", C.c_void_p),
        ("ranks", C.c_void_p),
        ("extents", C.c_void_p),
        ("params", C.c_void_p),
        ("retained", C.c_void_p),
        ("adam_m", C.c_void_p),
        ("adam_v", C.c_void_p),
        ("nesterov_buf", C.c_void_p),
        ("adam_step", C.c_uint64),
        ("rng_seed", C.c_uint64),
        ("data_counter", C.c_uint64),
        ("shard", C.c_uint32),
        ("config_hash", C.c_uint8 * 32),
    ]


OP_OWN, OP_XFER, OP_QUANT, OP_APPLY = range(4)
TRANSPORT_AUTO, TRANSPORT_NCCL, TRANSPORT_P2P = range(3)

_lib = None


def lib() -> C.CDLL:
    """Load libemesh_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: the CUDA extension is not built (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i32, f32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_float
    P = C.POINTER
    sig = {
        "emesh_last_error": (C.c_char_p, []),
        "emesh_abi_version": (i32, []),
        "emesh_quantize": (i32, [vp, u64, vp, vp, vp, vp]),
        "emesh_quantize_segments": (i32, [vp, P(u64), P(u64), u32, vp, vp, vp, vp]),
        "emesh_codec_check": (i32, [vp]),
        "emesh_dequantize": (i32, [vp, vp, u64, vp, vp]),
        "emesh_dequantize_segments": (i32, [vp, vp, P(u64), P(u64), u32, vp, vp]),
        "emesh_encode_quant_chunk": (u64, [vp, vp, u32, vp]),
        "emesh_decode_quant_chunk": (i32, [vp, u64, vp, vp, P(u32)]),
        "emesh_engine_failed_rank": (i32, [vp]),
        "emesh_engine_set_job": (i32, [vp, u64]),
        "emesh_pseudo_gradient": (i32, [vp, vp, vp, u64, vp]),
        "emesh_nesterov_outer_step": (i32, [vp, vp, vp, u64, f32, f32, vp]),
        "emesh_plan_segments": (u64, [u64, u32, u32, vp, vp]),
        "emesh_adamw_step": (i32, [vp, vp, vp, vp, u64, u64] + [C.c_float] * 6 + [vp, vp]),
        "emesh_plan_tensor_segments": (u64, [vp, u32, u32, u32, vp, vp]),
        "emesh_ring_schedule": (u64, [u64, u32, u32, u64, u32, vp, u64]),
        "emesh_nccl_unique_id": (i32, [vp]),
        "emesh_engine_create": (i32, [P(EngineConfig), P(vp)]),
        "emesh_engine_destroy": (i32, [vp]),
        "emesh_engine_segments": (u64, [vp, vp, vp]),
        "emesh_engine_ring_allreduce": (i32, [vp, P(vp), P(vp), vp]),
        "emesh_engine_outer_sync": (i32, [vp, P(vp), P(vp), P(vp), f32, f32, i32, vp]),
        "emesh_engine_outer_sync_host": (i32, [vp, P(vp), P(vp), P(vp), f32, f32, i32]),
        "emesh_engine_check": (i32, [vp]),
        "emesh_engine_payload": (i32, [vp, u32, P(vp), P(vp), P(vp), P(u64)]),
        "emesh_engine_payload_host": (i32, [vp, u32, vp, vp, vp]),
        "emesh_engine_launches": (u64, [vp]),
        "emesh_engine_profile": (i32, [vp, i32]),
        "emesh_engine_profile_read": (i32, [vp, u32, P(u64), P(C.c_double), P(C.c_double)]),
        "emesh_engine_timeline": (u64, [vp, P(C.c_double), u64]),
        "emesh_engine_transport": (i32, [vp]),
        "emesh_checkpoint_encoded_size": (i32, [P(CheckpointView), P(u64)]),
        "emesh_checkpoint_encode": (i32, [P(CheckpointView), vp, u64, P(u64), vp]),
        "emesh_checkpoint_decode": (i32, [vp, u64, P(CheckpointView), vp]),
        "emesh_checkpoint_probe": (i32, [vp, u64, P(u32), P(u64), P(u64), P(u32)]),
        "emesh_checkpoint_layout": (i32, [vp, u64, vp, u64, vp, vp, u32]),
        "emesh_checkpoint_write_file": (i32, [C.c_char_p, P(CheckpointView), vp]),
        "emesh_checkpoint_read_file": (i32, [C.c_char_p, P(CheckpointView), vp]),
        "emesh_sha256": (i32, [vp, u64, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def last_error() -> str:
    return lib().emesh_last_error().decode(errors="replace")


def ptr_array(ptrs):
    return (C.c_void_p * len(ptrs))(*ptrs)
