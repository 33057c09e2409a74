"""Python mirror of the reference's `emesh` API for the outer-sync hot path.

Same names, argument meaning and error behaviour as the C++ reference
(proj/include/emesh/{quant,optim,allreduce,tensor,errors}.hpp), backed by
the sm_100a kernels in libemesh_b200.so through the C ABI
(include/emesh_b200.h). Tensors are CUDA ``torch.Tensor`` s — torch is the
device-memory / stream plumbing, never the compute path. There is no CPU
fallback: without the built library or a GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _capi

# ---------------------------------------------------------------- errors.hpp:10-73


class Error(RuntimeError):
    """emesh::Error"""


class ShapeError(Error):
    """emesh::ShapeError"""


class NumericError(Error):
    """emesh::NumericError"""


class DecodeError(Error):
    """emesh::DecodeError"""


class ConfigError(Error):
    """emesh::ConfigError"""


class RingFailureError(Error):
    """emesh::RingFailureError (errors.hpp): ``failed_node`` names the culprit when known."""

    def __init__(self, msg: str = "", failed_node: str = ""):
        super().__init__(msg)
        self.failed_node = failed_node


class StalePlanError(Error):
    """emesh::StalePlanError: a ring peer runs a newer plan epoch (allreduce.hpp:272)."""


class FatalError(Error):
    """emesh::FatalError"""


class CudaError(FatalError):
    pass


class NcclError(RingFailureError):
    pass


_ERRS = {
    _capi.ESHAPE: ShapeError, _capi.ENUMERIC: NumericError, _capi.EDECODE: DecodeError,
    _capi.ECUDA: CudaError, _capi.ENCCL: NcclError, _capi.ERING: RingFailureError,
    _capi.ECONFIG: ConfigError, _capi.EIO: Error, _capi.ESTALE: StalePlanError, _capi.EPROTO: Error,
}


def _check(rc: int) -> None:
    if rc != _capi.OK:
        raise _ERRS.get(rc, Error)(_capi.last_error())


def _stream(stream=None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dev_f32(t: torch.Tensor, what: str) -> torch.Tensor:
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ShapeError(f"{what}: expected a contiguous CUDA float32 tensor")
    return t


def _aligned_empty(n: int, dtype, device) -> torch.Tensor:
    """Fresh allocations are 512-B aligned by the caching allocator; pad by 32
    so the quantizer's 32-byte octet reads of the last slot stay inside the allocation."""
    itemsize = torch.empty((), dtype=dtype).element_size()
    pad = max(1, 32 // itemsize)
    return torch.empty(n + pad, dtype=dtype, device=device)[:n]


# ---------------------------------------------------------------- quant.hpp:19-131

BUCKETS = 256


@dataclass
class QuantChunk:
    """quant.hpp:19-26 — ``codebook`` (256 f32, nondecreasing) + ``indices`` (u8)."""

    codebook: torch.Tensor
    indices: torch.Tensor
    stats: Optional[torch.Tensor] = None  # {mu, sigma, lo, width} (fp64), diagnostic

    def count(self) -> int:
        return int(self.indices.numel())


def quantize(values: torch.Tensor, stream=None) -> QuantChunk:
    """quant.hpp:28 ``quantize(std::span<const float>)``. Raises ShapeError on
    an empty chunk, NumericError on non-finite input (synchronous, like the
    reference)."""
    _dev_f32(values, "quantize")
    n = values.numel()
    if n == 0:
        raise ShapeError("quantize: empty chunk")
    if values.data_ptr() % 32:  # the quantizer reads 32-byte octets
        values = values.clone()
    dev = values.device
    codes = _aligned_empty(n, torch.uint8, dev)
    cb = torch.empty(BUCKETS, dtype=torch.float32, device=dev)
    st = torch.empty(4, dtype=torch.float64, device=dev)
    _check(_capi.lib().emesh_quantize(values.data_ptr(), n, codes.data_ptr(), cb.data_ptr(), st.data_ptr(),
                                      _stream(stream)))
    return QuantChunk(cb, codes, st)


def quantize_segments(values: torch.Tensor, seg_lo: Sequence[int], seg_len: Sequence[int], stream=None):
    """Batched quantize over a segment table (allreduce.hpp:326-336): returns
    (codes [n], codebooks [nseg,256], stats [nseg,4]). Asynchronous; call
    ``codec_check()`` for the NumericError of a non-finite segment."""
    _dev_f32(values, "quantize_segments")
    lo = np.ascontiguousarray(seg_lo, np.uint64)
    ln = np.ascontiguousarray(seg_len, np.uint64)
    if np.any(ln == 0):
        raise ShapeError("quantize: empty chunk")
    dev = values.device
    codes = _aligned_empty(values.numel(), torch.uint8, dev)
    cbs = torch.empty((len(lo), BUCKETS), dtype=torch.float32, device=dev)
    st = torch.empty((len(lo), 4), dtype=torch.float64, device=dev)
    P = C.POINTER(C.c_uint64)
    _check(_capi.lib().emesh_quantize_segments(values.data_ptr(), lo.ctypes.data_as(P), ln.ctypes.data_as(P), len(lo),
                                               codes.data_ptr(), cbs.data_ptr(), st.data_ptr(), _stream(stream)))
    return codes, cbs, st


def codec_check(stream=None) -> None:
    _check(_capi.lib().emesh_codec_check(_stream(stream)))


def dequantize_into(chunk: QuantChunk, out: torch.Tensor, stream=None) -> None:
    """quant.hpp:89 ``dequantize_into``."""
    _dev_f32(out, "dequantize")
    if out.numel() != chunk.count():
        raise ShapeError("dequantize: output size mismatch")
    if chunk.codebook.numel() != BUCKETS:
        raise ShapeError("dequantize: malformed codebook")
    if chunk.count() == 0:
        return
    codes = chunk.indices
    if codes.data_ptr() % 4 or out.data_ptr() % 16:
        tmp = _aligned_empty(out.numel(), torch.float32, out.device)
        c2 = _aligned_empty(codes.numel(), torch.uint8, out.device)
        c2.copy_(codes)
        _check(_capi.lib().emesh_dequantize(c2.data_ptr(), chunk.codebook.data_ptr(), chunk.count(), tmp.data_ptr(),
                                            _stream(stream)))
        out.copy_(tmp)
        return
    _check(_capi.lib().emesh_dequantize(codes.data_ptr(), chunk.codebook.contiguous().data_ptr(), chunk.count(),
                                        out.data_ptr(), _stream(stream)))


def dequantize(chunk: QuantChunk, stream=None) -> torch.Tensor:
    """quant.hpp:96 ``dequantize``."""
    out = _aligned_empty(chunk.count(), torch.float32, chunk.indices.device)
    dequantize_into(chunk, out, stream)
    return out


def encode_quant_chunk(chunk: QuantChunk) -> bytes:
    """quant.hpp:102-115 wire layout: u32 LE count, 256 f32 LE, count u8."""
    if chunk.codebook.numel() != BUCKETS:
        raise ShapeError("encode_quant_chunk: malformed codebook")
    codes = np.ascontiguousarray(chunk.indices.cpu().numpy(), np.uint8)
    cb = np.ascontiguousarray(chunk.codebook.cpu().numpy(), np.float32)
    out = np.empty(4 + 4 * BUCKETS + len(codes), np.uint8)
    n = _capi.lib().emesh_encode_quant_chunk(codes.ctypes.data, cb.ctypes.data, len(codes), out.ctypes.data)
    return out[:n].tobytes()


def decode_quant_chunk(buf: bytes, device="cuda") -> QuantChunk:
    """quant.hpp:117-131; raises DecodeError like the reference."""
    b = np.frombuffer(bytes(buf), np.uint8)
    codes = np.empty(max(len(b), 1), np.uint8)
    cb = np.empty(BUCKETS, np.float32)
    cnt = C.c_uint32(0)
    _check(_capi.lib().emesh_decode_quant_chunk(b.ctypes.data if len(b) else None, len(b), codes.ctypes.data,
                                                cb.ctypes.data, C.byref(cnt)))
    return QuantChunk(torch.from_numpy(cb).to(device), torch.from_numpy(codes[: cnt.value].copy()).to(device))


# ---------------------------------------------------------------- tensor.hpp:54-109


class ModelParams:
    """tensor.hpp:54-109, B200 layout: ONE flat fp32 arena in HBM in canonical
    order with per-tensor views, so ``flatten()`` is free (trainer.hpp:356)."""

    def __init__(self, shapes: Dict[str, Sequence[int]] | List, device="cuda", arena: Optional[torch.Tensor] = None):
        items = list(shapes.items()) if isinstance(shapes, dict) else list(shapes)
        self.names = [nm for nm, _ in items]
        if len(set(self.names)) != len(self.names):
            raise ShapeError("duplicate parameter name")
        self.shapes = [tuple(int(e) for e in sh) for _, sh in items]
        for sh in self.shapes:
            if any(e == 0 for e in sh):
                raise ShapeError("zero extent in tensor shape")
        self.sizes = [int(np.prod(sh)) if sh else 1 for sh in self.shapes]
        n = sum(self.sizes)
        self.arena = arena if arena is not None else _aligned_empty(n, torch.float32, device).zero_()
        if self.arena.numel() != n:
            raise ShapeError("flat buffer size mismatch")

    def element_count(self) -> int:
        return self.arena.numel()

    def same_shapes(self, other: "ModelParams") -> bool:
        return self.names == other.names and self.shapes == other.shapes

    def entries(self):
        off = 0
        for nm, sh, sz in zip(self.names, self.shapes, self.sizes):
            yield nm, self.arena[off: off + sz].view(sh)
            off += sz

    def at(self, name: str) -> torch.Tensor:
        for nm, t in self.entries():
            if nm == name:
                return t
        raise ShapeError(f"no parameter named {name}")

    def flatten(self) -> torch.Tensor:
        return self.arena

    def unflatten(self, flat: torch.Tensor) -> None:
        if flat.numel() != self.element_count():
            raise ShapeError("flat buffer size mismatch")
        if flat.data_ptr() != self.arena.data_ptr():
            self.arena.copy_(flat)

    def zeros_like(self) -> "ModelParams":
        return ModelParams(list(zip(self.names, self.shapes)), device=self.arena.device)

    def clone(self) -> "ModelParams":
        p = self.zeros_like()
        p.arena.copy_(self.arena)
        return p


# ---------------------------------------------------------------- optim.hpp:12-132


@dataclass
class HyperParams:
    """optim.hpp:12-33 (outer fields are the ones this path uses)."""

    inner_lr: float = 7.5e-5
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1
    outer_lr: float = 0.7
    outer_momentum: float = 0.9
    warmup_steps: int = 1000
    total_steps: int = 10000
    cooldown_fraction: float = 0.2

    def validate(self) -> None:
        if not (0.0 <= self.beta1 < 1.0):
            raise ConfigError("beta1 must be in [0,1)")
        if not (0.0 <= self.beta2 < 1.0):
            raise ConfigError("beta2 must be in [0,1)")
        if not self.inner_lr > 0.0:
            raise ConfigError("inner_lr must be > 0")
        if not self.outer_lr > 0.0:
            raise ConfigError("outer_lr must be > 0")
        if not (0.0 <= self.cooldown_fraction < 1.0):
            raise ConfigError("cooldown_fraction must be in [0,1)")
        if self.total_steps < 1:
            raise ConfigError("total_steps must be >= 1")


@dataclass
class NesterovState:
    """optim.hpp:48-56"""

    buffer: ModelParams

    @staticmethod
    def zeros_like(params: ModelParams) -> "NesterovState":
        return NesterovState(params.zeros_like())


@dataclass
class AdamWState:
    """optim.hpp:35-46"""

    step: int
    m: ModelParams
    v: ModelParams

    @staticmethod
    def zeros_like(params: ModelParams) -> "AdamWState":
        return AdamWState(0, params.zeros_like(), params.zeros_like())


# ---------------------------------------------------------------- checkpoint.hpp:19-68,190-224


@dataclass
class Checkpoint:
    """checkpoint.hpp:19-29. The five parameter sets are device ModelParams
    (flat HBM arenas); (de)serialization moves them straight between HBM and
    the canonical bytes (include/emesh_b200.h, emesh_checkpoint_*)."""

    outer_step: int
    params: ModelParams
    retained: ModelParams
    inner: AdamWState
    outer: NesterovState
    rng_seed: int = 0
    data_counter: int = 0
    shard: int = 0
    config_hash: bytes = bytes(32)

    @staticmethod
    def zeros_like(params: ModelParams) -> "Checkpoint":
        return Checkpoint(0, params.zeros_like(), params.zeros_like(), AdamWState.zeros_like(params),
                          NesterovState.zeros_like(params))


def _ck_view(ck: Checkpoint):
    sets = (ck.params, ck.retained, ck.inner.m, ck.inner.v, ck.outer.buffer)
    for other in sets[1:]:
        if not sets[0].same_shapes(other):
            raise ShapeError("checkpoint tensor shapes inconsistent")
    p = sets[0]
    names = [nm.encode() for nm in p.names]
    c_names = (C.c_char_p * max(len(names), 1))(*names)
    ranks = (C.c_uint32 * max(len(p.shapes), 1))(*[len(sh) for sh in p.shapes])
    ext = [e for sh in p.shapes for e in sh]
    c_ext = (C.c_uint32 * max(len(ext), 1))(*ext)
    v = _capi.CheckpointView()
    v.outer_step, v.ntensors = ck.outer_step, len(names)
    v.names, v.ranks, v.extents = C.cast(c_names, C.c_void_p), C.cast(ranks, C.c_void_p), C.cast(c_ext, C.c_void_p)
    v.params, v.retained, v.adam_m, v.adam_v, v.nesterov_buf = (s_.arena.data_ptr() for s_ in sets)
    v.adam_step, v.rng_seed, v.data_counter, v.shard = ck.inner.step, ck.rng_seed, ck.data_counter, ck.shard
    if len(ck.config_hash) != 32:
        raise ShapeError("config_hash must be 32 bytes")
    v.config_hash[:] = list(ck.config_hash)
    return v, (c_names, ranks, c_ext)  # keep the arrays alive with the view


def _ck_scalars_back(ck: Checkpoint, v) -> None:
    ck.outer_step, ck.inner.step, ck.rng_seed = int(v.outer_step), int(v.adam_step), int(v.rng_seed)
    ck.data_counter, ck.shard, ck.config_hash = int(v.data_counter), int(v.shard), bytes(v.config_hash)


def encode_checkpoint(ck: Checkpoint, stream=None) -> bytes:
    """checkpoint.hpp:32-47, straight from the device arenas."""
    v, keep = _ck_view(ck)
    n = C.c_uint64()
    _check(_capi.lib().emesh_checkpoint_encoded_size(C.byref(v), C.byref(n)))
    out = C.create_string_buffer(n.value)
    _check(_capi.lib().emesh_checkpoint_encode(C.byref(v), C.addressof(out), n.value, C.byref(n), _stream(stream)))
    return out.raw


def checkpoint_layout(buf: bytes) -> List:
    """The (name, shape) list a checkpoint's bytes hold (its params set)."""
    L = _capi.lib()
    nt, numel, nb, rs = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint32()
    _check(L.emesh_checkpoint_probe(buf, len(buf), C.byref(nt), C.byref(numel), C.byref(nb), C.byref(rs)))
    names = C.create_string_buffer(max(nb.value, 1))
    ranks = (C.c_uint32 * max(nt.value, 1))()
    ext = (C.c_uint32 * max(rs.value, 1))()
    _check(L.emesh_checkpoint_layout(buf, len(buf), names, nb.value, ranks, ext, rs.value))
    out, at, e = [], 0, 0
    raw = names.raw
    for i in range(nt.value):
        end = raw.index(b"\0", at)
        out.append((raw[at:end].decode(), tuple(ext[e: e + ranks[i]])))
        at, e = end + 1, e + ranks[i]
    return out


def decode_checkpoint(buf: bytes, like: Optional[ModelParams] = None, device="cuda", stream=None) -> Checkpoint:
    """checkpoint.hpp:49-66 into device arenas shaped like ``like`` (else
    the layout the bytes hold); raises DecodeError / ShapeError like the
    reference."""
    if like is None:
        like = ModelParams(checkpoint_layout(buf), device=device)
    ck = Checkpoint.zeros_like(like)
    v, keep = _ck_view(ck)
    _check(_capi.lib().emesh_checkpoint_decode(buf, len(buf), C.byref(v), _stream(stream)))
    _ck_scalars_back(ck, v)
    return ck


def write_checkpoint_file(path: str, ck: Checkpoint, stream=None) -> None:
    """checkpoint.hpp:190-203 (length + sha256 head, payload streamed from HBM)."""
    v, keep = _ck_view(ck)
    _check(_capi.lib().emesh_checkpoint_write_file(os.fsencode(path), C.byref(v), _stream(stream)))


def read_checkpoint_file(path: str, like: Optional[ModelParams] = None, device="cuda", stream=None) -> Checkpoint:
    """checkpoint.hpp:205-224: Error on a missing file / hash mismatch,
    DecodeError on truncation, then decode_checkpoint."""
    if like is None:
        try:
            with open(path, "rb") as f:
                body = f.read()[40:]
        except OSError as e:
            raise Error(f"cannot read checkpoint file {path}") from e
        like = ModelParams(checkpoint_layout(body), device=device)
    ck = Checkpoint.zeros_like(like)
    v, keep = _ck_view(ck)
    _check(_capi.lib().emesh_checkpoint_read_file(os.fsencode(path), C.byref(v), _stream(stream)))
    _ck_scalars_back(ck, v)
    return ck


def sha256(data: bytes) -> bytes:
    """sha256.hpp Sha256::hash (host)."""
    out = (C.c_uint8 * 32)()
    _check(_capi.lib().emesh_sha256(data, len(data), out))
    return bytes(out)


def adamw_step(params: ModelParams, grads: ModelParams, state: AdamWState, hp: HyperParams, lr_scale: float,
               stream=None) -> None:
    """optim.hpp:63-94 — one AdamW step on the device arenas (bit-exact fp32),
    the inner step whose result becomes theta_l for the next outer sync."""
    if not params.same_shapes(grads):
        raise ShapeError("adamw_step: params/grads shape mismatch")
    if not params.same_shapes(state.m) or not params.same_shapes(state.v):
        raise ShapeError("adamw_step: optimizer state shape mismatch")
    if not (0.0 <= lr_scale <= 1.0):
        raise ConfigError("lr_scale must be in [0,1]")
    state.step += 1
    err = torch.zeros(1, dtype=torch.int32, device=params.arena.device)
    _check(_capi.lib().emesh_adamw_step(params.arena.data_ptr(), grads.arena.data_ptr(), state.m.arena.data_ptr(),
                                        state.v.arena.data_ptr(), params.element_count(), state.step, hp.inner_lr,
                                        lr_scale, hp.beta1, hp.beta2, hp.eps, hp.weight_decay, err.data_ptr(),
                                        _stream(stream)))
    if int(err.item()):
        raise NumericError("non-finite gradient")


def compute_pseudo_gradient(theta_prev: ModelParams, theta_local: ModelParams, stream=None) -> ModelParams:
    """optim.hpp:99 — delta = theta_prev - theta_local (fp32, canonical order)."""
    if not theta_prev.same_shapes(theta_local):
        raise ShapeError("compute_pseudo_gradient: shape mismatch")
    delta = theta_prev.zeros_like()
    _check(_capi.lib().emesh_pseudo_gradient(theta_prev.arena.data_ptr(), theta_local.arena.data_ptr(),
                                             delta.arena.data_ptr(), delta.element_count(), _stream(stream)))
    return delta


def nesterov_outer_step(params: ModelParams, avg_delta: ModelParams, state: NesterovState, hp: HyperParams,
                        stream=None) -> None:
    """optim.hpp:116 — b = mu*b + d; theta -= lr*(d + mu*b), in place."""
    if not params.same_shapes(avg_delta):
        raise ShapeError("nesterov_outer_step: shape mismatch")
    if not params.same_shapes(state.buffer):
        raise ShapeError("nesterov_outer_step: momentum buffer shape mismatch")
    _check(_capi.lib().emesh_nesterov_outer_step(params.arena.data_ptr(), avg_delta.arena.data_ptr(),
                                                 state.buffer.arena.data_ptr(), params.element_count(),
                                                 hp.outer_lr, hp.outer_momentum, _stream(stream)))


# ---------------------------------------------------------------- allreduce.hpp:21-62


class ReduceMode(enum.IntEnum):
    fp32 = 0
    int8 = 1


@dataclass
class RingPlan:
    """allreduce.hpp:25-45 (NVSwitch is uniform: ring order = rank order)."""

    job_id: int = 0
    epoch: int = 0
    order: List[str] = field(default_factory=list)
    self_index: int = 0

    @staticmethod
    def from_mesh(mesh: "MeshState", self_id: str, job_id: int) -> "RingPlan":
        """allreduce.hpp:31-44."""
        if self_id not in mesh.ring:
            raise ShapeError(f"node {self_id} is not in the ring")
        return RingPlan(job_id, int(mesh.epoch), list(mesh.ring), mesh.ring.index(self_id))


@dataclass
class MeshState:
    """The part of the reference's MeshState (mesh.hpp) the ring consumes: the
    membership epoch and the ring order of the current members."""

    epoch: int
    ring: List[str]


@dataclass
class RetryResult:
    """allreduce.hpp:477-482."""

    value: torch.Tensor
    participants: int = 0
    attempts: int = 0  # failures survived
    epoch: int = 0


@dataclass
class ReduceJob:
    """allreduce.hpp:49-53 — the input is preserved for retries."""

    id: int
    input: torch.Tensor
    mode: ReduceMode = ReduceMode.int8


@dataclass
class ReduceOptions:
    """allreduce.hpp:55-62; pipeline_subchunks defines the segmentation."""

    pipeline_subchunks: int = 4
    pipelined: bool = True
    codec_sec_per_element: float = 0.0
    step_timeout: float = 30.0
    max_retries: int = 5
    evict_wait: float = 20.0


def segment_table(n: int, k: int, S: int):
    """allreduce.hpp:107-118 + :326-336, chunk-major: list of (lo, len)."""
    out = []
    base, rem = divmod(n, k)
    off = 0
    for c in range(k):
        ln = base + (1 if c < rem else 0)
        ns = 1 if ln == 0 else min(S, ln)
        b2, r2 = divmod(ln, ns)
        o2 = off
        for j in range(ns):
            l2 = b2 + (1 if j < r2 else 0)
            out.append((o2, l2))
            o2 += l2
        off += ln
    return out


def plan_segments(n: int, k: int, S: int):
    """Segment table from the C++ planner (host-only, no GPU)."""
    cnt = _capi.lib().emesh_plan_segments(n, k, S, None, None)
    lo = np.empty(cnt, np.uint64)
    ln = np.empty(cnt, np.uint64)
    _capi.lib().emesh_plan_segments(n, k, S, lo.ctypes.data, ln.ctypes.data)
    return lo, ln


def plan_tensor_segments(sizes, k: int, S: int):
    """Segment table of a multi-tensor engine (one ReduceJob per tensor; host-only)."""
    sz = np.ascontiguousarray(np.asarray(sizes, dtype=np.uint64))
    cnt = _capi.lib().emesh_plan_tensor_segments(sz.ctypes.data, len(sz), k, S, None, None)
    lo = np.empty(cnt, np.uint64)
    ln = np.empty(cnt, np.uint64)
    _capi.lib().emesh_plan_tensor_segments(sz.ctypes.data, len(sz), k, S, lo.ctypes.data, ln.ctypes.data)
    return lo, ln


def ring_schedule(n: int, k: int, S: int, rank: int, window_elems: int = 0):
    """The NCCL engine's program for one ring position (host-only, no GPU)."""
    cnt = _capi.lib().emesh_ring_schedule(n, k, S, window_elems, rank, None, 0)
    ops = (_capi.RingOp * max(cnt, 1))()
    _capi.lib().emesh_ring_schedule(n, k, S, window_elems, rank, ops, cnt)
    return [ops[i] for i in range(cnt)]


class RingEngine:
    """One ring position (NCCL mode: ``rank`` of ``k`` processes, one GPU each)
    or all ``k`` DiLoCo workers on this GPU (``virtual=True``). Owns every
    device buffer the round needs; nothing is allocated per round."""

    def __init__(self, n: int, k: int, rank: int = 0, opts: Optional[ReduceOptions] = None, virtual: bool = False,
                 nccl_id: Optional[bytes] = None, window_elems: int = 0, device: Optional[int] = None,
                 transport: str = "auto", mode: "ReduceMode" = None, tensor_sizes: Optional[Sequence[int]] = None,
                 plan: Optional["RingPlan"] = None):
        opts = opts or ReduceOptions()
        # RingPlan (allreduce.hpp:25-45): its epoch goes into every payload's ChunkMsg header; its
        # order names the culprit of a failed round (RingFailureError.failed_node)
        self.plan = plan
        if opts.pipeline_subchunks < 1:
            raise ConfigError("pipeline_subchunks must be >= 1")
        self.n, self.k, self.rank = int(n), int(k), int(rank)
        self.S = int(opts.pipeline_subchunks)
        self.virtual = bool(virtual) or k == 1
        self.workers = k if (virtual and k > 1) else 1
        self._idbuf = None
        cfg = _capi.EngineConfig()
        cfg.n, cfg.k, cfg.rank = self.n, self.k, self.rank
        cfg.pipeline_subchunks = self.S
        cfg.virtual_workers = k if (virtual and k > 1) else 0
        cfg.window_elems = int(window_elems)
        tmap = {"auto": _capi.TRANSPORT_AUTO, "nccl": _capi.TRANSPORT_NCCL, "p2p": _capi.TRANSPORT_P2P}
        if transport not in tmap:
            raise ConfigError(f"transport must be one of {sorted(tmap)}")
        cfg.transport = tmap[transport]
        self.mode = ReduceMode.int8 if mode is None else ReduceMode(mode)
        cfg.reduce_fp32 = 1 if self.mode == ReduceMode.fp32 else 0
        cfg.step_timeout_s = float(opts.step_timeout)
        cfg.plan_epoch = int(plan.epoch) if plan is not None else 0
        self._sizes = None
        if tensor_sizes is not None:  # one ReduceJob per tensor (config 5)
            self._sizes = np.ascontiguousarray(np.asarray(tensor_sizes, dtype=np.uint64))
            cfg.tensor_numel = self._sizes.ctypes.data
            cfg.ntensors = len(self._sizes)
        if nccl_id is not None:
            self._idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_id = C.cast(self._idbuf, C.c_void_p)
        cfg.device = torch.cuda.current_device() if device is None else int(device)
        h = C.c_void_p()
        _check(_capi.lib().emesh_engine_create(C.byref(cfg), C.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_capi.lib().emesh_nccl_unique_id(buf))
        return buf.raw

    def close(self) -> None:
        if getattr(self, "_h", None):
            _capi.lib().emesh_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def transport(self) -> str:
        """The resolved transport: "p2p", "nccl", or "local" (virtual ring / k == 1)."""
        return {1: "nccl", 2: "p2p"}.get(_capi.lib().emesh_engine_transport(self._h), "local")

    def segments(self):
        cnt = _capi.lib().emesh_engine_segments(self._h, None, None)
        lo = np.empty(cnt, np.uint64)
        ln = np.empty(cnt, np.uint64)
        _capi.lib().emesh_engine_segments(self._h, lo.ctypes.data, ln.ctypes.data)
        return lo, ln

    def launches(self) -> int:
        return int(_capi.lib().emesh_engine_launches(self._h))

    PROFILE_KINDS = ("reserved0", "reserved1", "quant_pg", "quant_hop", "quant_final", "quant_plain",
                     "dequant_nesterov", "dequantize", "fused_pg_nesterov_k1", "f32_hop", "f32_apply")

    def profile(self, enable: bool = True) -> None:
        """Per-kernel CUDA-event timing on the engine's launching stream."""
        _check(_capi.lib().emesh_engine_profile(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        out = {}
        for i, name in enumerate(self.PROFILE_KINDS):
            c, ms, by = C.c_uint64(), C.c_double(), C.c_double()
            _check(_capi.lib().emesh_engine_profile_read(self._h, i, C.byref(c), C.byref(ms), C.byref(by)))
            if c.value:
                out[name] = {"launches": c.value, "ms": ms.value, "alg_bytes": by.value}
        return out

    def timeline(self, max_rows: int = 1 << 16):
        """NCCL-mode op timeline since profile(True): list of
        (kind, phase, hop, window, start_ms, end_ms); kind in OP_* of _capi."""
        import numpy as np
        buf = np.zeros((max_rows, 6), dtype=np.float64)
        m = _capi.lib().emesh_engine_timeline(self._h, buf.ctypes.data_as(C.POINTER(C.c_double)), max_rows)
        return [tuple(r) for r in buf[:min(m, max_rows)]]

    def _ptrs(self, ts: Sequence[torch.Tensor], what: str):
        if len(ts) != self.workers:
            raise ShapeError(f"{what}: expected {self.workers} worker tensors")
        for t in ts:
            _dev_f32(t, what)
            if t.numel() != self.n:
                raise ShapeError(f"{what}: flat buffer size mismatch")
        return _capi.ptr_array([t.data_ptr() for t in ts])

    def ring_allreduce(self, inputs: Sequence[torch.Tensor], outputs: Sequence[torch.Tensor], stream=None) -> None:
        """allreduce.hpp:314 in this engine's ReduceMode, stream-ordered."""
        self._rc(_capi.lib().emesh_engine_ring_allreduce(self._h, self._ptrs(inputs, "input"),
                                                       self._ptrs(outputs, "output"), _stream(stream)))

    def outer_sync(self, theta_g: Sequence[torch.Tensor], theta_l: Sequence[torch.Tensor],
                   momentum: Sequence[torch.Tensor], hp: Optional[HyperParams] = None, write_local: bool = True,
                   stream=None) -> None:
        """trainer.hpp:355-382: PG -> ring all-reduce (this engine's ReduceMode) -> Nesterov, in place."""
        hp = hp or HyperParams()
        self._rc(_capi.lib().emesh_engine_outer_sync(self._h, self._ptrs(theta_g, "theta_g"),
                                                   self._ptrs(theta_l, "theta_l"), self._ptrs(momentum, "momentum"),
                                                   hp.outer_lr, hp.outer_momentum, 1 if write_local else 0,
                                                   _stream(stream)))

    def outer_sync_host(self, theta_g, theta_l, momentum, hp: Optional[HyperParams] = None,
                        write_local: bool = True) -> None:
        """Same round on HOST (ideally pinned) buffers: H2D, round, D2H."""
        hp = hp or HyperParams()

        def ptrs(ts):
            if len(ts) != self.workers:
                raise ShapeError("expected one host tensor per local worker")
            for t in ts:
                if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != self.n:
                    raise ShapeError("host buffers must be contiguous CPU float32 of length n")
            return _capi.ptr_array([t.data_ptr() for t in ts])

        self._rc(_capi.lib().emesh_engine_outer_sync_host(self._h, ptrs(theta_g), ptrs(theta_l), ptrs(momentum),
                                                        hp.outer_lr, hp.outer_momentum, 1 if write_local else 0))

    def _rc(self, rc: int) -> None:
        """_check, with the culprit of a failed round (emesh_engine_failed_rank) as
        RingFailureError.failed_node (allreduce.hpp:466-470)."""
        if rc == _capi.ERING:
            who = int(_capi.lib().emesh_engine_failed_rank(self._h))
            node = ""
            if who >= 0:
                node = self.plan.order[who] if self.plan is not None and who < len(self.plan.order) else str(who)
            raise RingFailureError(_capi.last_error(), failed_node=node)
        _check(rc)

    def check(self) -> None:
        """Synchronize; raise NumericError if any quantize saw non-finite data, RingFailureError
        (with failed_node) / StalePlanError if the round failed (then nothing was committed)."""
        self._rc(_capi.lib().emesh_engine_check(self._h))

    def set_job(self, job_id: int) -> None:
        """ReduceJob.id of the next round (the ChunkMsg job id every payload carries)."""
        _check(_capi.lib().emesh_engine_set_job(self._h, int(job_id)))

    def payload(self, worker: int = 0):
        """Host copies (codes u8[n], codebooks f32[nseg,256], stats f64[nseg,4]
        = {mu, sigma, lo, width}) of a local worker's final payload arena."""
        nseg = len(self.segments()[0])
        codes = np.empty(max(self.n, 1), np.uint8)
        cbs = np.empty((nseg, BUCKETS), np.float32)
        stats = np.empty((nseg, 4), np.float64)
        _check(_capi.lib().emesh_engine_payload_host(self._h, worker, codes.ctypes.data, cbs.ctypes.data,
                                                     stats.ctypes.data))
        return codes[: self.n], cbs, stats


def allreduce_with_retry(make_engine, mesh, mesh_state: MeshState, self_id: str, job: ReduceJob,
                         opts: Optional[ReduceOptions] = None) -> RetryResult:
    """allreduce.hpp:485-518 over GPU engines. ``make_engine(plan)`` builds the
    engine of one membership epoch (the caller exchanges the NCCL id among
    ``plan.order``; build it with ``ReduceOptions(step_timeout=...)`` so a peer
    that stops makes the round fail instead of hang); ``mesh`` is the
    membership service (the reference's MeshClient): ``report_failure(node)``,
    ``wait_epoch_change(epoch, timeout) -> MeshState`` (may raise TimeoutError)
    and ``fetch_mesh() -> MeshState``. A failed round (RingFailureError: a peer
    timed out, NCCL failed) is retried over the survivors from the preserved
    ``job.input``; the result is the mean over the final plan's participants."""
    opts = opts or ReduceOptions()
    failures = 0
    while True:
        if self_id not in mesh_state.ring:
            raise FatalError("this node is no longer in the mesh")
        if len(mesh_state.ring) < 1:
            raise FatalError("no participants left")
        plan = RingPlan.from_mesh(mesh_state, self_id, job.id)
        eng = None
        try:
            eng = make_engine(plan)
            value = ring_allreduce(eng, job, opts)
            eng.check()
            return RetryResult(value, len(plan.order), failures, int(mesh_state.epoch))
        except RingFailureError as rf:
            failures += 1
            if failures > opts.max_retries:
                raise FatalError(f"all-reduce retries exhausted: {rf}") from rf
            failed = getattr(rf, "failed_node", "")
            if failed and failed != self_id:
                mesh.report_failure(failed)
            try:
                mesh_state = mesh.wait_epoch_change(mesh_state.epoch, opts.evict_wait)
            except TimeoutError:
                mesh_state = mesh.fetch_mesh()  # maybe it changed and we missed it
        except StalePlanError as sp:  # allreduce.hpp:512-515: this node's plan is behind
            failures += 1
            if failures > opts.max_retries:
                raise FatalError("all-reduce retries exhausted") from sp
            mesh_state = mesh.fetch_mesh()
        finally:
            if eng is not None and hasattr(eng, "close"):
                eng.close()


def ring_allreduce(engine: RingEngine, job: ReduceJob, opts: Optional[ReduceOptions] = None,
                   stream=None) -> torch.Tensor:
    """allreduce.hpp:314 ``ring_allreduce`` for this process's ring position:
    returns the mean every rank decodes; ``job.input`` is untouched."""
    if ReduceMode(job.mode) != engine.mode:
        raise ConfigError(f"job mode {ReduceMode(job.mode).name} != engine mode {engine.mode.name} (one engine per mode)")
    out = _aligned_empty(engine.n, torch.float32, job.input.device)
    engine.ring_allreduce([job.input], [out], stream)
    return out
