"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

* ``Oracle``   — oracle/liboracle.so, the plain-C restatement of the reference
  path (oracle/emesh_oracle.c; each function cites the reference file:line).
* ``Reference`` — oracle/_ref/libemesh_ref.so, the UNMODIFIED reference
  headers compiled by oracle/Makefile (extern "C" shims in ref_wrap.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference legs may import this module, and only as the checker / the
baseline being timed — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libemesh_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")

OK, ESHAPE, ENUMERIC, EDECODE = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: error code {code}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle). The reference half needs
    /root/reference (this container); the GPU box only uses prebuilt files."""
    targets = ["all"] if ref and os.path.isdir("/root/reference/proj/include") else [ORACLE_SO]
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _ptr_array(arrs):
    return (C.POINTER(C.c_float) * len(arrs))(*[a.ctypes.data_as(C.POINTER(C.c_float)) for a in arrs])


class Oracle:
    """The plain-C restatement (oracle/emesh_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.orc_rng_word.restype = C.c_uint64
        L.orc_rng_word.argtypes = [C.c_uint64] * 4
        L.orc_rng_uniform.restype = C.c_float
        L.orc_rng_uniform.argtypes = [C.c_uint64] * 4
        L.orc_fill_uniform.argtypes = [_f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float]
        L.orc_segment_table.restype = C.c_uint64
        L.orc_segment_table.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
        L.orc_quantize.restype = C.c_int
        L.orc_quantize.argtypes = [_f32p, C.c_uint64, _u8p, _f32p, _f64p]
        L.orc_dequantize.argtypes = [_u8p, _f32p, C.c_uint64, _f32p]
        L.orc_boundary_margin.restype = C.c_double
        L.orc_boundary_margin.argtypes = [_f32p, C.c_uint64, C.c_double, C.c_double, C.c_double]
        L.orc_pseudo_gradient.argtypes = [_f32p, _f32p, C.c_uint64, _f32p]
        L.orc_nesterov.argtypes = [_f32p, _f32p, _f32p, C.c_uint64, C.c_float, C.c_float]
        L.orc_adamw.restype = C.c_int
        L.orc_adamw.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_uint64, C.c_uint64] + [C.c_float] * 6
        L.orc_ring_allreduce.restype = C.c_int
        L.orc_ring_allreduce.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int,
                                         _f32p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_outer_sync.restype = C.c_int
        L.orc_outer_sync.argtypes = [_f32p, C.c_void_p, _f32p, C.c_uint32, C.c_uint64, C.c_uint32,
                                     C.c_int, C.c_float, C.c_float]
        L.orc_segment_chain.restype = C.c_int
        L.orc_segment_chain.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_encode_quant_chunk.restype = C.c_uint64
        L.orc_encode_quant_chunk.argtypes = [_u8p, _f32p, C.c_uint32, _u8p]
        L.orc_decode_quant_chunk.restype = C.c_int
        L.orc_decode_quant_chunk.argtypes = [_u8p, C.c_uint64, _u8p, _f32p, C.POINTER(C.c_uint32)]
        self.L = L

    # -- rng.hpp
    def rng_word(self, seed, stream, counter, index):
        return self.L.orc_rng_word(seed, stream, counter, index)

    def uniform(self, n, seed, stream=0, counter=0, first=0, scale=1.0):
        out = np.empty(n, np.float32)
        self.L.orc_fill_uniform(out, n, seed, stream, counter, first, scale)
        return out

    # -- allreduce.hpp:107-118,326-336
    def segment_table(self, n, k, S):
        cnt = self.L.orc_segment_table(n, k, S, None, None)
        lo = np.empty(cnt, np.uint64)
        ln = np.empty(cnt, np.uint64)
        self.L.orc_segment_table(n, k, S, lo.ctypes.data, ln.ctypes.data)
        return lo, ln

    # -- quant.hpp
    def quantize(self, x):
        x = np.ascontiguousarray(x, np.float32)
        codes = np.empty(max(len(x), 1), np.uint8)
        cb = np.empty(256, np.float32)
        st = np.empty(4, np.float64)
        rc = self.L.orc_quantize(x, len(x), codes, cb, st)
        if rc:
            raise OracleError(rc, "quantize")
        return codes[: len(x)], cb, st

    def dequantize(self, codes, cb):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.empty(len(codes), np.float32)
        self.L.orc_dequantize(codes, np.ascontiguousarray(cb, np.float32), len(codes), out)
        return out

    def boundary_margin(self, x, stats):
        mu, sigma, lo, width = stats
        return self.L.orc_boundary_margin(np.ascontiguousarray(x, np.float32), len(x), lo, width, mu + 6.0 * sigma)

    # -- optim.hpp
    def pseudo_gradient(self, prev, local):
        out = np.empty_like(prev)
        self.L.orc_pseudo_gradient(prev, local, len(prev), out)
        return out

    def nesterov(self, theta, avg, buf, lr=0.7, momentum=0.9):
        theta = theta.copy()
        buf = buf.copy()
        self.L.orc_nesterov(theta, np.ascontiguousarray(avg, np.float32), buf, len(theta), lr, momentum)
        return theta, buf

    def adamw(self, p, g, m, v, step, inner_lr=7.5e-5, lr_scale=1.0, beta1=0.9, beta2=0.95, eps=1e-8,
              weight_decay=0.1):
        """optim.hpp:63-94; `step` = the state's step after the increment. Returns (p, m, v)."""
        p, m, v = (np.array(a, np.float32, copy=True) for a in (p, m, v))
        rc = self.L.orc_adamw(p, np.ascontiguousarray(g, np.float32), m, v, len(p), step, inner_lr, lr_scale,
                              beta1, beta2, eps, weight_decay)
        if rc:
            raise OracleError(rc, "orc adamw")
        return p, m, v

    # -- allreduce.hpp:314-473 (transport-free)
    def ring_allreduce(self, inputs, S=4, mode="int8", with_payloads=False):
        inputs = [np.ascontiguousarray(a, np.float32) for a in inputs]
        k, n = len(inputs), len(inputs[0])
        out = np.empty(max(n, 1), np.float32)
        codes = cbs = stats = None
        if with_payloads:
            nseg = len(self.segment_table(n, k, S)[0])
            codes = np.zeros(max(n, 1), np.uint8)
            cbs = np.zeros((nseg, 256), np.float32)
            stats = np.zeros((nseg, 4), np.float64)
        rc = self.L.orc_ring_allreduce(_ptr_array(inputs), k, n, S, 1 if mode == "int8" else 0, out,
                                       codes.ctypes.data if with_payloads else None,
                                       cbs.ctypes.data if with_payloads else None,
                                       stats.ctypes.data if with_payloads else None)
        if rc:
            raise OracleError(rc, "ring_allreduce")
        if with_payloads:
            return out[:n], codes[:n], cbs, stats
        return out[:n]

    def segment_chain(self, theta_g, theta_ls, chunk, mode="int8", want_mean=False):
        """One segment's reduce-scatter chain (emesh_oracle.c:orc_segment_chain): theta_g (or None: theta_ls
        are the ring inputs) and every worker's slice of the segment; chunk = the segment's ring chunk.
        Returns (codes, cb, stats, mean-or-None) of the owner's final payload."""
        k = len(theta_ls)
        ls = [np.ascontiguousarray(a, np.float32) for a in theta_ls]
        n = len(ls[0])
        g = None if theta_g is None else np.ascontiguousarray(theta_g, np.float32)
        codes = np.empty(max(n, 1), np.uint8)
        cb = np.zeros(256, np.float32)
        st = np.zeros(4, np.float64)
        mean = np.empty(max(n, 1), np.float32) if want_mean or mode != "int8" else None
        arr = _ptr_array(ls)
        rc = self.L.orc_segment_chain(None if g is None else g.ctypes.data, C.cast(arr, C.c_void_p), k, chunk, n,
                                      1 if mode == "int8" else 0, codes.ctypes.data, cb.ctypes.data, st.ctypes.data,
                                      None if mean is None else mean.ctypes.data)
        if rc:
            raise OracleError(rc, "segment_chain")
        return codes[:n], cb, st, (mean[:n] if mean is not None else None)

    def segment_chains(self, jobs, threads=None, want_mean=False):
        """Many independent segment chains in parallel (ctypes releases the GIL): jobs = iterable of
        (theta_g_slice | None, [theta_l slices], chunk). Returns the results in order."""
        from concurrent.futures import ThreadPoolExecutor
        threads = threads or max(1, min(64, os.cpu_count() or 1))
        with ThreadPoolExecutor(threads) as ex:
            return list(ex.map(lambda j: self.segment_chain(j[0], j[1], j[2], want_mean=want_mean), jobs))

    def outer_sync(self, theta_g, theta_ls, buf, S=4, mode="int8", lr=0.7, momentum=0.9):
        theta_g = np.array(theta_g, np.float32, copy=True)
        buf = np.array(buf, np.float32, copy=True)
        ls = [np.ascontiguousarray(a, np.float32) for a in theta_ls]
        rc = self.L.orc_outer_sync(theta_g, _ptr_array(ls), buf, len(ls), len(theta_g), S,
                                   1 if mode == "int8" else 0, lr, momentum)
        if rc:
            raise OracleError(rc, "outer_sync")
        return theta_g, buf

    # -- quant.hpp:102-131
    def encode_quant_chunk(self, codes, cb):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.empty(4 + 1024 + len(codes), np.uint8)
        n = self.L.orc_encode_quant_chunk(codes if len(codes) else np.zeros(1, np.uint8),
                                          np.ascontiguousarray(cb, np.float32), len(codes), out)
        return out[:n]

    def decode_quant_chunk(self, buf):
        buf = np.ascontiguousarray(buf, np.uint8)
        codes = np.empty(max(len(buf), 1), np.uint8)
        cb = np.empty(256, np.float32)
        cnt = C.c_uint32(0)
        rc = self.L.orc_decode_quant_chunk(buf if len(buf) else np.zeros(1, np.uint8), len(buf), codes, cb, C.byref(cnt))
        if rc:
            raise OracleError(rc, "decode_quant_chunk")
        return codes[: cnt.value], cb



# ---- checkpoint byte format: a pure-Python restatement (byte packing) ----

def checkpoint_encode(layout, sets, outer_step, adam_step, rng_seed, data_counter, shard, config_hash):
    """checkpoint.hpp:32-47 encode_checkpoint over write_params / write_tensor
    (tensor.hpp:115-120,144-147; ByteWriter LE, bytes.hpp:20-45). layout =
    [(name, shape)], sets = 5 flat fp32 arrays (params, retained, inner.m,
    inner.v, outer.buffer)."""
    import struct
    out = bytearray()

    def params(flat):
        out.extend(struct.pack("<I", len(layout)))
        off = 0
        for name, shape in layout:
            nb = name.encode()
            out.extend(struct.pack("<I", len(nb)) + nb + struct.pack("<I", len(shape)))
            for e in shape:
                out.extend(struct.pack("<I", e))
            n = int(np.prod(shape)) if len(shape) else 1
            out.extend(np.ascontiguousarray(flat[off: off + n], "<f4").tobytes())
            off += n

    out.extend(struct.pack("<Q", outer_step))
    params(sets[0])
    params(sets[1])
    out.extend(struct.pack("<Q", adam_step))
    params(sets[2])
    params(sets[3])
    params(sets[4])
    out.extend(struct.pack("<QQI", rng_seed, data_counter, shard))
    out.extend(bytes(config_hash))
    return bytes(out)


def checkpoint_file_bytes(payload):
    """checkpoint.hpp:190-203: u64 LE length, sha256(payload), payload."""
    import hashlib
    import struct
    return struct.pack("<Q", len(payload)) + hashlib.sha256(payload).digest() + payload


class Reference:
    """The unmodified reference library (oracle/_ref/libemesh_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        L.ref_quantize.restype = C.c_int
        L.ref_quantize.argtypes = [_f32p, C.c_uint64, _u8p, _f32p]
        L.ref_dequantize.restype = C.c_int
        L.ref_dequantize.argtypes = [_u8p, _f32p, C.c_uint64, _f32p]
        L.ref_encode_quant_chunk.restype = C.c_int
        L.ref_encode_quant_chunk.argtypes = [_u8p, _f32p, C.c_uint64, _u8p, C.POINTER(C.c_uint64)]
        L.ref_decode_quant_chunk.restype = C.c_int
        L.ref_decode_quant_chunk.argtypes = [_u8p, C.c_uint64, _u8p, _f32p, C.POINTER(C.c_uint64)]
        L.ref_pseudo_gradient.restype = C.c_int
        L.ref_pseudo_gradient.argtypes = [_f32p, _f32p, C.c_uint64, _f32p]
        L.ref_nesterov.restype = C.c_int
        L.ref_nesterov.argtypes = [_f32p, _f32p, _f32p, C.c_uint64, C.c_float, C.c_float]
        L.ref_adamw.restype = C.c_int
        L.ref_adamw.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_uint64, C.c_uint64] + [C.c_float] * 6
        L.ref_ring_allreduce_sim.restype = C.c_int
        L.ref_ring_allreduce_sim.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, C.c_int,
                                             _f32p, _u64p]
        L.ref_outer_sync_tcp.restype = C.c_int
        L.ref_outer_sync_tcp.argtypes = [_f32p, C.c_void_p, _f32p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int,
                                         C.c_float, C.c_float, _f64p]
        vp, u64 = C.c_void_p, C.c_uint64
        L.ref_encode_checkpoint.restype = C.c_int
        L.ref_encode_checkpoint.argtypes = [u64, C.c_uint32, vp, vp, vp, vp, u64, u64, u64, C.c_uint32, vp, vp, u64,
                                            C.POINTER(u64)]
        L.ref_decode_checkpoint.restype = C.c_int
        L.ref_decode_checkpoint.argtypes = [vp, u64, vp, u64, vp, vp, vp, u64]
        L.ref_write_checkpoint_file.restype = C.c_int
        L.ref_write_checkpoint_file.argtypes = [C.c_char_p, u64, C.c_uint32, vp, vp, vp, vp, u64, u64, u64,
                                                C.c_uint32, vp]
        L.ref_read_checkpoint_file.restype = C.c_int
        L.ref_read_checkpoint_file.argtypes = [C.c_char_p, vp, u64, vp, vp, vp, u64]
        L.ref_sha256.restype = C.c_int
        L.ref_sha256.argtypes = [vp, u64, vp]
        self.L = L

    def quantize(self, x):
        x = np.ascontiguousarray(x, np.float32)
        codes = np.empty(max(len(x), 1), np.uint8)
        cb = np.empty(256, np.float32)
        rc = self.L.ref_quantize(x if len(x) else np.zeros(1, np.float32), len(x), codes, cb)
        if rc:
            raise OracleError(rc, "ref quantize")
        return codes[: len(x)], cb

    def dequantize(self, codes, cb):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.empty(max(len(codes), 1), np.float32)
        rc = self.L.ref_dequantize(codes if len(codes) else np.zeros(1, np.uint8), np.ascontiguousarray(cb, np.float32),
                                   len(codes), out)
        if rc:
            raise OracleError(rc, "ref dequantize")
        return out[: len(codes)]

    def encode_quant_chunk(self, codes, cb):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.empty(4 + 1024 + len(codes), np.uint8)
        n = C.c_uint64(0)
        rc = self.L.ref_encode_quant_chunk(codes if len(codes) else np.zeros(1, np.uint8),
                                           np.ascontiguousarray(cb, np.float32), len(codes), out, C.byref(n))
        if rc:
            raise OracleError(rc, "ref encode")
        return out[: n.value]

    def decode_quant_chunk(self, buf):
        buf = np.ascontiguousarray(buf, np.uint8)
        codes = np.empty(max(len(buf), 1), np.uint8)
        cb = np.empty(256, np.float32)
        cnt = C.c_uint64(0)
        rc = self.L.ref_decode_quant_chunk(buf if len(buf) else np.zeros(1, np.uint8), len(buf), codes, cb,
                                           C.byref(cnt))
        if rc:
            raise OracleError(rc, "ref decode")
        return codes[: cnt.value], cb

    def pseudo_gradient(self, prev, local):
        out = np.empty_like(prev)
        rc = self.L.ref_pseudo_gradient(prev, local, len(prev), out)
        if rc:
            raise OracleError(rc, "ref pg")
        return out

    def nesterov(self, theta, avg, buf, lr=0.7, momentum=0.9):
        theta = theta.copy()
        buf = buf.copy()
        rc = self.L.ref_nesterov(theta, np.ascontiguousarray(avg, np.float32), buf, len(theta), lr, momentum)
        if rc:
            raise OracleError(rc, "ref nesterov")
        return theta, buf

    def adamw(self, p, g, m, v, step, inner_lr=7.5e-5, lr_scale=1.0, beta1=0.9, beta2=0.95, eps=1e-8,
              weight_decay=0.1):
        """emesh::adamw_step itself (state.step = step - 1 before the call)."""
        p, m, v = (np.array(a, np.float32, copy=True) for a in (p, m, v))
        rc = self.L.ref_adamw(p, np.ascontiguousarray(g, np.float32), m, v, len(p), step - 1, inner_lr, lr_scale,
                              beta1, beta2, eps, weight_decay)
        if rc:
            raise OracleError(rc, "ref adamw")
        return p, m, v

    def ring_allreduce_sim(self, inputs, S=4, mode="int8", pipelined=True):
        inputs = [np.ascontiguousarray(a, np.float32) for a in inputs]
        k, n = len(inputs), len(inputs[0])
        outs = np.empty(max(k * n, 1), np.float32)
        sent = np.zeros(k, np.uint64)
        rc = self.L.ref_ring_allreduce_sim(_ptr_array(inputs), k, n, S, 1 if mode == "int8" else 0,
                                           1 if pipelined else 0, outs, sent)
        if rc:
            raise OracleError(rc, "ref ring (sim)")
        return outs[: k * n].reshape(k, n), sent

    def outer_sync_tcp(self, theta_g, theta_ls, buf, S=4, mode="int8", lr=0.7, momentum=0.9):
        theta_g = np.array(theta_g, np.float32, copy=True)
        buf = np.array(buf, np.float32, copy=True)
        ls = [np.ascontiguousarray(a, np.float32) for a in theta_ls]
        secs = np.zeros(1, np.float64)
        rc = self.L.ref_outer_sync_tcp(theta_g, _ptr_array(ls), buf, len(ls), len(theta_g), S,
                                       1 if mode == "int8" else 0, lr, momentum, secs)
        if rc:
            raise OracleError(rc, "ref outer sync (tcp)")
        return theta_g, buf, float(secs[0])


    @staticmethod
    def _ck_args(layout, sets):
        names = (C.c_char_p * max(len(layout), 1))(*[nm.encode() for nm, _ in layout])
        ranks = np.array([len(sh) for _, sh in layout] or [0], np.uint32)
        ext = np.array([e for _, sh in layout for e in sh] or [0], np.uint32)
        arrs = [np.ascontiguousarray(a, np.float32) for a in sets]
        ptrs = (C.c_void_p * 5)(*[a.ctypes.data for a in arrs])
        return names, ranks, ext, arrs, ptrs

    def encode_checkpoint(self, layout, sets, outer_step, adam_step, rng_seed, data_counter, shard, config_hash):
        """emesh::encode_checkpoint itself."""
        names, ranks, ext, arrs, ptrs = self._ck_args(layout, sets)
        h = np.frombuffer(bytes(config_hash), np.uint8).copy()
        n = C.c_uint64(0)
        self.L.ref_encode_checkpoint(outer_step, len(layout), C.cast(names, C.c_void_p), ranks.ctypes.data,
                                     ext.ctypes.data, ptrs, adam_step, rng_seed, data_counter, shard, h.ctypes.data,
                                     None, 0, C.byref(n))
        out = np.empty(n.value, np.uint8)
        rc = self.L.ref_encode_checkpoint(outer_step, len(layout), C.cast(names, C.c_void_p), ranks.ctypes.data,
                                          ext.ctypes.data, ptrs, adam_step, rng_seed, data_counter, shard,
                                          h.ctypes.data, out.ctypes.data, n.value, C.byref(n))
        if rc:
            raise OracleError(rc, "ref encode_checkpoint")
        return out.tobytes()

    def decode_checkpoint(self, buf, numel_cap):
        """emesh::decode_checkpoint: (code, message, sets, scalars, hash)."""
        sets = [np.zeros(max(numel_cap, 1), np.float32) for _ in range(5)]
        ptrs = (C.c_void_p * 5)(*[a.ctypes.data for a in sets])
        sc = np.zeros(5, np.uint64)
        h = np.zeros(32, np.uint8)
        msg = C.create_string_buffer(512)
        b = np.frombuffer(bytes(buf), np.uint8) if len(buf) else np.zeros(1, np.uint8)
        rc = self.L.ref_decode_checkpoint(b.ctypes.data, len(buf), ptrs, numel_cap, sc.ctypes.data, h.ctypes.data,
                                          msg, 512)
        return rc, msg.value.decode(errors="replace"), sets, [int(x) for x in sc], h.tobytes()

    def write_checkpoint_file(self, path, layout, sets, outer_step, adam_step, rng_seed, data_counter, shard,
                              config_hash):
        names, ranks, ext, arrs, ptrs = self._ck_args(layout, sets)
        h = np.frombuffer(bytes(config_hash), np.uint8).copy()
        rc = self.L.ref_write_checkpoint_file(path.encode(), outer_step, len(layout), C.cast(names, C.c_void_p),
                                              ranks.ctypes.data, ext.ctypes.data, ptrs, adam_step, rng_seed,
                                              data_counter, shard, h.ctypes.data)
        if rc:
            raise OracleError(rc, "ref write_checkpoint_file")

    def read_checkpoint_file(self, path, numel_cap):
        sets = [np.zeros(max(numel_cap, 1), np.float32) for _ in range(5)]
        ptrs = (C.c_void_p * 5)(*[a.ctypes.data for a in sets])
        sc = np.zeros(5, np.uint64)
        h = np.zeros(32, np.uint8)
        msg = C.create_string_buffer(512)
        rc = self.L.ref_read_checkpoint_file(path.encode(), ptrs, numel_cap, sc.ctypes.data, h.ctypes.data, msg, 512)
        return rc, msg.value.decode(errors="replace"), sets, [int(x) for x in sc], h.tobytes()

    def sha256(self, data):
        out = np.zeros(32, np.uint8)
        b = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
        self.L.ref_sha256(b.ctypes.data, len(data), out.ctypes.data)
        return out.tobytes()


def have_reference() -> bool:
    return os.path.exists(REF_SO)
