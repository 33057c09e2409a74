"""Checkpoint (de)serialization throughput from / into device arenas
(payload GB/s; staged pageable vs page-locked host buffers; file write/read
incl. SHA-256). Usage: python tools/ckpt_speed.py [params]"""
import ctypes as C
import os
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_01152_b200 as E  # noqa: E402
from paper_2412_01152_b200 import _capi  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
t = 1 << 24
layout = [(f"t{i}", (min(t, n - i * t),)) for i in range((n + t - 1) // t)]
like = E.ModelParams(layout)
c = E.Checkpoint.zeros_like(like)
for mp in (c.params, c.retained, c.inner.m, c.inner.v, c.outer.buffer):
    mp.arena.normal_()
v, keep = E.emesh._ck_view(c)
L = _capi.lib()
size = C.c_uint64()
L.emesh_checkpoint_encoded_size(C.byref(v), C.byref(size))
N = size.value
pageable = C.create_string_buffer(N)
pinned = torch.empty(N, dtype=torch.uint8, pin_memory=True)
w = C.c_uint64()


def timed(f, reps=3):
    f()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


res = {}
res["encode_pageable"] = timed(lambda: L.emesh_checkpoint_encode(C.byref(v), C.addressof(pageable), N, C.byref(w), None))
res["encode_pinned"] = timed(lambda: L.emesh_checkpoint_encode(C.byref(v), pinned.data_ptr(), N, C.byref(w), None))
assert bytes(pageable.raw) == pinned.numpy().tobytes()
res["decode_pageable"] = timed(lambda: L.emesh_checkpoint_decode(C.addressof(pageable), N, C.byref(v), None))
res["decode_pinned"] = timed(lambda: L.emesh_checkpoint_decode(pinned.data_ptr(), N, C.byref(v), None))
res["sha256"] = timed(lambda: E.sha256(pinned.numpy()[: 1 << 30].tobytes()), reps=1) * N / min(N, 1 << 30)
with tempfile.TemporaryDirectory(dir=os.environ.get("CKPT_DIR", "/tmp")) as td:
    p = os.path.join(td, "ck.bin").encode()
    res["write_file"] = timed(lambda: L.emesh_checkpoint_write_file(p, C.byref(v), None), reps=1)
    res["read_file"] = timed(lambda: L.emesh_checkpoint_read_file(p, C.byref(v), None), reps=1)
print(f"payload {N / 1e9:.2f} GB ({n} params x 5 sets)")
for k_, s in res.items():
    print(f"{k_:16s} {s * 1e3:9.1f} ms  {N / s / 1e9:6.2f} GB/s")
