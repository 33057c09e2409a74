"""Checkpoint fixtures from the UNMODIFIED reference (oracle/_ref): the bytes
emesh::encode_checkpoint / write_checkpoint_file produce for a sample
Checkpoint, and emesh::decode_checkpoint's verdict (error class + message)
on a set of malformed variants of them. Run in the build container:

    make -C oracle && python tests/golden/make_checkpoint_golden.py
"""
import hashlib
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# a small model with every shape kind: matrices, vectors, a rank-0 scalar,
# a rank-3 tensor and a non-ASCII name
LAYOUT = [("embed.weight", (96, 16)), ("layers.0.attn.q", (16, 16)), ("layers.0.norm", (16,)),
          ("layers.0.mlp.up", (16, 40)), ("conv", (2, 3, 5)), ("temperature", ()), ("tête", (7,))]


def numel(shape):
    return int(np.prod(shape)) if len(shape) else 1


def sample():
    n = sum(numel(s) for _, s in LAYOUT)
    rs = np.random.RandomState(11)
    params = rs.standard_normal(n).astype(np.float32)
    retained = (params + np.float32(2.0 ** -10) * rs.standard_normal(n).astype(np.float32)).astype(np.float32)
    m = (np.float32(0.001) * (np.arange(n) % 7).astype(np.float32)).astype(np.float32)  # test_checkpoint.cpp:22-23
    v = np.abs(rs.standard_normal(n)).astype(np.float32) * np.float32(1e-4)
    buf = rs.standard_normal(n).astype(np.float32) * np.float32(1e-3)
    scalars = dict(outer_step=7, adam_step=35, rng_seed=11, data_counter=42, shard=3,
                   config_hash=hashlib.sha256(b"cfg").digest())
    return [params, retained, m, v, buf], scalars


def tensor_offsets(buf):
    """(name_len_at, rank_at, first extent_at, data_at, numel) of every tensor in stream order."""
    pos = 8
    out = []

    def params(pos):
        cnt, = struct.unpack_from("<I", buf, pos)
        pos += 4
        for _ in range(cnt):
            nl, = struct.unpack_from("<I", buf, pos)
            rank_at = pos + 4 + nl
            rank, = struct.unpack_from("<I", buf, rank_at)
            ext = struct.unpack_from("<%dI" % rank, buf, rank_at + 4)
            data_at = rank_at + 4 + 4 * rank
            out.append((pos, rank_at, rank_at + 4, data_at, numel(ext)))
            pos = data_at + 4 * numel(ext)
        return pos

    pos = params(pos)
    pos = params(pos)
    pos += 8
    for _ in range(3):
        pos = params(pos)
    return out


def variants(good):
    T = tensor_offsets(good)
    nt = len(LAYOUT)
    v = {}
    b = bytearray(good)

    def put(name, data):
        v[name] = bytes(data)

    for cut in (0, 4, 8, 11, T[0][3] + 5, T[nt][3], len(good) - 33, len(good) - 1):
        put(f"truncated@{cut}", good[:cut])
    put("trailing", good + b"\0")
    x = bytearray(b); struct.pack_into("<I", x, T[1][1], 9); put("rank9", x)
    x = bytearray(b); struct.pack_into("<I", x, T[1][2], 0); put("zero_extent", x)
    x = bytearray(b); struct.pack_into("<I", x, T[0][2], 1 << 20); put("implausible_size", x)
    x = bytearray(b); struct.pack_into("<I", x, T[0][2], 1 << 28); put("implausible_size_2p28", x)
    x = bytearray(b); struct.pack_into("<I", x, T[4][2] + 4, 1 << 27); put("implausible_size_rank3", x)
    x = bytearray(b); struct.pack_into("<I", x, T[0][0], 1 << 30); put("name_len_huge", x)
    for s_, t_ in ((0, 0), (1, 3), (2, 6), (4, 2)):
        x = bytearray(b); d = T[s_ * nt + t_][3]; struct.pack_into("<f", x, d + 4, float("nan")); put(f"nan@set{s_}t{t_}", x)
    x = bytearray(b); struct.pack_into("<f", x, T[3 * nt + 1][3], float("inf")); put("inf@set3t1", x)
    # duplicate name: tensor 1 of the params set ("layers.0.attn.q", 15 bytes) renamed to the
    # equal-length name of tensor 3 ("layers.0.mlp.up"): ShapeError when tensor 3 is added
    x = bytearray(b)
    t1 = T[1]
    x[t1[0] + 4: t1[0] + 4 + 15] = b"layers.0.mlp.up"
    put("duplicate_name_set0", x)
    y = bytearray(x); struct.pack_into("<f", y, T[0][3], float("nan")); put("nan_before_duplicate", y)
    y = bytearray(x); struct.pack_into("<f", y, T[3][3] + 8, float("nan")); put("nan_in_duplicate", y)
    y = bytearray(x); struct.pack_into("<f", y, T[4][3], float("nan")); put("nan_after_duplicate", y)
    # shape inconsistent: rename a tensor only in the retained set (same length) -> decodes, then fails same_shapes
    x = bytearray(b); t = T[nt + 2]; x[t[0] + 4: t[0] + 4 + 5] = b"LAYER"; put("name_mismatch_set1", x)
    # count mismatch in the retained set: its tensor count says nt-1 -> the stream misparses
    x = bytearray(b); struct.pack_into("<I", x, T[nt][0] - 4, nt - 1); put("count_mismatch_set1", x)
    return v


def main():
    R = Reference()
    sets, sc = sample()
    n = sum(numel(s) for _, s in LAYOUT)
    good = R.encode_checkpoint(LAYOUT, sets, sc["outer_step"], sc["adam_step"], sc["rng_seed"], sc["data_counter"],
                               sc["shard"], sc["config_hash"])
    path = os.path.join("/tmp", "emesh_golden_ckpt.bin")
    R.write_checkpoint_file(path, LAYOUT, sets, sc["outer_step"], sc["adam_step"], sc["rng_seed"],
                            sc["data_counter"], sc["shard"], sc["config_hash"])
    with open(path, "rb") as f:
        file_bytes = f.read()
    os.remove(path)
    names, bufs, codes, msgs = [], [], [], []
    for name, buf in variants(good).items():
        rc, msg, *_ = R.decode_checkpoint(buf, n)
        names.append(name)
        bufs.append(np.frombuffer(buf, np.uint8))
        codes.append(rc)
        msgs.append(msg)
        print(f"{name:24s} -> {rc} {msg}")
    np.savez_compressed(
        os.path.join(OUT, "checkpoint_cases.npz"),
        layout_names=np.array([nm for nm, _ in LAYOUT]),
        layout_shapes=np.array([",".join(map(str, s)) for _, s in LAYOUT]),
        sets=np.stack(sets), scalars=np.array([sc["outer_step"], sc["adam_step"], sc["rng_seed"],
                                               sc["data_counter"], sc["shard"]], np.uint64),
        config_hash=np.frombuffer(sc["config_hash"], np.uint8), encoded=np.frombuffer(good, np.uint8),
        file_bytes=np.frombuffer(file_bytes, np.uint8),
        var_names=np.array(names), var_codes=np.array(codes, np.int32), var_msgs=np.array(msgs),
        **{f"var_{i}": b for i, b in enumerate(bufs)})


if __name__ == "__main__":
    main()
