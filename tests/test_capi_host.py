"""CPU: the C-ABI library loads without a GPU, exports every symbol
include/emesh_b200.h declares, and its host-only entry points (wire codec,
segment planner) agree with the oracle."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def capi():
    from paper_2412_01152_b200 import _capi
    if not os.path.exists(_capi.LIB_PATH):
        from paper_2412_01152_b200 import build
        build.build_product()
    return _capi


def header_functions():
    src = open(os.path.join(ROOT, "include", "emesh_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(emesh_[a-z0-9_]+)\s*\(", src))


def test_exports_every_declared_symbol(capi):
    L = capi.lib()
    declared = header_functions()
    assert len(declared) >= 20
    assert declared == set(capi.EXPORTS), declared ^ set(capi.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.emesh_abi_version() == 1


def test_library_links_cuda_and_nccl(capi):
    # no CPU fallback: the product library is the CUDA build (sm_100a cubin inside)
    data = open(capi.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data
    assert b"ncclSend" in data


def test_wire_codec_matches_oracle(capi, oracle, golden):
    import ctypes as C
    from paper_2412_01152_b200 import emesh as E
    g = golden["quant_cases"]
    for name in sorted({k.split("/")[0] for k in g.files}):
        codes, cb = g[f"{name}/codes"], g[f"{name}/cb"]
        wire = g[f"{name}/wire"]
        out = np.empty(4 + 1024 + len(codes), np.uint8)
        n = capi.lib().emesh_encode_quant_chunk(codes.ctypes.data, cb.ctypes.data, len(codes), out.ctypes.data)
        assert n == len(wire) and np.array_equal(out[:n], wire)
        c2 = np.empty(len(codes), np.uint8)
        cb2 = np.empty(256, np.float32)
        cnt = C.c_uint32()
        assert capi.lib().emesh_decode_quant_chunk(wire.ctypes.data, len(wire), c2.ctypes.data, cb2.ctypes.data,
                                                   C.byref(cnt)) == 0
        assert cnt.value == len(codes) and np.array_equal(c2, codes)


def test_wire_decode_rejects_malformed(capi, golden):
    # test_quant.cpp:152-169: truncated, count mismatch; quant.hpp:124 non-finite codebook
    import ctypes as C
    wire = golden["quant_cases"]["normal_300/wire"].copy()
    c2 = np.empty(4096, np.uint8)
    cb2 = np.empty(256, np.float32)
    cnt = C.c_uint32()

    def dec(buf):
        return capi.lib().emesh_decode_quant_chunk(buf.ctypes.data, len(buf), c2.ctypes.data, cb2.ctypes.data,
                                                   C.byref(cnt))

    assert dec(wire) == 0
    assert dec(wire[:-5].copy()) == capi.EDECODE
    bad = wire.copy()
    bad[0] = 200
    assert dec(bad) == capi.EDECODE
    nf = wire.copy()
    nf[4:8] = np.frombuffer(np.float32(np.inf).tobytes(), np.uint8)
    assert dec(nf) == capi.EDECODE
    assert dec(np.zeros(3, np.uint8)) == capi.EDECODE


@pytest.mark.parametrize("n,k,S", [(17, 4, 4), (3, 4, 4), (0, 2, 4), (100003, 8, 16), (16777216, 2, 4),
                                   (1_000_000_000, 4, 16), (10_211_381_248, 8, 80)])
def test_plan_segments_match_oracle(capi, oracle, n, k, S):
    from paper_2412_01152_b200 import emesh as E
    lo, ln = E.plan_segments(n, k, S)
    if n < 50_000_000:
        olo, oln = oracle.segment_table(n, k, S)
        assert np.array_equal(lo, olo) and np.array_equal(ln, oln)
    py = E.segment_table(n, k, S)
    assert [int(a) for a in lo] == [a for a, _ in py] and [int(b) for b in ln] == [b for _, b in py]
    assert int(ln.sum()) == n


# INTELLECT-1 shape: 42 layers, d=4096, 32/8 heads, FFN 14336, vocab 128256
def intellect1_tensor_sizes():
    d, kv, ffn, vocab = 4096, 1024, 14336, 128256
    sizes = [vocab * d]
    for _ in range(42):
        sizes += [d, d * d, d * kv, d * kv, d * d, d, d * ffn, d * ffn, ffn * d]
    sizes += [d, vocab * d]
    return sizes


def test_intellect1_shape():
    s = intellect1_tensor_sizes()
    assert len(s) == 381 and sum(s) == 10_211_381_248


@pytest.mark.parametrize("sizes,k,S", [([5, 17, 0, 100], 4, 4), ([1, 2, 3], 8, 4), ([4096] * 3 + [100_003], 2, 16),
                                       (None, 8, 4)])
def test_plan_tensor_segments_match_per_tensor_oracle(capi, oracle, sizes, k, S):
    """Multi-tensor engine (config 5): one ReduceJob per tensor, every tensor's segment table as the
    reference builds it (allreduce.hpp:107-118, 326-336), chunk-major across tensors."""
    from paper_2412_01152_b200 import emesh as E
    if sizes is None:
        sizes = intellect1_tensor_sizes()
    lo, ln = E.plan_tensor_segments(sizes, k, S)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    per = []
    for t, n_t in enumerate(sizes):
        tl, tn = oracle.segment_table(int(n_t), k, S) if n_t < 50_000_000 else E.plan_segments(int(n_t), k, S)
        # per-tensor table is chunk-major: split it back into its k chunks
        chunks, i = [], 0
        for c in range(k):
            clen = n_t // k + (1 if c < n_t % k else 0)
            ns = 1 if clen == 0 else min(S, clen)
            chunks.append([(int(off[t] + tl[j]), int(tn[j])) for j in range(i, i + ns)])
            i += ns
        per.append(chunks)
    want = [seg for c in range(k) for t in range(len(sizes)) for seg in per[t][c]]
    assert [(int(a), int(b)) for a, b in zip(lo, ln)] == want
    assert int(ln.sum()) == sum(sizes)

