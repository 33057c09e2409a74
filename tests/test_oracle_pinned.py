"""CPU: pin the oracle restatement (oracle/emesh_oracle.c) against the
reference's own known answers, the golden fixtures generated from the
UNMODIFIED reference (tests/golden/make_golden.py), and — where this
container has /root/reference — the compiled reference itself."""
import numpy as np
import pytest

from oracle.pyoracle import Oracle, OracleError, Reference, have_reference


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_known_answers(oracle):
    # test_quant.cpp:62-79
    c, cb, st = oracle.quantize(np.array([-1.0, 1.0], np.float32))
    assert list(c) == [106, 149] and cb[106] == -1.0 and cb[149] == 1.0
    c, cb, _ = oracle.quantize(np.full(4, 5.0, np.float32))
    assert (c == 0).all() and (oracle.dequantize(c, cb) == 5.0).all()
    # test_optim.cpp:86-145
    d = oracle.pseudo_gradient(np.array([1, 1], np.float32), np.array([0, 2], np.float32))
    assert list(d) == [1.0, -1.0]
    th, b = oracle.nesterov(np.array([10.0], np.float32), np.array([1.0], np.float32), np.zeros(1, np.float32))
    assert b[0] == 1.0 and abs(th[0] - 8.67) <= 8.67e-6
    th, _ = oracle.nesterov(np.array([3.0], np.float32), np.array([0.5], np.float32), np.zeros(1, np.float32), 1.0, 0.0)
    assert th[0] == 2.5
    # test_allreduce.cpp:195-200 (fp32 ring {1,2},{3,4} -> {2,3})
    out = oracle.ring_allreduce([np.array([1, 2], np.float32), np.array([3, 4], np.float32)], 4, "fp32")
    assert list(out) == [2.0, 3.0]
    # test_allreduce.cpp:218-223
    out = oracle.ring_allreduce([np.full(64, 2.5, np.float32)] * 4, 4, "int8")
    assert (out == 2.5).all()


def test_errors(oracle):
    with pytest.raises(OracleError):
        oracle.quantize(np.zeros(0, np.float32))
    with pytest.raises(OracleError):
        oracle.quantize(np.array([1.0, np.nan], np.float32))


def test_quant_golden(oracle, golden):
    g = golden["quant_cases"]
    names = sorted({k.split("/")[0] for k in g.files})
    for name in names:
        c, cb, _ = oracle.quantize(g[f"{name}/x"])
        assert np.array_equal(c, g[f"{name}/codes"]), name
        assert np.array_equal(bits(cb), bits(g[f"{name}/cb"])), name
        assert np.array_equal(oracle.encode_quant_chunk(c, cb), g[f"{name}/wire"]), name
        c2, cb2 = oracle.decode_quant_chunk(g[f"{name}/wire"])
        assert np.array_equal(c2, c) and np.array_equal(bits(cb2), bits(cb))


def test_ring_golden(oracle, golden):
    g = golden["ring_cases"]
    keys = sorted({k.rsplit("/", 1)[0] for k in g.files})
    for key in keys:
        ins = list(g[f"{key}/inputs"])
        S = int(key.split("_S")[1].split("_")[0])
        mode = key.rsplit("_", 1)[1]
        out = oracle.ring_allreduce(ins, S, mode)
        assert np.array_equal(bits(out), bits(g[f"{key}/out"])), key


def test_wire_volume_golden(golden):
    # test_allreduce.cpp:263-275 and SURVEY §2: rank bytes = 2(k-1)/k * payload + per-frame overhead
    g = golden["ring_cases"]
    for key in sorted({k.rsplit("/", 1)[0] for k in g.files}):
        k, n = g[f"{key}/inputs"].shape
        if k == 1 or n < 1000:
            continue
        per = 4 if key.endswith("fp32") else 1
        expect = 2 * (k - 1) / k * n * per
        sent = g[f"{key}/bytes_sent"].astype(np.float64)
        assert (sent >= expect * 0.95).all()


def test_outer_sync_golden(oracle, golden):
    g = golden["outer_sync_case"]
    tg, tb = oracle.outer_sync(g["theta_g"], list(g["theta_l"]), g["buf"], int(g["S"]), "int8", 0.7, 0.9)
    assert np.array_equal(bits(tg), bits(g["theta_g_out"]))
    assert np.array_equal(bits(tb), bits(g["buf_out"]))


def test_segment_table_matches_reference_rule(oracle):
    # allreduce.hpp:107-118 (first n%k chunks +1), :327-336 (min(S, len) subs, len 0 -> one empty)
    for n, k, S in [(17, 4, 4), (3, 4, 4), (100003, 8, 16), (16777216, 2, 4), (0, 2, 4)]:
        lo, ln = oracle.segment_table(n, k, S)
        assert int(ln.sum()) == n
        assert all(int(lo[i]) + int(ln[i]) == int(lo[i + 1]) for i in range(len(lo) - 1))


def test_decode_fuzz_never_crashes(oracle):
    # test_quant.cpp:171-184
    for seed in range(200):
        ln = oracle.rng_word(seed, 9, 0, 0) % 2000
        buf = np.array([oracle.rng_word(seed, 9, 1, i) & 0xFF for i in range(ln)], np.uint8)
        try:
            c, cb = oracle.decode_quant_chunk(buf)
            assert len(cb) == 256
        except OracleError:
            pass


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_vs_compiled_reference_live(oracle):
    R = Reference()
    for seed in range(6):
        x = oracle.uniform(50_001, seed, 1, 0, 0, 1e-3)
        if seed % 2:
            x[::13] += np.float32(0.05)
        a, b = oracle.quantize(x)[:2], R.quantize(x)
        assert np.array_equal(a[0], b[0]) and np.array_equal(bits(a[1]), bits(b[1]))
    for k in (2, 3, 4):
        for n in (1, 17, 4096):
            ins = [oracle.uniform(n, 100 + n, i) for i in range(k)]
            for mode in ("fp32", "int8"):
                want = oracle.ring_allreduce(ins, 4, mode)
                got, _ = R.ring_allreduce_sim(ins, 4, mode)
                for r in got:
                    assert np.array_equal(bits(r), bits(want)), (k, n, mode)
    # pipelined vs serial schedules are byte-identical (test_allreduce.cpp:277-289)
    ins = [oracle.uniform(2048, 88, i) for i in range(4)]
    a, _ = R.ring_allreduce_sim(ins, 4, "int8", True)
    b, _ = R.ring_allreduce_sim(ins, 4, "int8", False)
    assert np.array_equal(bits(a), bits(b))


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (needs /root/reference)")
def test_adamw_oracle_vs_compiled_reference(oracle):
    """optim.hpp:63-94: the restated AdamW step equals emesh::adamw_step bit for bit."""
    R = Reference()
    n = 20_011
    p = oracle.uniform(n, 1, 0)
    m = oracle.uniform(n, 2, 0, 0, 0, 1e-3)
    v = np.abs(oracle.uniform(n, 3, 0, 0, 0, 1e-5)).astype(np.float32)
    for step, scale in ((1, 1.0), (2, 0.5), (37, 0.01), (5000, 1.0)):
        g = oracle.uniform(n, 10 + step, 0, 0, 0, 1e-2)
        a = oracle.adamw(p, g, m, v, step, 7.5e-5, scale)
        b = R.adamw(p, g, m, v, step, 7.5e-5, scale)
        for x, y in zip(a, b):
            assert np.array_equal(bits(x), bits(y)), step
        p, m, v = a
    g = np.zeros(n, np.float32)
    g[7] = np.inf
    with pytest.raises(OracleError):
        oracle.adamw(p, g, m, v, 1)
    with pytest.raises(OracleError):
        R.adamw(p, g, m, v, 1)
