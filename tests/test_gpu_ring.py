"""GPU parity of the int8 ring engine and the fused outer-sync round against
the oracle restatement (transport-free ring_allreduce, allreduce.hpp:314-473)
and the reference's own golden outputs (SimWorld ring, TCP outer sync)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def E():
    import paper_2412_01152_b200 as E
    return E


def run_virtual_allreduce(E, ins, S, window=0):
    k, n = len(ins), len(ins[0])
    eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=True, window_elems=window)
    tin = [T(a) for a in ins]
    outs = [torch.empty(n + 4, dtype=torch.float32, device="cuda:0")[:n] for _ in range(k)]
    eng.ring_allreduce(tin, outs)
    eng.check()
    res = [o.cpu().numpy() for o in outs]
    for a, t in zip(ins, tin):  # ReduceJob.input is preserved (allreduce.hpp:47-48)
        assert np.array_equal(bits(t.cpu().numpy()), bits(a))
    return eng, res


def test_ring_golden_reference_outputs(E, golden):
    g = golden["ring_cases"]
    keys = sorted({k.rsplit("/", 1)[0] for k in g.files if k.endswith("_int8/out")})
    assert keys
    for key in keys:
        ins = list(g[f"{key}/inputs"])
        S = int(key.split("_S")[1].split("_")[0])
        eng, res = run_virtual_allreduce(E, ins, S)
        for r in res:
            assert np.array_equal(bits(r), bits(g[f"{key}/out"])), key
        eng.close()


@pytest.mark.parametrize("k", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 5, 17, 4096, 100_003])
def test_ring_vs_oracle(E, oracle, k, n):
    ins = [oracle.uniform(n, 100 + n, i) for i in range(k)]
    S = 4
    want, codes, cbs, stats = oracle.ring_allreduce(ins, S, "int8", with_payloads=True)
    eng, res = run_virtual_allreduce(E, ins, S)
    for r in res:  # every worker decodes the owners' bytes -> bit-identical
        assert np.array_equal(bits(r), bits(want))
    # owners' final payloads: codes + codebooks bit-exact
    lo, ln = eng.segments()
    for c in range(k):
        owner = (c + k - 1) % k
        pc, pcb, pst = eng.payload(owner)
        base, rem = divmod(n, k)
        for i, (a, b) in enumerate(zip(lo, ln)):
            a, b = int(a), int(b)
            cstart = c * base + min(c, rem)
            clen = base + (1 if c < rem else 0)
            if b == 0 or not (cstart <= a < cstart + clen):
                continue
            assert np.array_equal(pc[a:a + b], codes[a:a + b]), (c, i)
            assert np.array_equal(bits(pcb[i]), bits(cbs[i])), (c, i)
    eng.close()


@pytest.mark.parametrize("S", [1, 3, 16])
def test_ring_subchunks_and_windows(E, oracle, S):
    k, n = 4, 262_147
    ins = [oracle.uniform(n, 5, i, 0, 0, 2.0 ** -8) for i in range(k)]
    want = oracle.ring_allreduce(ins, S, "int8")
    for window in (0, 1, 40_000):  # one segment per window / auto
        eng, res = run_virtual_allreduce(E, ins, S, window)
        assert np.array_equal(bits(res[0]), bits(want)), window
        eng.close()


def test_ring_constant_inputs_exact(E):
    # test_allreduce.cpp:218-223
    ins = [np.full(64, 2.5, np.float32) for _ in range(4)]
    _, res = run_virtual_allreduce(E, ins, 4)
    assert all((r == 2.5).all() for r in res)


def test_ring_nonfinite_raises(E, oracle):
    ins = [oracle.uniform(1000, 1, i) for i in range(2)]
    ins[1][17] = np.nan
    eng = E.RingEngine(1000, 2, virtual=True)
    outs = [torch.empty(1000, dtype=torch.float32, device="cuda:0") for _ in range(2)]
    eng.ring_allreduce([T(a) for a in ins], outs)
    with pytest.raises(E.NumericError):
        eng.check()
    eng.check()  # consumed
    eng.close()


def test_outer_sync_golden_reference_round(E, golden):
    g = golden["outer_sync_case"]
    k, S = int(g["k"]), int(g["S"])
    n = g["theta_g"].shape[0]
    eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=True)
    tg = [T(g["theta_g"]) for _ in range(k)]
    tl = [T(x) for x in g["theta_l"]]
    tb = [T(g["buf"]) for _ in range(k)]
    eng.outer_sync(tg, tl, tb, E.HyperParams(), write_local=True)
    eng.check()
    for w in range(k):
        assert np.array_equal(bits(tg[w].cpu().numpy()), bits(g["theta_g_out"]))
        assert np.array_equal(bits(tb[w].cpu().numpy()), bits(g["buf_out"]))
        assert np.array_equal(bits(tl[w].cpu().numpy()), bits(g["theta_g_out"]))  # local = retained
    eng.close()


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_outer_sync_vs_oracle_two_rounds(E, oracle, k):
    n, S = 300_007, 4
    g0 = oracle.uniform(n, 3, 0)
    b0 = np.zeros(n, np.float32)
    eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=(k > 1))
    tg = [T(g0) for _ in range(k)]
    tb = [T(b0) for _ in range(k)]
    eg, eb = g0, b0
    for rnd in range(2):  # round 2 exercises a non-zero momentum buffer
        ls = [(eg - oracle.uniform(n, 3 + rnd, 1 + w, 0, 0, 2.0 ** -10)).astype(np.float32) for w in range(k)]
        tl = [T(a) for a in ls]
        eng.outer_sync(tg, tl, tb, E.HyperParams(), write_local=False)
        eng.check()
        eg, eb = oracle.outer_sync(eg, ls, eb, S, "int8", 0.7, 0.9)
        for w in range(k):
            assert np.array_equal(bits(tg[w].cpu().numpy()), bits(eg)), (rnd, w)
            assert np.array_equal(bits(tb[w].cpu().numpy()), bits(eb)), (rnd, w)
    eng.close()


@pytest.mark.parametrize("k", [2, 3, 4])
def test_outer_sync_host_api(E, oracle, k):
    """Host buffers, chunk-pipelined copies (emesh_engine_outer_sync_host): bit-exact vs the oracle."""
    n, S = 100_003, 4
    g = oracle.uniform(n, 8, 0)
    ls = [(g - oracle.uniform(n, 8, 1 + w, 0, 0, 2.0 ** -10)).astype(np.float32) for w in range(k)]
    b = oracle.uniform(n, 8, 7, 0, 0, 1e-3)
    eg, eb = oracle.outer_sync(g, ls, b, S, "int8", 0.7, 0.9)
    eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=True)
    hg = [torch.from_numpy(g.copy()).pin_memory() for _ in range(k)]
    hl = [torch.from_numpy(a.copy()).pin_memory() for a in ls]
    hb = [torch.from_numpy(b.copy()).pin_memory() for _ in range(k)]
    eng.outer_sync_host(hg, hl, hb, E.HyperParams(), write_local=True)
    for w in range(k):
        assert np.array_equal(bits(hg[w].numpy()), bits(eg))
        assert np.array_equal(bits(hb[w].numpy()), bits(eb))
        assert np.array_equal(bits(hl[w].numpy()), bits(eg))
    eng.close()


def test_outer_sync_host_multi_tensor_two_rounds(E):
    """Host path over a multi-tensor plan (per-tensor chunk runs), two rounds: identical to the device path."""
    sizes = [4096, 1_000_003, 17, 250_000, 4096 * 3]
    n, k = sum(sizes), 4
    gen = torch.Generator().manual_seed(3)
    g0 = torch.randn(n, generator=gen)
    ls = [[g0 - 1e-3 * torch.randn(n, generator=gen) for _ in range(k)] for _ in range(2)]
    eng_h = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=4), virtual=True, tensor_sizes=sizes)
    eng_d = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=4), virtual=True, tensor_sizes=sizes)
    hg = [g0.clone().pin_memory() for _ in range(k)]
    hb = [torch.zeros(n).pin_memory() for _ in range(k)]
    dg = [g0.cuda() for _ in range(k)]
    db = [torch.zeros(n, device="cuda") for _ in range(k)]
    for rnd in range(2):
        hl = [a.clone().pin_memory() for a in ls[rnd]]
        dl = [a.cuda() for a in ls[rnd]]
        eng_h.outer_sync_host(hg, hl, hb, E.HyperParams(), write_local=False)
        eng_d.outer_sync(dg, dl, db, E.HyperParams(), write_local=False)
        eng_d.check()
        for w in range(k):
            assert torch.equal(hg[w].view(torch.int32), dg[w].cpu().view(torch.int32)), (rnd, w)
            assert torch.equal(hb[w].view(torch.int32), db[w].cpu().view(torch.int32)), (rnd, w)
    eng_h.close()
    eng_d.close()


def test_full_size_properties_config1(E, oracle):
    """Config 1 at full size (N=16,777,216, k=2, S=4): bit-exact vs the
    oracle's hop-by-hop restatement, all workers identical."""
    n, k, S = 16_777_216, 2, 4
    ins = [oracle.uniform(n, 1, 1 + w, 0, 0, 2.0 ** -10) for w in range(k)]
    want = oracle.ring_allreduce(ins, S, "int8")
    _, res = run_virtual_allreduce(E, ins, S)
    for r in res:
        assert np.array_equal(bits(r), bits(want))


# ---------------------------------------------------------------- ReduceMode::fp32


def run_virtual_allreduce_f32(E, ins, S, window=0):
    k, n = len(ins), len(ins[0])
    eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=True, window_elems=window,
                       mode=E.ReduceMode.fp32)
    tin = [T(a) for a in ins]
    outs = [torch.empty(n + 4, dtype=torch.float32, device="cuda:0")[:n] for _ in range(k)]
    eng.ring_allreduce(tin, outs)
    eng.check()
    res = [o.cpu().numpy() for o in outs]
    for a, t in zip(ins, tin):
        assert np.array_equal(bits(t.cpu().numpy()), bits(a))
    return eng, res


def test_ring_fp32_golden_reference_outputs(E, golden):
    """The reference's own SimWorld ring in ReduceMode::fp32 (test_allreduce.cpp:195-216 style)."""
    g = golden["ring_cases"]
    keys = sorted({k.rsplit("/", 1)[0] for k in g.files if k.endswith("_fp32/out")})
    assert keys
    for key in keys:
        ins = list(g[f"{key}/inputs"])
        S = int(key.split("_S")[1].split("_")[0])
        eng, res = run_virtual_allreduce_f32(E, ins, S)
        for r in res:
            assert np.array_equal(bits(r), bits(g[f"{key}/out"])), key
        eng.close()


def test_ring_fp32_known_answer(E):
    """test_allreduce.cpp:195-200: {1,2},{3,4} -> {2,3} on both ranks."""
    eng, res = run_virtual_allreduce_f32(E, [np.array([1, 2], np.float32), np.array([3, 4], np.float32)], 4)
    for r in res:
        assert r.tolist() == [2.0, 3.0]
    eng.close()


@pytest.mark.parametrize("k", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 17, 4096, 100_003])
def test_ring_fp32_vs_oracle(E, oracle, k, n):
    ins = [oracle.uniform(n, 100 + n, i) for i in range(k)]
    want = oracle.ring_allreduce(ins, 4, "fp32")
    eng, res = run_virtual_allreduce_f32(E, ins, 4)
    for r in res:
        assert np.array_equal(bits(r), bits(want))
    eng.close()


@pytest.mark.parametrize("k", [2, 4])
def test_outer_sync_fp32_vs_oracle_two_rounds(E, oracle, k):
    n, S = 200_003, 4
    g0 = oracle.uniform(n, 3, 0)
    b0 = np.zeros(n, np.float32)
    eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=True, mode=E.ReduceMode.fp32)
    tg = [T(g0) for _ in range(k)]
    tb = [T(b0) for _ in range(k)]
    eg, eb = g0, b0
    for rnd in range(2):
        ls = [(eg - oracle.uniform(n, 3 + rnd, 1 + w, 0, 0, 2.0 ** -10)).astype(np.float32) for w in range(k)]
        tl = [T(a) for a in ls]
        eng.outer_sync(tg, tl, tb, E.HyperParams(), write_local=True)
        eng.check()
        eg, eb = oracle.outer_sync(eg, ls, eb, S, "fp32", 0.7, 0.9)
        for w in range(k):
            assert np.array_equal(bits(tg[w].cpu().numpy()), bits(eg)), (rnd, w)
            assert np.array_equal(bits(tb[w].cpu().numpy()), bits(eb)), (rnd, w)
            assert np.array_equal(bits(tl[w].cpu().numpy()), bits(eg)), (rnd, w)
    eng.close()


def test_ring_allreduce_job_mode_checked(E):
    eng = E.RingEngine(8, 2, virtual=True)
    with pytest.raises(E.ConfigError):
        E.ring_allreduce(eng, E.ReduceJob(1, torch.zeros(8, device="cuda:0"), E.ReduceMode.fp32))
    eng.close()


# ---------------------------------------------------------------- multi-tensor engines (config 5)

MT_SIZES = [4096, 17, 0, 100_003, 1, 65_536, 3, 250_000]


@pytest.mark.parametrize("mode", ["int8", "fp32"])
@pytest.mark.parametrize("k", [2, 4])
def test_multi_tensor_ring_vs_per_tensor_oracle(E, oracle, k, mode):
    """One ReduceJob per tensor, all tensors' chunks bucketed per hop: equal to
    running the reference's ring on every tensor separately."""
    n = sum(MT_SIZES)
    off = np.concatenate([[0], np.cumsum(MT_SIZES)])
    ins = [oracle.uniform(n, 77, i, 0, 0, 2.0 ** -4) for i in range(k)]
    want = np.concatenate([oracle.ring_allreduce([a[off[t]:off[t + 1]] for a in ins], 4, mode)[:MT_SIZES[t]]
                           for t in range(len(MT_SIZES))])
    eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=4), virtual=True, mode=E.ReduceMode[mode],
                       tensor_sizes=MT_SIZES)
    tin = [T(a) for a in ins]
    outs = [torch.empty(n + 4, dtype=torch.float32, device="cuda:0")[:n] for _ in range(k)]
    eng.ring_allreduce(tin, outs)
    eng.check()
    for o in outs:
        assert np.array_equal(bits(o.cpu().numpy()), bits(want))
    eng.close()


def test_multi_tensor_outer_sync_vs_per_tensor_oracle(E, oracle):
    k, S = 4, 4
    n = sum(MT_SIZES)
    off = np.concatenate([[0], np.cumsum(MT_SIZES)])
    g0 = oracle.uniform(n, 5, 0)
    ls = [(g0 - oracle.uniform(n, 6, 1 + w, 0, 0, 2.0 ** -10)).astype(np.float32) for w in range(k)]
    b0 = oracle.uniform(n, 7, 0, 0, 0, 2.0 ** -12)
    eg, eb = [], []
    for t in range(len(MT_SIZES)):
        if MT_SIZES[t] == 0:
            continue
        sl = slice(off[t], off[t + 1])
        g_t, b_t = oracle.outer_sync(g0[sl], [a[sl] for a in ls], b0[sl], S, "int8", 0.7, 0.9)
        eg.append(g_t[:MT_SIZES[t]])
        eb.append(b_t[:MT_SIZES[t]])
    eg, eb = np.concatenate(eg), np.concatenate(eb)
    eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=True, tensor_sizes=MT_SIZES)
    tg = [T(g0) for _ in range(k)]
    tb = [T(b0) for _ in range(k)]
    eng.outer_sync(tg, [T(a) for a in ls], tb, E.HyperParams(), write_local=False)
    eng.check()
    for w in range(k):
        assert np.array_equal(bits(tg[w].cpu().numpy()), bits(eg))
        assert np.array_equal(bits(tb[w].cpu().numpy()), bits(eb))
    eng.close()
