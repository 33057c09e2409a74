"""B200: checkpoints straight from / into device arenas (
checkpoint.hpp:32-66,190-224) — byte-identical to the reference's encoding
(golden fixture from the UNMODIFIED reference), every malformed variant gets
the reference's verdict (including the device-side non-finite scan), and the
file framing round-trips and detects corruption."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2412_01152_b200 as E  # noqa: E402
from paper_2412_01152_b200 import _capi  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ck():
    return np.load(os.path.join(ROOT, "tests", "golden", "checkpoint_cases.npz"))


def layout_of(ck):
    return [(str(nm), tuple(int(e) for e in sh.split(",") if e)) for nm, sh in zip(ck["layout_names"],
                                                                                   ck["layout_shapes"])]


def device_checkpoint(ck):
    like = E.ModelParams(layout_of(ck))
    c = E.Checkpoint.zeros_like(like)
    for mp, flat in zip((c.params, c.retained, c.inner.m, c.inner.v, c.outer.buffer), ck["sets"]):
        mp.arena.copy_(torch.from_numpy(flat))
    sc = [int(x) for x in ck["scalars"]]
    c.outer_step, c.inner.step, c.rng_seed, c.data_counter, c.shard = sc
    c.config_hash = ck["config_hash"].tobytes()
    return c


def host_sets(c):
    return [mp.arena.cpu().numpy() for mp in (c.params, c.retained, c.inner.m, c.inner.v, c.outer.buffer)]


def test_encode_from_device_is_reference_bytes(ck):
    c = device_checkpoint(ck)
    assert E.encode_checkpoint(c) == ck["encoded"].tobytes()


def test_encode_into_pinned_buffer(ck):
    c = device_checkpoint(ck)
    v, keep = E.emesh._ck_view(c)
    n = len(ck["encoded"])
    out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    w = C.c_uint64()
    assert _capi.lib().emesh_checkpoint_encode(C.byref(v), out.data_ptr(), n, C.byref(w), None) == 0
    assert w.value == n and out.numpy().tobytes() == ck["encoded"].tobytes()
    # short buffer: ShapeError and the size needed
    assert _capi.lib().emesh_checkpoint_encode(C.byref(v), out.data_ptr(), n - 1, C.byref(w), None) == _capi.ESHAPE
    assert w.value == n


@pytest.mark.parametrize("with_like", [False, True])
def test_decode_into_device(ck, with_like):
    like = E.ModelParams(layout_of(ck)) if with_like else None
    c = E.decode_checkpoint(ck["encoded"].tobytes(), like=like)
    for got, want in zip(host_sets(c), ck["sets"]):
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert [c.outer_step, c.inner.step, c.rng_seed, c.data_counter, c.shard] == [int(x) for x in ck["scalars"]]
    assert c.config_hash == ck["config_hash"].tobytes()
    assert c.params.names == [nm for nm, _ in layout_of(ck)]


def test_decode_from_pinned_buffer(ck):
    buf = torch.from_numpy(ck["encoded"].copy()).pin_memory()
    c = E.Checkpoint.zeros_like(E.ModelParams(layout_of(ck)))
    v, keep = E.emesh._ck_view(c)
    assert _capi.lib().emesh_checkpoint_decode(buf.data_ptr(), buf.numel(), C.byref(v), None) == 0
    for got, want in zip(host_sets(c), ck["sets"]):
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_every_variant_gets_the_reference_verdict(ck):
    like = E.ModelParams(layout_of(ck))
    kinds = {0: None, 1: E.ShapeError, 3: E.DecodeError}
    for i, name in enumerate(ck["var_names"]):
        want = kinds[int(ck["var_codes"][i])]
        with pytest.raises(want) as ei:
            E.decode_checkpoint(ck[f"var_{i}"].tobytes(), like=like)
        assert type(ei.value) is want, name
        assert str(ei.value) == str(ck["var_msgs"][i]), name


def test_file_round_trip_and_integrity(ck, tmp_path):
    c = device_checkpoint(ck)
    p = str(tmp_path / "ck.bin")
    E.write_checkpoint_file(p, c)
    assert open(p, "rb").read() == ck["file_bytes"].tobytes()
    back = E.read_checkpoint_file(p)
    for got, want in zip(host_sets(back), ck["sets"]):
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # test_checkpoint.cpp:56-62: one corrupted byte -> the hash check fires (emesh::Error)
    bad = bytearray(open(p, "rb").read())
    bad[60] ^= 0x5A
    open(p, "wb").write(bytes(bad))
    with pytest.raises(E.Error) as ei:
        E.read_checkpoint_file(p, like=E.ModelParams(layout_of(ck)))
    assert "hash mismatch" in str(ei.value)
    with pytest.raises(E.Error):
        E.read_checkpoint_file(str(tmp_path / "missing.bin"), like=E.ModelParams(layout_of(ck)))


def test_large_round_trip_matches_oracle():
    """A Llama-shaped slice (~13M params, 2 tensors larger than a staging
    block): encode -> bytes identical to the oracle restatement; file write ->
    read -> arenas bit-identical; staged and pinned paths agree."""
    from oracle.pyoracle import checkpoint_encode, checkpoint_file_bytes
    d, ffn, vocab = 512, 1536, 8000
    layout = [("embed", (vocab, d))]
    for i in range(2):
        layout += [(f"l{i}.q", (d, d)), (f"l{i}.kv", (2, d, d // 4)), (f"l{i}.up", (d, ffn)),
                   (f"l{i}.down", (ffn, d)), (f"l{i}.norm", (d,))]
    layout += [("head", (d, vocab)), ("bias", ())]
    like = E.ModelParams(layout)
    c = E.Checkpoint.zeros_like(like)
    g = torch.Generator(device="cuda").manual_seed(5)
    for mp in (c.params, c.retained, c.inner.m, c.inner.v, c.outer.buffer):
        mp.arena.copy_(torch.randn(mp.element_count(), device="cuda", generator=g))
    c.outer_step, c.inner.step, c.rng_seed, c.data_counter, c.shard = 3, 15, 99, 7, 1
    c.config_hash = bytes(range(32))
    enc = E.encode_checkpoint(c)
    want = checkpoint_encode(layout, host_sets(c), 3, 15, 99, 7, 1, bytes(range(32)))
    assert enc == want
    back = E.decode_checkpoint(enc, like=like)
    for a, b in zip(host_sets(back), host_sets(c)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "big.bin")
        E.write_checkpoint_file(p, c)
        assert open(p, "rb").read() == checkpoint_file_bytes(want)
        back = E.read_checkpoint_file(p, like=like)
        for a, b in zip(host_sets(back), host_sets(c)):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_nonfinite_in_large_arena_is_found_on_device():
    layout = [("a", (3_000_001,)), ("b", (5,)), ("c", (1_000_003,))]
    like = E.ModelParams(layout)
    c = E.Checkpoint.zeros_like(like)
    enc = bytearray(E.encode_checkpoint(c))
    # last element of tensor "c" in the Nesterov buffer set (the very last float of the stream)
    tail = 8 + 8 + 4 + 32  # rng_seed, data_counter, shard, hash
    pos = len(enc) - tail - 4
    enc[pos: pos + 4] = np.array([np.inf], np.float32).tobytes()
    with pytest.raises(E.DecodeError, match="non-finite"):
        E.decode_checkpoint(bytes(enc), like=like)
