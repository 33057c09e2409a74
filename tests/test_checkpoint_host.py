"""CPU: checkpoint serialization (tensor.hpp:111-161,
checkpoint.hpp:19-68,190-224). Pins the oracle restatement to the
reference's bytes (golden fixture made by the UNMODIFIED reference), checks
SHA-256 (both host code paths) and every structural decode error of the
product library against the reference's verdicts. Structural errors are
decided on the host before any device work, so they run without a GPU."""
import ctypes as C
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ck():
    return np.load(os.path.join(ROOT, "tests", "golden", "checkpoint_cases.npz"))


@pytest.fixture(scope="module")
def capi():
    from paper_2412_01152_b200 import _capi
    if not os.path.exists(_capi.LIB_PATH):
        from paper_2412_01152_b200 import build
        build.build_product()
    return _capi


def layout_of(ck):
    return [(str(nm), tuple(int(e) for e in sh.split(",") if e)) for nm, sh in zip(ck["layout_names"],
                                                                                   ck["layout_shapes"])]


def view_of(capi, layout, arenas=(0, 0, 0, 0, 0)):
    names = (C.c_char_p * len(layout))(*[nm.encode() for nm, _ in layout])
    ranks = (C.c_uint32 * len(layout))(*[len(s) for _, s in layout])
    ext = [e for _, s in layout for e in s]
    c_ext = (C.c_uint32 * max(len(ext), 1))(*ext)
    v = capi.CheckpointView()
    v.ntensors = len(layout)
    v.names, v.ranks, v.extents = C.cast(names, C.c_void_p), C.cast(ranks, C.c_void_p), C.cast(c_ext, C.c_void_p)
    v.params, v.retained, v.adam_m, v.adam_v, v.nesterov_buf = arenas
    return v, (names, ranks, c_ext)


def test_oracle_restatement_matches_reference_bytes(ck):
    from oracle.pyoracle import checkpoint_encode, checkpoint_file_bytes
    sc = [int(x) for x in ck["scalars"]]
    enc = checkpoint_encode(layout_of(ck), list(ck["sets"]), sc[0], sc[1], sc[2], sc[3], sc[4],
                            ck["config_hash"].tobytes())
    assert enc == ck["encoded"].tobytes()
    assert checkpoint_file_bytes(enc) == ck["file_bytes"].tobytes()


def test_fixture_is_the_reference_output(ck):
    from oracle.pyoracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    R = Reference()
    sc = [int(x) for x in ck["scalars"]]
    enc = R.encode_checkpoint(layout_of(ck), list(ck["sets"]), *sc, ck["config_hash"].tobytes())
    assert enc == ck["encoded"].tobytes()
    for i, name in enumerate(ck["var_names"]):
        rc, msg, *_ = R.decode_checkpoint(ck[f"var_{i}"].tobytes(), ck["sets"].shape[1])
        assert (rc, msg) == (int(ck["var_codes"][i]), str(ck["var_msgs"][i])), name


@pytest.mark.parametrize("scalar", [False, True])
def test_sha256_matches_hashlib(capi, scalar):
    # the SHA-NI and the portable compression, in a fresh process each (the path is picked at load)
    code = ("import hashlib, os, sys; sys.path.insert(0, %r)\n"
            "import paper_2412_01152_b200 as E\n"
            "for n in [0, 1, 55, 56, 63, 64, 65, 119, 120, 128, 1000, 4096 + 17, 1 << 20]:\n"
            "    d = os.urandom(n)\n"
            "    assert E.sha256(d) == hashlib.sha256(d).digest(), n\n"
            "print('ok')\n") % ROOT
    env = dict(os.environ)
    if scalar:
        env["EMESH_SHA_SCALAR"] = "1"
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_sha256_matches_reference(capi):
    from oracle.pyoracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    import paper_2412_01152_b200 as E
    R = Reference()
    for n in (0, 3, 64, 1000, 123457):
        d = os.urandom(n)
        assert E.sha256(d) == R.sha256(d)


def test_probe_and_layout(capi, ck):
    import paper_2412_01152_b200 as E
    assert E.checkpoint_layout(ck["encoded"].tobytes()) == layout_of(ck)


def test_encoded_size(capi, ck):
    v, keep = view_of(capi, layout_of(ck))
    n = C.c_uint64()
    assert capi.lib().emesh_checkpoint_encoded_size(C.byref(v), C.byref(n)) == 0
    assert n.value == len(ck["encoded"])


def test_structural_errors_match_reference(capi, ck):
    """Every malformed variant whose verdict is reached before any data is
    uploaded: same error class and message as emesh::decode_checkpoint
    (non-finite-only variants need the device scan: tests/test_gpu_checkpoint.py)."""
    L = capi.lib()
    v, keep = view_of(capi, layout_of(ck))
    checked = 0
    for i, name in enumerate(ck["var_names"]):
        buf = ck[f"var_{i}"].tobytes()
        rc = L.emesh_checkpoint_decode(buf, len(buf), C.byref(v), None)
        if rc == capi.ECONFIG:  # structure valid: the verdict needs the device arenas
            assert str(ck["var_msgs"][i]) == "non-finite value in tensor payload", name
            continue
        assert (rc, capi.last_error()) == (int(ck["var_codes"][i]), str(ck["var_msgs"][i])), name
        checked += 1
    assert checked >= 15


def test_layout_mismatch_is_decode_error(capi, ck):
    lay = layout_of(ck)
    lay[2] = (lay[2][0], (8, 2))
    v, keep = view_of(capi, lay)
    buf = ck["encoded"].tobytes()
    assert capi.lib().emesh_checkpoint_decode(buf, len(buf), C.byref(v), None) == capi.EDECODE
    assert "differs" in capi.last_error()


def test_read_file_errors_without_device(capi, ck, tmp_path):
    L = capi.lib()
    v, keep = view_of(capi, layout_of(ck))
    assert L.emesh_checkpoint_read_file(str(tmp_path / "missing.bin").encode(), C.byref(v), None) == capi.EIO
    p = tmp_path / "trunc.bin"
    p.write_bytes(ck["file_bytes"].tobytes()[:30])
    assert L.emesh_checkpoint_read_file(str(p).encode(), C.byref(v), None) == capi.EDECODE
    p.write_bytes(ck["file_bytes"].tobytes()[:-5])
    assert L.emesh_checkpoint_read_file(str(p).encode(), C.byref(v), None) == capi.EDECODE
    bad = bytearray(ck["file_bytes"].tobytes())
    bad[60] ^= 0x5A  # test_checkpoint.cpp:56-62: one corrupted byte -> hash check fires
    p.write_bytes(bytes(bad))
    assert L.emesh_checkpoint_read_file(str(p).encode(), C.byref(v), None) == capi.EIO
    assert "hash mismatch" in capi.last_error()


def test_random_mutations_match_reference(capi, ck):
    """Seeded fuzz over the golden bytes (truncations, byte flips in the headers, u32 rewrites):
    every verdict reached on the host equals emesh::decode_checkpoint's (bytes.hpp:52-92 reader,
    tensor.hpp:122-154, checkpoint.hpp:49-66)."""
    from oracle.pyoracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    R = Reference()
    L = capi.lib()
    layout = layout_of(ck)
    v, keep = view_of(capi, layout)
    good = ck["encoded"].tobytes()
    n = ck["sets"].shape[1]
    rng = np.random.RandomState(1234)
    # header byte positions: every tensor record's name length, name, rank and extents
    hdr = []
    pos = 8
    for s_ in range(5):
        if s_ == 2:
            pos += 8
        pos += 4
        for nm, sh in layout:
            rec = 4 + len(nm.encode()) + 4 + 4 * len(sh)
            hdr.extend(range(pos, pos + rec))
            pos += rec + 4 * (int(np.prod(sh)) if sh else 1)
    checked = 0
    for it in range(300):
        b = bytearray(good)
        kind = it % 3
        if kind == 0:
            b = b[: rng.randint(0, len(good))]
        elif kind == 1:
            for _ in range(rng.randint(1, 4)):
                b[hdr[rng.randint(len(hdr))]] ^= 1 << rng.randint(8)
        else:
            at = hdr[rng.randint(len(hdr))]
            b[at: at + 4] = int(rng.choice([0, 1, 9, 1 << 20, 1 << 28, 0xFFFFFFFF])).to_bytes(4, "little")
        b = bytes(b)
        rc = L.emesh_checkpoint_decode(b, len(b), C.byref(v), None)
        ref_rc, ref_msg, *_ = R.decode_checkpoint(b, n)
        if rc == capi.ECONFIG:  # structurally valid: the verdict needs the device (the reference decoded or
            assert ref_rc in (0, 3), (it, ref_rc, ref_msg)  # found a non-finite value)
            continue
        if rc == capi.EDECODE and "differs from the destination" in capi.last_error():
            assert ref_rc == 0 or ref_msg == "non-finite value in tensor payload", (it, ref_msg)
            continue
        assert (rc, capi.last_error()) == (ref_rc, ref_msg), it
        checked += 1
    assert checked > 150
