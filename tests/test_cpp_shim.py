"""The C++ drop-in (include/emesh_b200.hpp): emesh::b200::* against the
reference's own emesh::* functions, bit for bit (tests/cpp/shim_test.cpp,
built against the reference headers by build() / tests/cpp/Makefile)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "shim_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/_bin/shim_test not built (needs the reference headers)")
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_cpp_dropin_matches_reference_functions():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "cpp shim OK" in out.stdout
