"""The C++ drop-in's allreduce_with_retry (include/emesh_b200.hpp) against the
reference's retry contract (allreduce.hpp:485-518, test_allreduce.cpp:416-481),
host-only: scripted engines and mesh (tests/cpp/retry_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "retry_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/_bin/retry_test not built (needs the reference headers)")
def test_cpp_allreduce_with_retry_contract():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "cpp retry OK" in out.stdout
