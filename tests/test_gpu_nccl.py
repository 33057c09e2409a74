"""Multi-GPU: the NCCL ring engine (one DiLoCo worker per GPU) bit-exact vs
the oracle, launched with torchrun on every visible GPU (skips below 2)."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_nccl_ring_parity():
    n = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "tests", "nccl_parity_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "NCCL parity OK" in out.stdout


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_retry_after_peer_stops(transport):
    """allreduce_with_retry: a peer stops mid-collective, the survivors time out (RingFailureError; the
    peer transport's device-side wait budget, or the bounded NCCL wait + communicator abort), re-plan and
    return the survivor mean (test_allreduce.cpp:431-445 analogue)."""
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29534" if transport == "p2p" else "29535",
           os.path.join(ROOT, "tests", "retry_worker.py"), transport]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert out.stdout.count("retry OK") == n - 1


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_slow_peer_fails_every_rank_and_commits_nothing(transport):
    """a peer alive but later than step_timeout. The ranks that time out poison the
    flags they still owe (the peer transport) or abort the communicator (NCCL), so EVERY rank, the
    late one included, reports RingFailureError, and the round's commit gate leaves theta_g /
    momentum / theta_l untouched everywhere (allreduce_with_retry can restart from them)."""
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29536" if transport == "p2p" else "29537",
           os.path.join(ROOT, "tests", "slow_worker.py"), transport]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert out.stdout.count("slow-peer OK") == n
