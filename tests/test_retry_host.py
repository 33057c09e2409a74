"""allreduce_with_retry (allreduce.hpp:478-518) driver logic on CPU: the
reference's retry tests (test_allreduce.cpp:416-481) with a scripted
membership service and stand-in engines (the GPU path is exercised by
tests/test_gpu_nccl.py::test_retry_after_peer_stops)."""
import numpy as np
import pytest
import torch

import paper_2412_01152_b200 as E


class World:
    """k workers' inputs; an 'engine' for a plan returns the fp32 mean over the
    plan's members, or raises RingFailureError while a crashed member is in it."""

    def __init__(self, inputs):
        self.inputs = inputs
        self.crashed = set()
        self.built = []

    def make_engine(self, plan):
        world = self

        class Eng:
            n = len(world.inputs["w0"])
            mode = E.ReduceMode.int8

            def ring_allreduce(self, ins, outs, stream=None):
                dead = [m for m in plan.order if m in world.crashed]
                if dead:
                    raise E.RingFailureError(f"peer {dead[0]} stopped")
                acc = np.zeros_like(world.inputs["w0"])
                for m in plan.order:
                    acc = (acc + world.inputs[m]).astype(np.float32)
                outs[0].copy_(torch.from_numpy(acc / np.float32(len(plan.order))))

            def check(self):
                pass

            def close(self):
                pass

        self.built.append(list(plan.order))
        return Eng()


class ScriptedMesh:
    """Each epoch change evicts the crashed nodes (the coordinator's job)."""

    def __init__(self, world, state):
        self.world, self.state, self.reports = world, state, []

    def report_failure(self, node):
        self.reports.append(node)

    def wait_epoch_change(self, epoch, timeout):
        ring = [m for m in self.state.ring if m not in self.world.crashed]
        self.state = E.MeshState(epoch + 1, ring)
        return self.state

    def fetch_mesh(self):
        return self.state


def setup(k, crashed=()):
    inputs = {f"w{i}": np.full(8, float(i + 1), np.float32) for i in range(k)}
    w = World(inputs)
    w.crashed = set(crashed)
    st = E.MeshState(1, list(inputs))
    return w, ScriptedMesh(w, st), st


def job_for(w, me):
    return E.ReduceJob(1, torch.from_numpy(w.inputs[me].copy()))


def test_no_failure_returns_plain_result():
    w, mesh, st = setup(3)
    res = E.allreduce_with_retry(w.make_engine, mesh, st, "w0", job_for(w, "w0"))
    assert res.participants == 3 and res.attempts == 0 and res.epoch == 1
    assert np.allclose(res.value.numpy(), 2.0)


def test_crash_survivors_return_survivor_mean():
    w, mesh, st = setup(4, crashed=["w2"])
    job = job_for(w, "w0")
    before = job.input.clone()
    res = E.allreduce_with_retry(w.make_engine, mesh, st, "w0", job)
    assert res.participants == 3 and res.attempts == 1 and res.epoch == 2
    assert np.array_equal(res.value.numpy(), np.full(8, (1 + 2 + 4) / 3, np.float32))
    assert torch.equal(job.input, before)  # the input is preserved across retries
    assert w.built == [["w0", "w1", "w2", "w3"], ["w0", "w1", "w3"]]


def test_retry_cap_exhaustion_is_fatal():
    w, mesh, st = setup(3, crashed=["w1"])

    class Stuck(ScriptedMesh):
        def wait_epoch_change(self, epoch, timeout):
            raise TimeoutError

    m = Stuck(w, st)
    with pytest.raises(E.FatalError, match="retries"):
        E.allreduce_with_retry(w.make_engine, m, st, "w0", job_for(w, "w0"), E.ReduceOptions(max_retries=1))


def test_evicted_self_is_fatal():
    w, mesh, st = setup(2)
    with pytest.raises(E.FatalError, match="no longer in the mesh"):
        E.allreduce_with_retry(w.make_engine, mesh, E.MeshState(3, ["w1"]), "w0", job_for(w, "w0"))
