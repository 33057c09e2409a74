"""Run under torchrun on 2+ GPUs (tests/test_gpu_nccl.py): the last rank stops
participating after the engine is built (a crashed peer); the others'
peer-transport waits time out (step_timeout), the round reports
RingFailureError, and allreduce_with_retry re-runs the job over the survivors
from the preserved input (allreduce.hpp:485-518). Exit 0 iff the survivors
get the survivor mean, bit-exact vs the oracle."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle  # noqa: E402  (checker)
import paper_2412_01152_b200 as E  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(90, exit=True)  # a hang fails the test with a stack, not a timeout
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    dist.init_process_group("nccl", device_id=dev)
    store = dist.distributed_c10d._get_default_store()
    O = Oracle()
    transport = sys.argv[1] if len(sys.argv) > 1 else "p2p"
    n, S = 300_007, 4
    ids = [f"r{i}" for i in range(world)]
    crashed = ids[-1]
    ins = {ids[w]: O.uniform(n, 90, w, 0, 0, 2.0 ** -6) for w in range(world)}
    opts = E.ReduceOptions(pipeline_subchunks=S, step_timeout=2.0, max_retries=2)

    def make_engine(plan):
        k = len(plan.order)
        print(f"{ids[rank]}: building engine for epoch {plan.epoch}, k={k}", flush=True)
        uid = None
        if k > 1:  # survivors exchange a fresh NCCL id through the store, keyed by epoch
            key = f"uid/{plan.epoch}"
            if plan.self_index == 0:
                uid = E.RingEngine.unique_id()
                store.set(key, uid)
            else:
                uid = bytes(store.get(key))
        return E.RingEngine(n, k, rank=plan.self_index, opts=opts, nccl_id=uid, transport=transport, plan=plan)

    class Mesh:  # the coordinator's view: the crashed rank is evicted at the next epoch
        def __init__(self):
            self.state = E.MeshState(1, list(ids))

        def report_failure(self, node):
            reported.append(node)

        def wait_epoch_change(self, epoch, timeout):
            self.state = E.MeshState(epoch + 1, [m for m in self.state.ring if m != crashed])
            return self.state

        def fetch_mesh(self):
            return self.state

    me = ids[rank]
    ok = True
    reported = []
    if me == crashed:
        # build the first engine with everyone (collective), then stop participating
        eng = make_engine(E.RingPlan.from_mesh(E.MeshState(1, list(ids)), me, 1))
        time.sleep(0.5)
        store.set("crashed_ready", b"1")
        store.get("survivors_done")  # stay alive (our memory stays mapped) until they finish
        print(f"{me}: released", flush=True)
        os._exit(0)  # a crash: no engine teardown, no collective goodbye
    else:
        job = E.ReduceJob(1, torch.from_numpy(ins[me]).to(dev))
        before = job.input.clone()
        res = E.allreduce_with_retry(make_engine, Mesh(), E.MeshState(1, list(ids)), me, job, opts)
        want = O.ring_allreduce([ins[m] for m in ids if m != crashed], S, "int8")
        got = res.value.cpu().numpy()
        if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
            print(f"{me}: survivor mean MISMATCH", flush=True)
            ok = False
        if res.participants != world - 1 or res.attempts != 1 or not torch.equal(job.input, before):
            print(f"{me}: participants {res.participants} attempts {res.attempts}", flush=True)
            ok = False
        # the culprit travels with the failure (allreduce.hpp:341-359, :505-506): poisoned peer flags
        # name it on the peer transport; an NCCL wait knows it only with a single peer (else unknown)
        want = [[crashed]] if transport == "p2p" or world == 2 else [[], [crashed]]
        if reported not in want:
            print(f"{me}: reported {reported}, expected [{crashed!r}]", flush=True)
            ok = False
        if rank == 0:
            store.set("survivors_done", b"1")
        print(f"{me}: retry {'OK' if ok else 'FAILED'} [{transport}]", flush=True)
        os._exit(0 if ok else 1)  # the crashed peer is gone: no collective teardown


if __name__ == "__main__":
    main()
