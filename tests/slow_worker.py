"""Run under torchrun on 2+ GPUs (tests/test_gpu_nccl.py): every rank runs an
on-time outer-sync round, then another that the last rank starts only after twice step_timeout
(alive, just late). The reference unwinds such an attempt on every rank
(abort frames carry the culprit, allreduce.hpp:341-359; Nesterov is applied
only to a completed all-reduce, trainer.hpp:375-381). Here: every rank must
report RingFailureError, and NO rank may have committed anything: theta_g,
momentum and theta_l bit-identical to their values before the round.
Exit 0 iff that holds on this rank."""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_01152_b200 as E  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(120, exit=True)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    dist.init_process_group("nccl", device_id=dev)
    store = dist.distributed_c10d._get_default_store()
    transport = sys.argv[1] if len(sys.argv) > 1 else "p2p"
    n, S, timeout = 1_000_003, 4, 2.0
    ids = [f"r{i}" for i in range(world)]
    plan = E.RingPlan.from_mesh(E.MeshState(1, list(ids)), ids[rank], 1)
    uid = [E.RingEngine.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    eng = E.RingEngine(n, world, rank=rank, opts=E.ReduceOptions(pipeline_subchunks=S, step_timeout=timeout),
                       nccl_id=uid[0], transport=transport, plan=plan)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    tg = torch.rand(n + 8, device=dev, generator=g)[:n]
    tl = (tg - 1e-3 * torch.rand(n + 8, device=dev, generator=g)[:n]).contiguous()
    tb = torch.rand(n + 8, device=dev, generator=g)[:n]
    # one on-time round first: NCCL connects send/recv peers lazily at their first use, and an
    # engine's first round waits with a setup floor over step_timeout; the late round is a later one
    eng.outer_sync([tg], [tl], [tb], E.HyperParams(), write_local=True)
    eng.check()
    before = [t.clone() for t in (tg, tl, tb)]
    dist.barrier()
    torch.cuda.synchronize()
    if rank == world - 1:
        time.sleep(2 * timeout)  # alive, but later than every peer's step_timeout
    failed, culprit = False, None
    try:
        eng.outer_sync([tg], [tl], [tb], E.HyperParams(), write_local=True)
        eng.check()
    except E.RingFailureError as ex:
        failed, culprit = True, ex.failed_node
        print(f"{ids[rank]}: RingFailureError (culprit {culprit!r}): {ex}", flush=True)
    torch.cuda.synchronize()
    untouched = all(torch.equal(a, b) for a, b in zip((tg, tl, tb), before))
    # the on-time ranks name the late one (or nobody); the late rank itself sees its peers gone
    ok = failed and untouched and (rank == world - 1 or culprit in (ids[-1], ""))  # "" = unknown
    print(f"{ids[rank]}: slow-peer {'OK' if ok else 'FAILED'} [{transport}] failed={failed} untouched={untouched}",
          flush=True)
    store.set(f"done/{rank}", b"1")
    for q in range(world):  # nobody tears down mapped memory while a peer may still read it
        store.get(f"done/{q}")
    os._exit(0 if ok else 1)


if __name__ == "__main__":
    main()
