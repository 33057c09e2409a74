"""Run under torchrun (one rank per GPU): the NCCL ring engine vs the oracle.
Used by tests/test_gpu_nccl.py. Exit code 0 iff every check passes."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle  # noqa: E402  (checker)
import paper_2412_01152_b200 as E  # noqa: E402


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    dist.init_process_group("nccl", device_id=dev)
    O = Oracle()
    ok = True
    cases = [(100_003, 4, 0), (4099, 3, 1), (5, 4, 0), (3, 4, 0), (2_000_000, 8, 300_000)]
    runs = [(c, t, m) for m in ("int8", "fp32") for t in ("nccl", "p2p") for c in cases]
    for (n, S, window), transport, mode in runs:
        obj = [E.RingEngine.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng = E.RingEngine(n, world, rank=rank, opts=E.ReduceOptions(pipeline_subchunks=S), nccl_id=obj[0],
                           window_elems=window, transport=transport, mode=E.ReduceMode[mode])
        if eng.transport != transport:
            print(f"rank {rank}: asked for {transport}, engine runs {eng.transport}", flush=True)
            ok = False
        ins = [O.uniform(n, 7 + n, w, 0, 0, 2.0 ** -6) for w in range(world)]
        want = O.ring_allreduce(ins, S, mode)
        out = torch.empty(n + 4, dtype=torch.float32, device=dev)[:n]
        eng.ring_allreduce([torch.from_numpy(ins[rank]).to(dev)], [out])
        eng.check()
        got = out.cpu().numpy()
        if not np.array_equal(bits(got), bits(want)):
            print(f"rank {rank}: [{transport} {mode}] ring n={n} S={S} MISMATCH ({int((bits(got) != bits(want)).sum())} elems)", flush=True)
            ok = False
        # two outer-sync rounds (trainer.hpp:355-382)
        g = O.uniform(n, 3, 0)
        b = np.zeros(n, np.float32)
        tg = torch.from_numpy(g).to(dev)
        tb = torch.from_numpy(b).to(dev)
        eg, eb = g, b
        for rnd in range(2):
            ls = [(eg - O.uniform(n, 30 + rnd, 1 + w, 0, 0, 2.0 ** -10)).astype(np.float32) for w in range(world)]
            eng.outer_sync([tg], [torch.from_numpy(ls[rank]).to(dev)], [tb], E.HyperParams(), write_local=False)
            eng.check()
            eg, eb = O.outer_sync(eg, ls, eb, S, mode, 0.7, 0.9)
            if not (np.array_equal(bits(tg.cpu().numpy()), bits(eg)) and np.array_equal(bits(tb.cpu().numpy()), bits(eb))):
                print(f"rank {rank}: [{transport} {mode}] outer sync n={n} round {rnd} MISMATCH", flush=True)
                ok = False
        # a third round through the host-buffer entry point (chunk-pipelined copies)
        ls = [(eg - O.uniform(n, 40, 1 + w, 0, 0, 2.0 ** -10)).astype(np.float32) for w in range(world)]
        hg = torch.from_numpy(tg.cpu().numpy().copy()).pin_memory()
        hb = torch.from_numpy(tb.cpu().numpy().copy()).pin_memory()
        hl = torch.from_numpy(ls[rank].copy()).pin_memory()
        eng.outer_sync_host([hg], [hl], [hb], E.HyperParams(), write_local=True)
        eg, eb = O.outer_sync(eg, ls, eb, S, mode, 0.7, 0.9)
        if not (np.array_equal(bits(hg.numpy()), bits(eg)) and np.array_equal(bits(hb.numpy()), bits(eb))
                and np.array_equal(bits(hl.numpy()), bits(eg))):
            print(f"rank {rank}: [{transport} {mode}] outer_sync_host n={n} MISMATCH", flush=True)
            ok = False
        eng.close()
    # multi-tensor engine (config 5): one ReduceJob per tensor, chunks bucketed per hop
    sizes = [4096, 17, 0, 100_003, 1, 65_536, 3, 250_000]
    n = sum(sizes)
    off = np.concatenate([[0], np.cumsum(sizes)])
    for transport in ("nccl", "p2p"):
        for mode in ("int8", "fp32"):
            obj = [E.RingEngine.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            eng = E.RingEngine(n, world, rank=rank, opts=E.ReduceOptions(pipeline_subchunks=4), nccl_id=obj[0],
                               transport=transport, mode=E.ReduceMode[mode], tensor_sizes=sizes,
                               window_elems=100_000)
            ins = [O.uniform(n, 78, w, 0, 0, 2.0 ** -4) for w in range(world)]
            want = np.concatenate([O.ring_allreduce([a[off[t]:off[t + 1]] for a in ins], 4, mode)[:sizes[t]]
                                   for t in range(len(sizes))])
            out = torch.empty(n + 4, dtype=torch.float32, device=dev)[:n]
            for _ in range(3):  # several rounds: parity buffers / epochs
                eng.ring_allreduce([torch.from_numpy(ins[rank]).to(dev)], [out])
            eng.check()
            if not np.array_equal(bits(out.cpu().numpy()), bits(want)):
                print(f"rank {rank}: [{transport} {mode}] multi-tensor ring MISMATCH", flush=True)
                ok = False
            eng.close()
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    dist.destroy_process_group()
    if rank == 0:
        print("NCCL parity", "OK" if flag.item() == 0 else "FAILED", flush=True)
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
