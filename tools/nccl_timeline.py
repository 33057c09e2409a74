"""NCCL-ring op timeline of one outer-sync round (development aid).
torchrun --nproc-per-node N tools/nccl_timeline.py [n] [window] [S]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2412_01152_b200 as E  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
lr = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(lr)
dev = torch.device("cuda", lr)
dist.init_process_group("nccl", device_id=dev)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
win = int(float(sys.argv[2])) if len(sys.argv) > 2 else 0
S = int(sys.argv[3]) if len(sys.argv) > 3 else 16
transport = sys.argv[4] if len(sys.argv) > 4 else "nccl"
obj = [E.RingEngine.unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
eng = E.RingEngine(n, world, rank=rank, opts=E.ReduceOptions(pipeline_subchunks=S), nccl_id=obj[0], window_elems=win,
                   transport=transport)
tg = torch.rand(n, device=dev) * 2 - 1
tl = tg - (torch.rand(n, device=dev) * 2 - 1) * 2 ** -10
tb = torch.zeros(n, device=dev)
for _ in range(3):
    eng.outer_sync([tg], [tl], [tb], write_local=False)
torch.cuda.synchronize()
dist.barrier()
eng.profile(True)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time  # noqa: E402
t0 = time.perf_counter()
ev0.record()
eng.outer_sync([tg], [tl], [tb], write_local=False)
t1 = time.perf_counter()
ev1.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"rank {rank}: host enqueue {1e3 * (t1 - t0):.3f} ms, enqueue+drain {1e3 * (t2 - t0):.3f} ms", flush=True)
rows = eng.timeline()
names = {0: "OWN", 1: "XFER", 2: "QUANT", 3: "APPLY"}
if rank == 0:
    print(f"world={world} n={n} window={win} S={S} transport={transport} round {ev0.elapsed_time(ev1):.3f} ms; ops {len(rows)}")
    for kd, ph, hop, w, t0, t1 in rows:
        print(f"  {names.get(int(kd), kd):5s} ph{int(ph)} hop{int(hop):2d} w{int(w)}  {t0:8.3f} -> {t1:8.3f}  ({t1 - t0:6.3f})")
dist.barrier()
dist.destroy_process_group()
