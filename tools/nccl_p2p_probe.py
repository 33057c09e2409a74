"""NCCL ring-shift bandwidth (each rank sends B bytes to rank+1, receives from rank-1), one
communicator vs several in parallel (the payload split across them), device time, max over ranks.
torchrun --nproc-per-node N tools/nccl_p2p_probe.py"""
import os

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dev = torch.device("cuda", torch.cuda.current_device())
dist.init_process_group("nccl", device_id=dev)
succ, pred = (rank + 1) % world, (rank - 1) % world
B = 64 << 20
groups = {1: [dist.group.WORLD]}
for c in (2, 4, 8):
    groups[c] = [dist.new_group(list(range(world))) for _ in range(c)]
src = torch.randint(0, 255, (B,), dtype=torch.uint8, device=dev)
dst = torch.empty_like(src)
streams = [torch.cuda.Stream() for _ in range(8)]


def shift(c):
    n = B // c
    evs = []
    cur = torch.cuda.current_stream()
    for i, g in enumerate(groups[c]):
        s = streams[i]
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            ops = [dist.P2POp(dist.isend, src[i * n:(i + 1) * n], succ, group=g),
                   dist.P2POp(dist.irecv, dst[i * n:(i + 1) * n], pred, group=g)]
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        cur.wait_stream(s)


for c in (1, 2, 4, 8):
    for _ in range(3):
        shift(c)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        shift(c)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 10], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"{c} communicator(s): {t.item():.3f} ms per 64 MB shift = {B / t.item() / 1e6:.0f} GB/s per direction", flush=True)
dist.destroy_process_group()
