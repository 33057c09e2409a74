"""Config 4: all-reduce message-size sweep, fp32 payload 1 MB .. 4 GB, at the launched
world size: this repo's int8 ring and fp32 ring (peer transport) vs NCCL's fp32 all-reduce
(ncclAllReduce sum + scale) on identical inputs. Device time (CUDA events), max over ranks.
torchrun --nproc-per-node N tools/sweep_msg.py [max_elems] [reps]"""
import json
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
max_n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 30
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
S = 4  # reference default pipeline_subchunks


def timed(fn):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


n = 1 << 18
rows = []
while n <= max_n:
    x = torch.rand(n, device=dev) * 2 - 1
    out = torch.empty(n + 4, device=dev)[:n]
    res = {"elems": n, "fp32_MB": 4 * n / 2**20}
    for mode in ("int8", "fp32"):
        obj = [E.RingEngine.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng = E.RingEngine(n, world, rank=rank, opts=E.ReduceOptions(pipeline_subchunks=S), nccl_id=obj[0],
                           mode=E.ReduceMode[mode])
        ms = timed(lambda: eng.ring_allreduce([x], [out]))
        res[f"ours_{mode}_ms"] = ms
        res["transport"] = eng.transport
        eng.close()
    y = x.clone()

    def nccl():  # ncclAllReduce(float, ncclAvg), in place
        dist.all_reduce(y, op=dist.ReduceOp.AVG)

    res["nccl_fp32_ms"] = timed(nccl)
    for key in ("ours_int8", "ours_fp32", "nccl_fp32"):
        t = res[f"{key}_ms"] / 1e3
        res[f"{key}_algbw_GBs"] = 4 * n / t / 1e9
        res[f"{key}_busbw_GBs"] = 2 * (world - 1) / world * 4 * n / t / 1e9
    rows.append(res)
    if rank == 0:
        print(json.dumps(res), flush=True)
    del x, out, y
    torch.cuda.empty_cache()
    n *= 4
dist.barrier()
dist.destroy_process_group()
