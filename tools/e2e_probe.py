"""outer_sync_host timing vs raw PCIe copies of the same bytes (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_01152_b200 as E
n, k = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000, 4
eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=16), virtual=True)
hp = E.HyperParams()
hg = [torch.randn(n).pin_memory() for _ in range(k)]
hl = [(a - 1e-3).pin_memory() for a in hg]
hb = [torch.zeros(n).pin_memory() for _ in range(k)]
eng.outer_sync_host(hg, hl, hb, hp, write_local=False)
for rep in range(3):
    t0 = time.perf_counter(); eng.outer_sync_host(hg, hl, hb, hp, write_local=False); t = time.perf_counter() - t0
    print(f"outer_sync_host {t*1e3:.0f} ms  {k*n/t/1e9:.2f} Gparam/s  ({os.environ.get('EMESH_HOST_SERIAL') and 'serial' or 'pipelined'})")
eng.close()
d = [torch.empty(n, device="cuda") for _ in range(3 * k)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
hs = hg + hl + hb
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1):
    for a, b in zip(d, hs): a.copy_(b, non_blocking=True)
torch.cuda.synchronize(); t_up = time.perf_counter() - t0
t0 = time.perf_counter()
with torch.cuda.stream(s2):
    for a, b in zip(hg + hb, d[:2 * k]): a.copy_(b, non_blocking=True)
torch.cuda.synchronize(); t_dn = time.perf_counter() - t0
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    for a, b in zip(d, hs): a.copy_(b, non_blocking=True)
with torch.cuda.stream(s2):
    for a, b in zip(hg + hb, d[:2 * k]): a.copy_(b, non_blocking=True)
torch.cuda.synchronize(); t_both = time.perf_counter() - t0
print(f"raw: up {12*k*n/1e9:.0f} GB {t_up*1e3:.0f} ms ({12*k*n/t_up/1e9:.1f} GB/s), down {8*k*n/1e9:.0f} GB {t_dn*1e3:.0f} ms, both {t_both*1e3:.0f} ms")
