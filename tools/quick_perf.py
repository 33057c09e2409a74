"""Quick per-kernel-family timing on one GPU (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2412_01152_b200 as E

def timeit(fn, iters=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3

dev = "cuda:0"
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 28
x = (torch.randn(n, device=dev) * 1e-3).contiguous()
q = E.quantize(x)
t = timeit(lambda: E.quantize(x))
print(f"quantize n={n}: {t*1e3:.3f} ms  {5*n/t/1e9:.1f} GB/s alg (5 B/elem)")
t = timeit(lambda: E.dequantize(q))
print(f"dequantize: {t*1e3:.3f} ms  {5*n/t/1e9:.1f} GB/s")
P = E.ModelParams({"w": (n,)}); L = E.ModelParams({"w": (n,)})
t = timeit(lambda: E.compute_pseudo_gradient(P, L))
print(f"pseudo_grad: {t*1e3:.3f} ms {12*n/t/1e9:.1f} GB/s")
for k in (1, 2, 4):
    N = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1 << 28
    eng = E.RingEngine(N, k, opts=E.ReduceOptions(pipeline_subchunks=16), virtual=(k > 1))
    tg = [torch.randn(N, device=dev) for _ in range(k)]
    tl = [a - 1e-3 * torch.randn(N, device=dev) for a in tg]
    tb = [torch.zeros(N, device=dev) for _ in range(k)]
    t = timeit(lambda: eng.outer_sync(tg, tl, tb, write_local=False), iters=3, warm=1)
    eng.check()
    A = 20 if k == 1 else 24 + (2*k-1)/k + 1
    print(f"outer_sync virtual k={k} N={N}: {t*1e3:.2f} ms  {k*N/t/1e9:.2f} Gparam/s  alg {k*N*A/t/1e9:.0f} GB/s")
    eng.close(); del tg, tl, tb
