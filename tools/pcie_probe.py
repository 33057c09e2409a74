"""Host<->device copy bandwidth: H2D alone, D2H alone, both at once (pinned)."""
import torch, time
n = 1 << 30  # 4 GB fp32
h1 = torch.empty(n, pin_memory=True); h2 = torch.empty(n, pin_memory=True)
d1 = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both(): h2d(); d2h()
a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {4*n/a/1e9:.1f} GB/s  D2H {4*n/b/1e9:.1f} GB/s  both {8*n/c/1e9:.1f} GB/s aggregate ({c*1e3:.0f} ms vs {a*1e3:.0f}+{b*1e3:.0f})")
