"""Task timeline of the persistent quantizer for one virtual-ring round
(development aid: emesh_trace_enable / emesh_trace_read)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_01152_b200 as E  # noqa: E402
from paper_2412_01152_b200 import _capi  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 256_000_000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 64
k = 4
eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=True)
tg = [torch.rand(n, device="cuda") * 2 - 1 for _ in range(k)]
tl = [a - (torch.rand(n, device="cuda") * 2 - 1) * 2 ** -10 for a in tg]
tb = [torch.zeros(n, device="cuda") for _ in range(k)]
eng.outer_sync(tg, tl, tb, write_local=False)
torch.cuda.synchronize()
L = _capi.lib()
L.emesh_trace_enable(1 << 20)
eng.outer_sync(tg, tl, tb, write_local=False)
torch.cuda.synchronize()
rec = np.zeros(1 << 20, dtype=[("t", "<u8", 4), ("kind", "<u4"), ("seg", "<u4"), ("tile", "<u4"), ("sm", "<u4")])
m = L.emesh_trace_read(rec.ctypes.data, len(rec))
rec = rec[:m]
L.emesh_trace_enable(0)
order = np.argsort(rec["t"][:, 0])
rec = rec[order]
t = rec["t"].astype(np.int64)
t0 = t[:, 0].min()
st = rec["kind"] == 0
bn = rec["kind"] == 2
dur = (t[:, 3] - t[:, 0]) / 1e3
wait = (t[:, 1] - t[:, 0]) / 1e3
main = (t[:, 2] - t[:, 1]) / 1e3
epi = (t[:, 3] - t[:, 2]) / 1e3
print(f"n={n} S={S}: records {m}; span {(t[:, 3].max() - t0) / 1e3:.1f} us")
for kd, nm in ((0, "stats"), (2, "bin")):
    msk = rec["kind"] == kd
    if msk.sum() == 0:
        continue
    line = (f"{nm:5s} n={msk.sum():6d} dur mean {dur[msk].mean():6.2f} us p50 {np.percentile(dur[msk], 50):.2f} "
            f"p90 {np.percentile(dur[msk], 90):.2f} max {dur[msk].max():.2f} | wait mean {wait[msk].mean():6.2f} max {wait[msk].max():.2f}")
    if kd in (0, 2):
        line += f" | main {main[msk].mean():6.2f} epilogue {epi[msk].mean():6.2f}"
    print(line)
ends = np.maximum.accumulate(t[:, 3])
gaps = np.nonzero(t[1:, 0] > ends[:-1] + 2000)[0]
bounds = [0] + list(gaps + 1) + [len(t)]
spans = [(t[b:e, 3].max() - t[b, 0]) / 1e3 for b, e in zip(bounds[:-1], bounds[1:])]
print("launch groups", len(spans), "span us: mean %.1f min %.1f max %.1f" % (np.mean(spans), np.min(spans), np.max(spans)))
print("sum of spans %.1f us; idle between %.1f us" % (np.sum(spans), (t[:, 3].max() - t0) / 1e3 - np.sum(spans)))
b, e = bounds[int(np.argmax(spans))], bounds[int(np.argmax(spans)) + 1]
g = t[b:e]
grid = np.linspace(g[:, 0].min(), g[:, 3].max(), 40)
conc = [int(((g[:, 0] <= x) & (g[:, 3] > x)).sum()) for x in grid]
print("concurrent tasks over the longest launch:", conc)
# time-weighted breakdown: SM-time spent per kind and in waits
tot = dur.sum()
for kd, nm in ((0, "stats"), (2, "bin")):
    msk = rec["kind"] == kd
    print(f"  {nm:5s} share of task time {dur[msk].sum() / tot:.3f} (waiting {wait[msk].sum() / tot:.3f})")
# kind mix over time inside the longest launch: share of running tasks that are STATS
kinds = rec["kind"][b:e]
mix = []
for x in grid:
    run = (g[:, 0] <= x) & (g[:, 3] > x)
    mix.append(round(float((kinds[run] == 0).mean()), 2) if run.any() else None)
print("STATS share of running tasks over the longest launch:", mix)
# grid utilization per launch group: busy CTA-time / (grid slots x span)
grid_slots = 444
util = []
for b0, e0 in zip(bounds[:-1], bounds[1:]):
    gg = t[b0:e0]
    span = gg[:, 3].max() - gg[:, 0].min()
    util.append(float((gg[:, 3] - gg[:, 0]).sum()) / (grid_slots * span))
print("grid utilization per launch: mean %.3f min %.3f max %.3f" % (np.mean(util), np.min(util), np.max(util)))
