"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in data:
    name = r[ki].split("(")[0][:70]
    v = float(r[vi]) * (1e-3 if r[ui] == "ns" else 1.0 if r[ui] == "us" else 1e3) / 1e3  # -> ms
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:70s} n={n:5d} total={ms:9.3f} ms share={ms / tot:.3f}")
