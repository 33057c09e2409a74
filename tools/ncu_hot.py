"""Summarize an ncu --set full report: stall reasons overall and by SASS opcode, and the hottest
instructions with their source line (needs -lineinfo). Usage: python tools/ncu_hot.py <rep> [top]"""
import collections
import csv
import io
import subprocess
import sys

def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
iS = h.index("Warp Stall Sampling (All Samples)")
iI = h.index("Instructions Executed")
iSrc = h.index("Source")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(num(r[iS]) for r in data)
print("samples", tot, "warp instructions", sum(num(r[iI]) for r in data))
agg = collections.Counter()
by = collections.defaultdict(collections.Counter)
for r in data:
    tok = r[iSrc].strip().split()
    if not tok:
        continue
    op = (tok[1] if tok[0].startswith("@") else tok[0]).split(".")[0]
    for c in reasons:
        v = num(r[h.index(c)])
        agg[c] += v
        by[op][c] += v
T = sum(agg.values()) or 1
print({k.replace("stall_", ""): round(v / T * 100, 1) for k, v in agg.most_common()})
for op, c in sorted(by.items(), key=lambda kv: -sum(kv[1].values()))[:15]:
    print(f"{op:12s} {sum(c.values()) / T * 100:5.1f}%", {k.replace('stall_', ''): round(v / T * 100, 1)
                                                         for k, v in c.most_common(3)})
print("--- hottest instructions")
for r in sorted(data, key=lambda r: -num(r[iS]))[:top]:
    print(f"{num(r[iS]) / tot * 100:5.2f}% {int(num(r[iI])):>10} {r[0][-5:]} {r[iSrc].strip()[:100]}")
