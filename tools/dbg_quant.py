import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2412_01152_b200 as E
from oracle.pyoracle import Oracle
O = Oracle()
g = np.load('tests/golden/quant_cases.npz')
for name in ["normal_10k", "normal_4096", "uniform_1e-3", "two_point"]:
    x = g[f"{name}/x"]
    q = E.quantize(torch.from_numpy(x).cuda())
    c = q.indices.cpu().numpy(); cb = q.codebook.cpu().numpy(); st = q.stats.cpu().numpy()
    oc, ocb, ost = O.quantize(x)
    d = np.nonzero(c != oc)[0]
    print(name, "ndiff", len(d), "cbdiff", int((cb.view(np.uint32) != ocb.view(np.uint32)).sum()), "stats", st, ost)
    for i in d[:5]:
        print("   i", i, "x", x[i], "got", c[i], "want", oc[i], "q", (np.float64(x[i]) - ost[2]) / ost[3])
