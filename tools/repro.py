import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2412_01152_b200 as E
for (n, k, S) in [(100003, 2, 4), (100003, 4, 4), (48000011, 2, 2)]:
    try:
        dev = torch.device('cuda:0')
        g = torch.rand(n + 8, device=dev)[:n]
        ls = [torch.rand(n + 8, device=dev)[:n] for _ in range(k)]
        eng = E.RingEngine(n, k, opts=E.ReduceOptions(pipeline_subchunks=S), virtual=True)
        tg = [g.clone() for _ in range(k)]; tb = [torch.zeros_like(g) for _ in range(k)]
        eng.outer_sync(tg, ls, tb, E.HyperParams(), write_local=False)
        eng.check(); print(n, k, S, 'ok', flush=True)
    except Exception as ex:
        print(n, k, S, 'FAIL', ex, flush=True); break
