"""Latency of one quantizer launch at small sizes (the small-round critical path): emesh_quantize_segments
on n elements in S segments, CUDA events over many back-to-back calls on one stream (device time per
call, includes the workspace memset and the launch gap)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_01152_b200 import _capi  # noqa: E402
from paper_2412_01152_b200.emesh import _check  # noqa: E402

L = _capi.lib()
st = torch.cuda.current_stream()
P = C.POINTER(C.c_uint64)
for n, S in [(8192, 1), (65536, 1), (65536, 4), (1 << 20, 4), (1 << 22, 4), (1 << 24, 4)]:
    x = (torch.rand(n, device="cuda") - 0.5) * 0.01
    codes = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    cbs = torch.empty(S * 256, dtype=torch.float32, device="cuda")
    lo = np.array([i * n // S for i in range(S)], np.uint64)
    ln = np.array([(i + 1) * n // S - i * n // S for i in range(S)], np.uint64)

    def q():
        _check(L.emesh_quantize_segments(x.data_ptr(), lo.ctypes.data_as(P), ln.ctypes.data_as(P), S, codes.data_ptr(),
                                         cbs.data_ptr(), None, C.c_void_p(st.cuda_stream)))
    for _ in range(20):
        q()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 200
    e0.record()
    for _ in range(reps):
        q()
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n} S={S}: {1e3 * e0.elapsed_time(e1) / reps:.1f} us per quantize launch", flush=True)
