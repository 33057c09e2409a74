"""NVLink evidence for the peer-memory ring, from ONE process driving two GPUs (so ncu may
profile it; NVML's NVLink counters are not exposed on these boxes, r02_nvlink_probe).

The peer transport's hop kernels are the product quantizer storing its payload (codes +
codebooks) straight into the successor GPU's arena, and the decode reading the owner's bytes.
Here the same library entry points run on cuda:0 with the payload arena on cuda:1 (peer access
enabled), at the bench's batch shape (one 250M-element chunk, 16 segments):

  quant_local   codes/codebooks on cuda:0 (the 1-GPU reference time)
  quant_peer    codes/codebooks on cuda:1: every code byte crosses NVLink as a store
  dequant_peer  codes/codebooks on cuda:1, output on cuda:0: every code byte crosses as a load

Prints CUDA-event times (no profiler) and the algorithmic NVLink bytes; under
`ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,...` the same launches give the link counters."""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_01152_b200 import _capi  # noqa: E402
from paper_2412_01152_b200.emesh import _check  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=250_000_000)
    ap.add_argument("--segments", type=int, default=16)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    n, S = args.n, args.segments
    torch.cuda.set_device(0)
    rt = C.CDLL("libcudart.so.12")
    rt.cudaSetDevice(0)
    rc = rt.cudaDeviceEnablePeerAccess(1, 0)
    assert rc in (0, 704), f"cudaDeviceEnablePeerAccess: {rc}"  # 704: already enabled
    g = torch.Generator(device="cuda:0")
    g.manual_seed(1)
    x = (torch.rand(n, device="cuda:0", generator=g) - 0.5).mul_(2.0 ** -8)
    lo = np.array([i * n // S for i in range(S)], np.uint64)
    ln = np.array([(i + 1) * n // S - i * n // S for i in range(S)], np.uint64)
    P = C.POINTER(C.c_uint64)
    arenas = {dev: (torch.empty(n + 64, dtype=torch.uint8, device=dev),
                    torch.empty(S * 256, dtype=torch.float32, device=dev)) for dev in ("cuda:0", "cuda:1")}
    out = torch.empty(n, dtype=torch.float32, device="cuda:0")
    stream = torch.cuda.current_stream(0)
    L = _capi.lib()

    def quant(dev):
        codes, cbs = arenas[dev]
        _check(L.emesh_quantize_segments(x.data_ptr(), lo.ctypes.data_as(P), ln.ctypes.data_as(P), S,
                                         codes.data_ptr(), cbs.data_ptr(), None, C.c_void_p(stream.cuda_stream)))

    def dequant(dev):
        codes, cbs = arenas[dev]
        _check(L.emesh_dequantize_segments(codes.data_ptr(), cbs.data_ptr(), lo.ctypes.data_as(P),
                                           ln.ctypes.data_as(P), S, out.data_ptr(), C.c_void_p(stream.cuda_stream)))

    cases = [("quant_local", lambda: quant("cuda:0"), 0),
             ("quant_peer", lambda: quant("cuda:1"), n + S * 1024),
             ("dequant_local", lambda: dequant("cuda:0"), 0),
             ("dequant_peer", lambda: dequant("cuda:1"), n + S * 1024)]
    for name, fn, link_bytes in cases:
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(0)
        ms = e0.elapsed_time(e1) / args.iters
        line = f"{name}: {ms:.4f} ms per launch ({n} elements, {S} segments)"
        if link_bytes:
            line += f"; NVLink payload {link_bytes} B -> {link_bytes / ms / 1e6:.1f} GB/s averaged over the launch"
        print(line, flush=True)
    _check(L.emesh_codec_check(C.c_void_p(stream.cuda_stream)))
    # the peer payload is the same bytes as the local one (same kernel, same input)
    same = torch.equal(arenas["cuda:0"][0][:n].cpu(), arenas["cuda:1"][0][:n].cpu()) and \
        torch.equal(arenas["cuda:0"][1].cpu(), arenas["cuda:1"][1].cpu())
    print(f"peer payload identical to local: {same}")
    return 0 if same else 1


if __name__ == "__main__":
    sys.exit(main())
