"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference by oracle/Makefile). Run in the build
container (the GPU box has no /root/reference):

    make -C oracle && python tests/golden/make_golden.py

Inputs are stored next to the reference's outputs, so the fixtures pin both
the oracle restatement (CPU tests) and the CUDA path (GPU tests) without the
reference being present.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def normal_samples(O, n, seed, stream=0, counter=0):
    # Box-Muller over the counter rng, the shape of test_quant.cpp:47-58
    u1 = (O.uniform(2 * n, seed, stream, counter)[0::2].astype(np.float64) + 1.0) * 0.5
    u2 = (O.uniform(2 * n, seed, stream, counter)[1::2].astype(np.float64) + 1.0) * 0.5
    u1 = np.maximum(u1, 1e-12)
    return (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).astype(np.float32)


def quant_inputs(O):
    cases = {
        "two_point": np.array([-1.0, 1.0], np.float32),          # test_quant.cpp:69-79
        "constant": np.full(4, 5.0, np.float32),                 # test_quant.cpp:62-67
        "single": np.array([0.25], np.float32),
        "normal_10k": normal_samples(O, 10000, 2024),           # test_quant.cpp:81-95
        "normal_4096": normal_samples(O, 4096, 7),               # :116-126
        "normal_2000": normal_samples(O, 2000, 31),              # :128-141
        "normal_300": normal_samples(O, 300, 5),                 # :152-169
        "uniform_1e-3": O.uniform(65537, 3, 1, 0, 0, 1e-3),
        "offset_0.5": (O.uniform(40000, 4, 1, 0, 0, 1e-3) + np.float32(0.5)).astype(np.float32),
        "tiny_sigma_big_mu": (np.float32(1000.0) + O.uniform(5000, 5, 2, 0, 0, 1e-4)).astype(np.float32),
    }
    for seed in (1, 2, 3):  # test_quant.cpp:97-114: outliers every 13th element
        x = 3.0 * O.uniform(777, seed, 4, 0)
        x[::13] += 20.0
        cases[f"outlier_s{seed}"] = x.astype(np.float32)
    return cases


def main():
    O, R = Oracle(), Reference()
    qi = quant_inputs(O)
    arrays = {}
    for name, x in qi.items():
        codes, cb = R.quantize(x)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/codes"] = codes
        arrays[f"{name}/cb"] = cb
        arrays[f"{name}/wire"] = R.encode_quant_chunk(codes, cb)
    np.savez_compressed(os.path.join(OUT, "quant_cases.npz"), **arrays)

    ring = {}
    for k, n, S in [(2, 4096, 4), (3, 17, 4), (4, 4096, 4), (8, 1000, 2), (4, 3, 4)]:
        ins = [normal_samples(O, n, 777 + k, i, 1) for i in range(k)]  # test_allreduce.cpp:137-150
        for mode in ("int8", "fp32"):
            outs, sent = R.ring_allreduce_sim(ins, S, mode)
            key = f"k{k}_n{n}_S{S}_{mode}"
            ring[f"{key}/inputs"] = np.stack(ins)
            ring[f"{key}/out"] = outs[0]
            assert all(np.array_equal(outs[0].view(np.uint32), o.view(np.uint32)) for o in outs)
            ring[f"{key}/bytes_sent"] = sent
    np.savez_compressed(os.path.join(OUT, "ring_cases.npz"), **ring)

    # one full outer-sync round of the reference (TCP, k node threads)
    n, k, S = 20_000, 4, 4
    g = O.uniform(n, 1, 0)
    ls = [(g - O.uniform(n, 1, 1 + w, 0, 0, 2.0 ** -10)).astype(np.float32) for w in range(k)]
    b = O.uniform(n, 1, 9, 0, 0, 1e-3)
    tg, tb, _ = R.outer_sync_tcp(g, ls, b, S, "int8", 0.7, 0.9)
    np.savez_compressed(os.path.join(OUT, "outer_sync_case.npz"), theta_g=g, theta_l=np.stack(ls), buf=b,
                        theta_g_out=tg, buf_out=tb, k=k, S=S)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
