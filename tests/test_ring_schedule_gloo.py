"""CPU, world_size 2 and 3 over gloo: execute the NCCL engine's OWN ring
program (emesh_ring_schedule, the same C++ plan run_nccl walks) with gloo
send/recv as the transport and the oracle codec as the compute, and check
every rank ends bit-identical to the oracle's transport-free ring
(allreduce.hpp:314-473). This pins the multi-GPU host logic — who sends
which window of which chunk at which hop, owner finalize, all-gather
forwarding — without a GPU. ag="bcast" executes the all-gather the way
run_nccl does (emesh_b200.cu bcast_window): at hop 0 of each window, one
broadcast per chunk from its owner; the later forwarding hops are skipped."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, S, window, q, ag="hops"):
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, ROOT)
    from oracle.pyoracle import Oracle
    from paper_2412_01152_b200 import _capi
    from paper_2412_01152_b200 import emesh as E

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()
    k = world
    inputs = [O.uniform(n, 1234 + n, w, 0, 0, 2.0 ** -6) for w in range(k)]
    delta = inputs[rank]
    lo, ln = E.plan_segments(n, k, S)
    codes = np.zeros(max(n, 1), np.uint8)
    cbs = np.zeros((len(lo), 256), np.float32)
    result = np.zeros(max(n, 1), np.float32)
    succ, pred = (rank + 1) % k, (rank + k - 1) % k

    def segs(s0, ns):
        return [(i, int(lo[i]), int(ln[i])) for i in range(s0, s0 + ns)]

    def quant_into(i, a, b, x):
        if b == 0:
            return
        c, cb, _ = O.quantize(x)
        codes[a:a + b] = c
        cbs[i] = cb

    ops = E.ring_schedule(n, k, S, rank, window)
    wins = {}  # (chunk, window) -> (first segment, segments): the batch table run_nccl broadcasts from
    for op in ops:
        if op.send_chunk >= 0:
            wins[(op.send_chunk, op.window)] = (op.send_seg0, op.send_nseg)
        if op.recv_chunk >= 0:
            wins[(op.recv_chunk, op.window)] = (op.recv_seg0, op.recv_nseg)
    for op in ops:
        if op.kind == _capi.OP_XFER and op.phase == 1 and ag == "bcast":
            if op.hop == 0:
                for c in range(k):  # k broadcasts, root = the chunk's owner (allreduce.hpp:428-445)
                    s0, ns = wins[(c, op.window)]
                    ss = segs(s0, ns)
                    buf = torch.from_numpy(np.concatenate([codes[a:a + b] for _, a, b in ss] + [np.zeros(0, np.uint8)]))
                    bcb = torch.from_numpy(cbs[s0:s0 + ns].copy())
                    root = (c + k - 1) % k
                    dist.broadcast(buf, src=root)
                    dist.broadcast(bcb, src=root)
                    off = 0
                    bn = buf.numpy()
                    for _, a, b in ss:
                        codes[a:a + b] = bn[off:off + b]
                        off += b
                    cbs[s0:s0 + ns] = bcb.numpy()
            continue
        if op.kind == _capi.OP_OWN:
            for i, a, b in segs(op.recv_seg0, op.recv_nseg):
                quant_into(i, a, b, delta[a:a + b])
        elif op.kind == _capi.OP_XFER:
            ss = segs(op.send_seg0, op.send_nseg)
            rs = segs(op.recv_seg0, op.recv_nseg)
            sc = torch.from_numpy(np.concatenate([codes[a:a + b] for _, a, b in ss] + [np.zeros(0, np.uint8)]))
            scb = torch.from_numpy(cbs[op.send_seg0:op.send_seg0 + op.send_nseg].copy())
            rc = torch.empty(sum(b for _, _, b in rs), dtype=torch.uint8)
            rcb = torch.empty((op.recv_nseg, 256), dtype=torch.float32)
            reqs = [dist.isend(sc, succ), dist.isend(scb, succ)]
            dist.recv(rc, pred)
            dist.recv(rcb, pred)
            for r_ in reqs:
                r_.wait()
            off = 0
            rcn = rc.numpy()
            for _, a, b in rs:
                codes[a:a + b] = rcn[off:off + b]
                off += b
            cbs[op.recv_seg0:op.recv_seg0 + op.recv_nseg] = rcb.numpy()
        elif op.kind == _capi.OP_QUANT:
            for i, a, b in segs(op.recv_seg0, op.recv_nseg):
                if b == 0:
                    continue
                x = (delta[a:a + b] + cbs[i][codes[a:a + b]]).astype(np.float32)  # allreduce.hpp:422
                if op.final_hop:
                    x = (x / np.float32(k)).astype(np.float32)  # :439
                quant_into(i, a, b, x)
        elif op.kind == _capi.OP_APPLY:
            for i, a, b in segs(op.recv_seg0, op.recv_nseg):
                result[a:a + b] = cbs[i][codes[a:a + b]]
    want = O.ring_allreduce(inputs, S, "int8")
    q.put((rank, bool(np.array_equal(result[:n].view(np.uint32), want.view(np.uint32)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,S,window,ag", [(2, 4099, 4, 0, "hops"), (2, 50_000, 4, 6000, "hops"),
                                                (3, 3001, 3, 1, "hops"), (3, 10, 4, 0, "hops"), (2, 1, 4, 0, "hops"),
                                                (3, 3001, 3, 1, "bcast"), (3, 50_000, 4, 6000, "bcast"),
                                                (2, 4099, 4, 0, "bcast")])
def test_schedule_over_gloo_matches_oracle(world, n, S, window, ag):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, S, window, q, ag)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)], res


def test_nccl_id_broadcast_over_gloo():
    """The bench's rank-0 ncclUniqueId creation + broadcast (host side only)."""
    from paper_2412_01152_b200 import _capi
    import ctypes as C
    buf = C.create_string_buffer(128)
    rc = _capi.lib().emesh_nccl_unique_id(buf)
    # creating an id needs no GPU; it may fail only without any network interface
    assert rc in (0, _capi.ENCCL)
