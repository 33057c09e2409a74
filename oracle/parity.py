"""TEST INFRASTRUCTURE ONLY — segment-level parity of a GPU outer-sync round
against the oracle (oracle/emesh_oracle.c:orc_segment_chain).

A segment's final payload depends only on that segment's elements of every
worker (quantization is per segment, allreduce.hpp:326-336; the chunk's
reduce-scatter chain visits ranks c, c+1, ..., c+k-1 = its owner,
allreduce.hpp:411-446), so any subset of segments of a round can be
re-derived on the host at any model size. Used by tests/ and by bench.py's
post-timing parity leg (after the timed region, as the checker only).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Callable, List, Sequence, Tuple

import numpy as np


@dataclass
class SegmentJob:
    slot: int        # global segment index (codebook row)
    chunk: int       # ring chunk the segment belongs to
    lo: int
    length: int


@dataclass
class ParityReport:
    checked_segments: int = 0
    elements: int = 0
    code_mismatches: int = 0
    cb_mismatches: int = 0
    theta_mismatches: int = 0
    momentum_mismatches: int = 0
    min_margin: float = 1.0          # oracle's boundary margin (buckets) over the checked segments
    flips_margin: List[float] = field(default_factory=list)  # margin of each segment that had a code flip

    def ok(self) -> bool:
        return (self.code_mismatches == 0 and self.cb_mismatches == 0 and self.theta_mismatches == 0 and
                self.momentum_mismatches == 0)

    def as_dict(self):
        return {"checked_segments": self.checked_segments, "elements": self.elements,
                "code_mismatches": self.code_mismatches, "cb_mismatches": self.cb_mismatches,
                "theta_mismatches": self.theta_mismatches, "momentum_mismatches": self.momentum_mismatches,
                "min_boundary_margin_buckets": self.min_margin, "flip_segment_margins": self.flips_margin}


def segment_jobs(seg_lo: Sequence[int], seg_len: Sequence[int], k: int, S: int, picks=None) -> List[SegmentJob]:
    """Flat-arena segment table (chunk-major, min(S, len) subs per chunk) -> jobs; picks = slot indices
    to keep (None: all)."""
    n = int(sum(int(x) for x in seg_len))
    base, rem = divmod(n, k)
    bounds = []
    off = 0
    for c in range(k):
        ln = base + (1 if c < rem else 0)
        bounds.append((off, off + ln))
        off += ln
    jobs = []
    for s, (a, b) in enumerate(zip(seg_lo, seg_len)):
        a, b = int(a), int(b)
        if b == 0 or (picks is not None and s not in picks):
            continue
        c = next(i for i, (x, y) in enumerate(bounds) if x <= a < y)
        jobs.append(SegmentJob(s, c, a, b))
    return jobs


def check(O, jobs: Sequence[SegmentJob], k: int,
          inputs: Callable[[SegmentJob], Tuple[np.ndarray, List[np.ndarray], np.ndarray]],
          gpu: Callable[[SegmentJob], Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]],
          lr: float = 0.7, momentum: float = 0.9, threads: int = 0) -> ParityReport:
    """inputs(job) -> (theta_g before the round, [theta_l of every worker], momentum before);
    gpu(job) -> (final codes, codebook row, theta_g after, momentum after) of the GPU round.
    Compares bit for bit: codes, codebook, updated theta_g and momentum (optim.hpp:127-130
    applied to the decoded mean)."""
    rep = ParityReport()

    def one(job: SegmentJob):
        g, ls, b = inputs(job)
        codes, cb, st, mean = O.segment_chain(g, ls, job.chunk, want_mean=True)
        gc, gcb, gth, gb = gpu(job)
        avg = O.dequantize(codes, cb)
        th_o, b_o = O.nesterov(g, avg, b, lr, momentum)
        cm = int(np.count_nonzero(gc != codes))
        cbm = int(np.count_nonzero(np.ascontiguousarray(gcb, np.float32).view(np.uint32) != cb.view(np.uint32)))
        thm = int(np.count_nonzero(np.ascontiguousarray(gth, np.float32).view(np.uint32) != th_o.view(np.uint32)))
        bm = int(np.count_nonzero(np.ascontiguousarray(gb, np.float32).view(np.uint32) != b_o.view(np.uint32)))
        # distance of the owner's mean to the nearest bucket edge (buckets): how far a last-bit
        # difference in mu / sigma would have to move an edge to flip a code
        margin = O.boundary_margin(mean, st) if st[3] > 0 else 1.0
        return len(gc), cm, cbm, thm, bm, margin

    threads = threads or max(1, min(32, os.cpu_count() or 1))
    with ThreadPoolExecutor(threads) as ex:
        for n, cm, cbm, thm, bm, margin in ex.map(one, jobs):
            rep.checked_segments += 1
            rep.elements += n
            rep.code_mismatches += cm
            rep.cb_mismatches += cbm
            rep.theta_mismatches += thm
            rep.momentum_mismatches += bm
            rep.min_margin = min(rep.min_margin, margin)
            if cm:
                rep.flips_margin.append(margin)
    return rep
