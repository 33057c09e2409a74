// Segment-resident persistent quantizer (k_quant): the reference's
// quantize (proj/include/emesh/quant.hpp:28-87) over every segment of one
// ring batch, with its producer fused in (pseudo-gradient optim.hpp:108, ring
// hop add allreduce.hpp:422, owner mean :435-439).
//
// quantize is two passes over a segment: statistics (mu, sigma over ALL of
// the segment, quant.hpp:33-43) before any bucket can be assigned
// (:57-76). The value being quantized, x, is produced by the first pass and
// consumed by the second. At the benchmarked shapes a segment is 15.6M-16M
// elements (62.5 MB of x) — twice the GPU's shared memory — so round 1 kept
// x in an L2/HBM scratch and paid 8 B/element of DRAM for it (4.46 GB per
// 2.50 GB algorithmic). Here x stays ON CHIP: every SM holds the x of the
// tiles it produced in its tensor memory (256 KB/SM: 4 tiles) and shared
// memory (2 tiles) until the segment's statistics are final, then bins its
// own tiles. Only tiles beyond an SM's on-chip capacity go to a global
// scratch (an L2-sized overflow, binned by any CTA).
//
// Grid: one 512-thread CTA per SM (persistent). A STATS tile is 16 warp
// units (one per warp) of 1024 elements = 16K elements of one segment; tiles
// are claimed in segment order with one atomicAdd. A CTA alternates one
// STATS tile with one BIN tile of a segment whose statistics are published,
// so every SM mixes HBM-bound and issue-bound work. A CTA only ever waits
// (for a segment's statistics) when no STATS tile is left to claim, so
// progress never depends on co-residency (a plain launch suffices).
//
// Element layout of a warp unit: 128 octets (8 floats = 32 B) of the arena's
// octet grid; lane l at step j (0..3) owns octet o0 + 128 u + 32 j + l, so one
// warp instruction moves 1 KB contiguous (256-bit LDG/STG, sm_100). The
// lane's 32 values x[8 j + e] are exactly one tcgen05 32x32b.x32 row of its
// TMEM lane: the warp that produced a unit bins it from the same registers
// layout (TMEM lane quadrant = warp % 4).
#pragma once

#include "kernels.cuh"

namespace emesh_b200 {

#ifndef EMESH_QWARPS
#define EMESH_QWARPS 16
#endif
constexpr int kQWarps = EMESH_QWARPS;       // warps per CTA (CTAs per SM: 16 / kQWarps)
constexpr int kQCtasPerSm = 16 / kQWarps;
constexpr int kQTmemCols = 128 * kQWarps / 4;  // this CTA's share of the SM's 512 TMEM columns
constexpr int kQThreads = kQWarps * 32;  // 512
constexpr int kQTmemSlots = 4;           // 4 x 32 TMEM columns per warp (its quadrant's 128-column share)
#ifndef EMESH_QSMEM_SLOTS
#define EMESH_QSMEM_SLOTS 2
#endif
constexpr int kQSmemSlots = EMESH_QSMEM_SLOTS;  // 4 KB of shared memory per warp each
constexpr int kQSlots = kQTmemSlots + kQSmemSlots;
constexpr uint32_t kSlotGlobal = 0xffu;
constexpr int kUnitOct = 128;                // octets per warp unit (1024 elements)
constexpr int kTileUnits = kQWarps;          // warp units per tile (one per warp)
constexpr int kTileElems = kTileUnits * kUnitOct * 8;  // 16384

// Bin-pass limbs, per warp PAIR over one BIN tile (<= 2048 members each):
// A = r[0:9) | 1 << 20 (count), B = r[9:29), C = r[29:42) (rare).
// 2048 * 511 < 2^20; 2048 < 2^12; 2048 * (2^20 - 1) < 2^31; 2048 * (2^13 - 1) < 2^32.
constexpr int kQLoBits = 9, kQCntShift = 20, kQMidEnd = 29;
constexpr int kQHists = kQWarps / 2;

// Per-segment sync words of one launch (zeroed per launch): base kSyncReady + 5 s.
enum : uint32_t { kSyReady = 0, kSyStats = 1, kSyBins = 2, kSyOvfCount = 3, kSyOvfClaim = 4, kSyPerSeg = 5 };

struct Q2Args {
    const SegInfo* segs;
    const uint4* tile_seg;     // STATS tile (batch order) -> {batch-local segment, tile within it, first octet, octets}
    uint32_t ntiles;           // STATS tiles of the batch
    uint32_t nseg;
    const float* a;
    const float* b;
    const uint8_t* in_codes;
    const float* in_cb;
    float divisor;
    float inv_divisor;  // 1/k when k is a power of two (exact), else 0
    float* scratch;     // overflow x, octet-addressed: segment s at octets [so0, so0 + units * 128)
    uint8_t* dcodes[kMaxDest];
    float* dcb[kMaxDest];
    uint32_t ndest;
    uint32_t* sflag[kMaxDest];
    uint32_t nflag;
    const uint32_t* in_flag;
    uint32_t epoch;
    unsigned long long timeout_ns;
    SegStat* stats;     // by slot
    StatP* leaf_stat;   // by batch tile
    SegAcc* acc;        // by batch-local segment (self-cleaning)
    uint32_t* seg_flags;
    uint32_t* err;
    uint32_t* sync;     // [0] STATS claim counter; per segment kSyPerSeg words from kSyncReady
    uint32_t* ovf;      // overflow tile lists: segment s's at [t0, t0 + ntile)
    // peer transport: ChunkMsg headers written next to every payload / checked on receipt
    ChunkHdr* dhdr[kMaxDest];
    const ChunkHdr* in_hdr;
    HdrRef hdr;
    uint32_t phase_out;  // kPhaseRS, or kPhaseAG for the owner's final payload
    uint32_t culprit_in; // rank that owes the incoming payloads (the predecessor)
};

struct QHeld {
    uint32_t seg, tile, slot;
};

// One step of a CTA (thread 0's decision, broadcast through shared memory).
struct QStep {
    uint32_t kind;                     // kQTaskStep / kQTaskFinStats / kQTaskFinCb / kQTaskExit
    uint32_t s_seg, s_tile, s_slot;    // STATS tile (s_seg == kNone: none)
    uint32_t b_seg, b_tile, b_slot;    // BIN tile (b_seg == kNone: none)
};
constexpr uint32_t kNone = 0xffffffffu;

struct Q2Smem {
    uint32_t hist[kQHists][kBuckets + 1][3];  // per warp pair; row 256: sink
    double2 bsk[kBuckets];                    // per bucket {s, K}: fixed point m = x * s + K (kInfoWide)
    float thr[kBuckets + 2];                  // exact thresholds; [256] = +inf, [257] = lo_up
    float lut[kBuckets];                      // incoming codebook (hop add)
    StatP wp[kQWarps];
    double red[2];
    float bp[6];                              // BIN params: c, inv_w, lo_up, hi_dn, margin, 1 - margin
    uint32_t clip[2];
    uint32_t degenerate;
    uint32_t flag;
    uint32_t tbase;                           // TMEM base address
    uint32_t ovf_seg;                         // lowest segment that may still hold unclaimed overflow tiles
    uint32_t freemask;                        // free on-chip slots
    uint32_t qh, qn;                          // held on-chip tiles (FIFO)
    QHeld q[kQSlots];
    int32_t lut_seg, bin_seg;
    uint32_t pf_o, pf_no;                     // next STATS tile's octets (L2 prefetch)
    QStep step;
};
constexpr size_t kQ2SmemX = (size_t)kQSmemSlots * kQWarps * 4096;
constexpr size_t kQ2SmemBytes = sizeof(Q2Smem) + 16 + kQ2SmemX;

enum : uint32_t { kQTaskStep = 1, kQTaskExit = 2, kQTaskFinStats = 3, kQTaskFinCb = 4 };

// ---------------------------------------------------------------------------
// tensor memory (tcgen05) as the on-chip x store

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&x)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]), "f"(x[7]), "f"(x[8]), "f"(x[9]),
        "f"(x[10]), "f"(x[11]), "f"(x[12]), "f"(x[13]), "f"(x[14]), "f"(x[15]), "f"(x[16]), "f"(x[17]), "f"(x[18]),
        "f"(x[19]), "f"(x[20]), "f"(x[21]), "f"(x[22]), "f"(x[23]), "f"(x[24]), "f"(x[25]), "f"(x[26]), "f"(x[27]),
        "f"(x[28]), "f"(x[29]), "f"(x[30]), "f"(x[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&x)[32]) {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7]), "=f"(x[8]),
          "=f"(x[9]), "=f"(x[10]), "=f"(x[11]), "=f"(x[12]), "=f"(x[13]), "=f"(x[14]), "=f"(x[15]), "=f"(x[16]),
          "=f"(x[17]), "=f"(x[18]), "=f"(x[19]), "=f"(x[20]), "=f"(x[21]), "=f"(x[22]), "=f"(x[23]), "=f"(x[24]),
          "=f"(x[25]), "=f"(x[26]), "=f"(x[27]), "=f"(x[28]), "=f"(x[29]), "=f"(x[30]), "=f"(x[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 256-bit streaming loads (read once: L1 no-allocate, L2 evict-first)
__device__ __forceinline__ void ld8_stream(const float* p, float* v) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}
// incoming codes of one octet (the predecessor may have written them during this launch's
// lifetime only under the peer transport, and then before its flag: not .nc)
__device__ __forceinline__ uint2 ld8_codes(const uint8_t* p) {
    uint2 v;
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st8_f32(float* p, const float* v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}
__device__ __forceinline__ void ld8_f32(const float* p, float* v) {
    asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p)
                 : "memory");
}

// smem histogram add with no compiler memory barrier: ordered against other
// shared-memory traffic by the block barriers around the tile only
__device__ __forceinline__ void red_shared_add_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v));
}
__device__ __forceinline__ void red_shared_add_nz_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q red.shared.add.u32 [%0], %1;\n\t}" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(p)),
                 "r"(v));
}

// ---------------------------------------------------------------------------
// tensor-memory halves (16 columns = octets j = 2h, 2h + 1 of a warp unit)

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* x) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]), "f"(x[7]), "f"(x[8]), "f"(x[9]),
        "f"(x[10]), "f"(x[11]), "f"(x[12]), "f"(x[13]), "f"(x[14]), "f"(x[15])
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* x) {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
        "[%16];"
        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7]), "=f"(x[8]),
          "=f"(x[9]), "=f"(x[10]), "=f"(x[11]), "=f"(x[12]), "=f"(x[13]), "=f"(x[14]), "=f"(x[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Where a warp unit's x lives between its STATS and BIN passes.
struct QSlotRef {
    uint32_t slot;    // < kQTmemSlots: TMEM; < kQSlots: smem; kSlotGlobal: overflow scratch
    uint32_t taddr;   // TMEM address of the unit's 32 columns
    float4* sp;       // smem unit (256 float4: [j][lane] low half, [j][32 + lane] high half)
    float* gp;        // overflow scratch of the segment, arena-indexed by element
};

__device__ __forceinline__ QSlotRef q2_slot(const Q2Args& a, const Q2Smem& sm, float4* xsm, const SegInfo& si,
                                            uint32_t slot) {
    const int warp = threadIdx.x >> 5;
    QSlotRef r;
    r.slot = slot;
    r.taddr = sm.tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 128u * (uint32_t)(warp >> 2) + 32u * (slot & 3u);
    r.sp = xsm + ((size_t)(((slot < kQSlots ? slot : kQTmemSlots) - kQTmemSlots) * kQWarps + warp) * 4) * 64;
    r.gp = a.scratch + ((int64_t)si.so0 - (int64_t)si.o0) * 8;
    return r;
}

// x of octets j = 2h, 2h + 1 (16 values per lane) into / out of the slot
__device__ __forceinline__ void q2_put_half(const QSlotRef& r, uint64_t obase, int h, const float* x) {
    const int lane = threadIdx.x & 31;
    if (r.slot < kQTmemSlots) {
        tmem_st16(r.taddr + 16u * (uint32_t)h, x);
    } else if (r.slot < kQSlots) {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = 2 * h + jj;
            r.sp[j * 64 + lane] = make_float4(x[8 * jj], x[8 * jj + 1], x[8 * jj + 2], x[8 * jj + 3]);
            r.sp[j * 64 + 32 + lane] = make_float4(x[8 * jj + 4], x[8 * jj + 5], x[8 * jj + 6], x[8 * jj + 7]);
        }
    } else {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) st8_f32(r.gp + (obase + (uint64_t)(2 * h + jj) * 32 + lane) * 8, &x[8 * jj]);
    }
}
__device__ __forceinline__ void q2_get_half(const QSlotRef& r, uint64_t obase, int h, float* x) {
    const int lane = threadIdx.x & 31;
    if (r.slot < kQTmemSlots) {
        tmem_ld16(r.taddr + 16u * (uint32_t)h, x);
    } else if (r.slot < kQSlots) {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = 2 * h + jj;
            const float4 v0 = r.sp[j * 64 + lane], v1 = r.sp[j * 64 + 32 + lane];
            x[8 * jj] = v0.x; x[8 * jj + 1] = v0.y; x[8 * jj + 2] = v0.z; x[8 * jj + 3] = v0.w;
            x[8 * jj + 4] = v1.x; x[8 * jj + 5] = v1.y; x[8 * jj + 6] = v1.z; x[8 * jj + 7] = v1.w;
        }
    } else {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) ld8_f32(r.gp + (obase + (uint64_t)(2 * h + jj) * 32 + lane) * 8, &x[8 * jj]);
    }
}

// ---------------------------------------------------------------------------
// STATS: the fused producer (PG / hop add / owner mean) + moments, per half unit

// Per-lane moments around a pivot (its first in-segment value), fp64.
struct QMoments {
    double s0, s1, d0, d1, q0, q1, piv;
    uint32_t cnt;
    bool have;
};

template <int SRC>
struct QLoads {
    float a[16];
    float b[(SRC & kSrcAminusB) ? 16 : 1];
    uint2 c[2];
};

template <int SRC>
__device__ __forceinline__ void q2_stats_load(const Q2Args& a, uint64_t obase, uint64_t hiel, bool interior, int h,
                                              QLoads<SRC>& L) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
        const uint64_t o = obase + (uint64_t)(2 * h + jj) * 32 + lane;
        if (interior || o * 8 < hiel) {  // octets past the segment end are not loaded
            ld8_stream(a.a + o * 8, &L.a[8 * jj]);
            if (SRC & kSrcAminusB) ld8_stream(a.b + o * 8, &L.b[8 * jj]);
            if (SRC & kHasIn) L.c[jj] = ld8_codes(a.in_codes + o * 8);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                L.a[8 * jj + e] = 0.f;
                if (SRC & kSrcAminusB) L.b[8 * jj + e] = 0.f;
            }
            L.c[jj] = make_uint2(0u, 0u);
        }
    }
}

// x = producer(loads) in place (L.a), accumulated into the lane's moments.
template <int SRC>
__device__ __forceinline__ void q2_stats_finish(const Q2Args& a, const Q2Smem& sm, const SegInfo& si, uint64_t obase,
                                                bool interior, int h, QLoads<SRC>& L, QMoments& m) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float v = L.a[i];
        if (SRC & kSrcAminusB) v = __fsub_rn(v, L.b[i]);  // optim.hpp:108
        if (SRC & kHasIn) {                                // allreduce.hpp:422
            const uint32_t w = (i & 7) < 4 ? L.c[i >> 3].x : L.c[i >> 3].y;
            v = __fadd_rn(v, sm.lut[(w >> (8 * (i & 3))) & 0xffu]);
        }
        if (SRC & kDivK) v = a.inv_divisor != 0.f ? __fmul_rn(v, a.inv_divisor) : __fdiv_rn(v, a.divisor);  // :439
        L.a[i] = v;
    }
#ifdef EMESH_Q_ABL_NOMOM  // ablation (timing only): no fp64 moments
    if (true) {
        m.s0 = __dadd_rn(m.s0, (double)(L.a[0] + L.a[15]));
        m.cnt += 16;
        return;
    }
#endif
    if (interior) {
        if (!m.have) {
            m.piv = (double)L.a[0];
            m.have = true;
        }
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            const double x0 = (double)L.a[i], x1 = (double)L.a[i + 1];
            const double v0 = __dsub_rn(x0, m.piv), v1 = __dsub_rn(x1, m.piv);
            m.s0 = __dadd_rn(m.s0, x0);
            m.s1 = __dadd_rn(m.s1, x1);
            m.d0 = __dadd_rn(m.d0, v0);
            m.d1 = __dadd_rn(m.d1, v1);
            m.q0 = __fma_rn(v0, v0, m.q0);
            m.q1 = __fma_rn(v1, v1, m.q1);
        }
        m.cnt += 16;
    } else {
        const uint64_t hiel = si.lo + si.len;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const uint64_t e0 = (obase + (uint64_t)(2 * h + jj) * 32 + lane) * 8;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (e0 + e >= si.lo && e0 + e < hiel) {
                    const double xd = (double)L.a[8 * jj + e];
                    if (!m.have) {
                        m.piv = xd;
                        m.have = true;
                    }
                    const double dv = __dsub_rn(xd, m.piv);
                    m.s0 = __dadd_rn(m.s0, xd);
                    m.d0 = __dadd_rn(m.d0, dv);
                    m.q0 = __fma_rn(dv, dv, m.q0);
                    m.cnt += 1;
                }
            }
        }
    }
}

__device__ void q2_finalize_stats(const Q2Args& a, Q2Smem& sm, uint32_t s, const SegInfo& si);
__device__ void q2_finalize_codebook(const Q2Args& a, uint32_t s, const SegInfo& si);

// Deferred arrival of a tile on its segment's counter: the atomic's result is
// only looked at in thread 0's next decision, so no block waits on it.
struct QArrive {
    uint32_t kind;  // kQTaskFinStats / kQTaskFinCb when pending, else 0
    uint32_t seg, last, old;
};

// Run by the last STATS tile of s: merge the leaves in a fixed order, then
// mu / sigma / lo / hi / width (quant.hpp:33-59), the exact threshold table
// and bucket encodings; publish SegStat(s) and the segment's ready flag.
__device__ void q2_finalize_stats(const Q2Args& a, Q2Smem& sm, uint32_t s, const SegInfo& si) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    StatP p{0.0, 0.0, 0.0, 0.0, 0};
    for (uint32_t i = threadIdx.x; i < si.ntile; i += kQThreads) {
        const StatP* src = &a.leaf_stat[si.t0 + i];
        StatP ch;
        ch.s = __ldcg(&src->s); ch.m2 = __ldcg(&src->m2); ch.d = __ldcg(&src->d);
        ch.piv = __ldcg(&src->piv); ch.n = __ldcg(&src->n);
        p = statp_merge(p, ch);
    }
    p = warp_merge(p);
    __syncthreads();  // sm.wp reuse
    if (lane == 0) sm.wp[warp] = p;
    __syncthreads();
    if (threadIdx.x == 0) {
        StatP t = sm.wp[0];
        for (int w = 1; w < kQWarps; ++w) t = statp_merge(t, sm.wp[w]);
        const double mu = __ddiv_rn(t.s, (double)si.len);
        const double dm = __dsub_rn(t.piv, mu);
        // sum (x - mu)^2 = M2 + 2 (p - mu) D + n (p - mu)^2
        double ss = __dadd_rn(t.m2, __dmul_rn(__dmul_rn(2.0, dm), t.d));
        ss = __dadd_rn(ss, __dmul_rn((double)t.n, __dmul_rn(dm, dm)));
        const double var = __ddiv_rn(ss < 0.0 ? 0.0 : ss, (double)si.len);
        sm.red[0] = mu;
        sm.red[1] = __dsqrt_rn(var);
    }
    __syncthreads();
    const double mu = sm.red[0], sigma = sm.red[1];
    SegStat* st = &a.stats[si.slot];
    if (threadIdx.x == 0) {
        st->mu = mu;
        st->sigma = sigma;
        st->flags = __ldcg(&a.seg_flags[s]) | (sigma == 0.0 ? kFlagDegenerate : 0u);
        a.seg_flags[s] = 0;
        if (sigma == 0.0) {
            st->lo = mu; st->hi = mu; st->width = 0.0;
            st->c_f = 0.f; st->inv_w_f = 0.f;
        }
    }
    if (sigma != 0.0) {
        const double six = __dmul_rn(6.0, sigma);
        const double lo = __dsub_rn(mu, six);
        const double hi = __dadd_rn(mu, six);
        const double w = __ddiv_rn(__dsub_rn(hi, lo), 256.0);
        float lo_up = (float)lo;  // smallest fp32 >= lo, largest fp32 <= hi
        if ((double)lo_up < lo) lo_up = key2f(f2key(lo_up) + 1);
        float hi_dn = (float)hi;
        if ((double)hi_dn > hi) hi_dn = key2f(f2key(hi_dn) - 1);
        const int b = threadIdx.x;
        if (b < kBuckets) sm.thr[b] = b == 0 ? lo_up : threshold(b, lo, hi, w);
        if (b == 0) sm.thr[kBuckets] = key2f(f2key(hi_dn) + 1);
        __syncthreads();
        if (b < kBuckets) {
            st->thr[b] = b == 0 ? -INFINITY : sm.thr[b];
            st->binfo[b] = bucket_info(sm.thr[b], sm.thr[b + 1]);
        }
        if (b == 0) {
            st->lo = lo; st->hi = hi; st->width = w;
            st->c_f = (float)__ddiv_rn(lo, w);
            st->inv_w_f = (float)__ddiv_rn(1.0, w);
            st->lo_up = lo_up;
            st->hi_dn = hi_dn;
            // error of g = fma(x, inv_w, -c) (fp32) vs (x - lo) / w in buckets, for lo <= x <= hi:
            // inv_w and c carry <= 2^-24 relative error each, the fma one rounding of |g| <= 256:
            // err <= ((max(|lo|, |hi|) + |lo|) / w + 256) 2^-24; x2 for safety
            const double mag = __ddiv_rn(fmax(fabs(lo), fabs(hi)) + fabs(lo), w);
            const double err = __dmul_rn(__dadd_rn(mag, 256.0), 1.01 / 16777216.0);
            const double mg = __dmul_rn(2.0, err) + 1e-6;
            st->margin = mg < 0.25 ? (float)mg : 2.0f;  // 2.0: always walk the table
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        sm.bin_seg = -1;  // sm.thr now holds this segment's raw table: force a reload
        st_release(a.sync + kSyncReady + kSyPerSeg * s + kSyReady, 1u);
    }
}

// ---------------------------------------------------------------------------
// BIN

// Bins one octet group of 8 values (codes + exact bucket sums).
template <bool INTERIOR>
__device__ __forceinline__ void q2_bin_octet(const Q2Args& a, Q2Smem& sm, const float* xe, uint64_t o,
                                             const SegInfo& si, uint32_t* hw, uint32_t& nclip_lo,
                                             uint32_t& nclip_hi) {
    const float c_f = sm.bp[0], inv_w = sm.bp[1], lo_up = sm.bp[2], hi_dn = sm.bp[3], margin = sm.bp[4],
                one_m = sm.bp[5];
    uint32_t vmask = 0xffu;
    if (!INTERIOR) {
        vmask = 0u;
        const uint64_t hiel = si.lo + si.len;
#pragma unroll
        for (int i = 0; i < 8; ++i) vmask |= (o * 8 + i >= si.lo && o * 8 + i < hiel) ? (1u << i) : 0u;
    }
    int cc[8];
    bool okall = true;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        // in range and clear of every bucket edge by the proven margin: trunc(g)
        // is the exact bucket (clipped x fails this test; see SegStat::margin)
        const float g = __fmaf_rn(xe[i], inv_w, -c_f);
        const int c = __float2int_rz(g);
        const float fr = __fsub_rn(g, __int2float_rz(c));
        okall &= (fr > margin) & (fr < one_m) & ((uint32_t)c < 256u);
        cc[i] = c;
    }
    if (!INTERIOR) {
#pragma unroll
        for (int i = 0; i < 8; ++i) cc[i] |= ((vmask >> i) & 1u) ? 0 : 256;  // outside the segment: sink row
    }
    if (!okall) {  // rare: near an edge (exact table) or clipped (quant.hpp:66-67)
        uint32_t clo_m = 0, chi_m = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float x = xe[i];
            const float g = __fmaf_rn(x, inv_w, -c_f);
            const int c0 = __float2int_rz(g);
            const float fr = __fsub_rn(g, __int2float_rz(c0));
            const int sink = cc[i] & 256;
            if (x < lo_up) {
                cc[i] = 256; clo_m |= 1u << i;
            } else if (x > hi_dn) {
                cc[i] = 256 | 255; chi_m |= 1u << i;
            } else if (!(fr > margin && fr < one_m && (uint32_t)c0 < 256u)) {
                cc[i] = sink | bucket_walk(x, min(max(c0, 0), 255), sm.thr);
            }
        }
        nclip_lo += __popc(clo_m & vmask);
        nclip_hi += __popc(chi_m & vmask);
    }
    // fixed point r of every member (kInfoWide): all 8 table loads first, then the fmas, then the
    // limb atomics (no compiler memory barrier between them: they only touch the histogram)
    double2 sk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) sk[i] = sm.bsk[cc[i] & 255];
    uint32_t rlo[8], rhi[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        // m = x * s + K in [2^52, 2^53): its mantissa is the member's fixed point r
        const double m = __fma_rn((double)xe[i], sk[i].x, sk[i].y);
        rlo[i] = (uint32_t)__double2loint(m);
        rhi[i] = (uint32_t)__double2hiint(m);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t* hc = hw + 3 * min(cc[i], kBuckets);
        red_shared_add_relaxed(hc, (rlo[i] & ((1u << kQLoBits) - 1u)) | (1u << kQCntShift));
        red_shared_add_relaxed(hc + 1, (rlo[i] >> kQLoBits) & ((1u << (kQMidEnd - kQLoBits)) - 1u));
        const uint32_t rc = __funnelshift_r(rlo[i], rhi[i], kQMidEnd) & ((1u << (42 - kQMidEnd)) - 1u);
        red_shared_add_nz_relaxed(hc + 2, rc);  // predicated: the high limb is rarely nonzero
    }
    const uint32_t p0 = __byte_perm(__byte_perm(cc[0], cc[1], 0x0040), __byte_perm(cc[2], cc[3], 0x0040), 0x5410);
    const uint32_t p1 = __byte_perm(__byte_perm(cc[4], cc[5], 0x0040), __byte_perm(cc[6], cc[7], 0x0040), 0x5410);
    if (INTERIOR) {
        *reinterpret_cast<uint2*>(a.dcodes[0] + o * 8) = make_uint2(p0, p1);
        for (uint32_t d = 1; d < a.ndest; ++d) *reinterpret_cast<uint2*>(a.dcodes[d] + o * 8) = make_uint2(p0, p1);
    } else {
        for (uint32_t d = 0; d < a.ndest; ++d) {
            uint8_t* oc = a.dcodes[d] + o * 8;
            if (vmask == 0xffu) {
                *reinterpret_cast<uint2*>(oc) = make_uint2(p0, p1);
            } else if (vmask) {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (vmask & (1u << e)) oc[e] = (uint8_t)((e < 4 ? p0 : p1) >> (8 * (e & 3)));
            }
        }
    }
}

// Run by the last BIN tile of s: the codebook from the exact bucket sums
// (quant.hpp:78-85); re-zeroes the accumulator; raises the arrival flags.
__device__ void q2_finalize_codebook(const Q2Args& a, uint32_t s, const SegInfo& si) {
    const SegStat* st = &a.stats[si.slot];
    const int b = threadIdx.x;
    SegAcc* acc = &a.acc[s];
    unsigned long long rl = 0, rh = 0, clip = 0, total = 0;
    if (b < kBuckets) {
        rl = __ldcg(&acc->rlo[b]);
        rh = __ldcg(&acc->rhi[b]);
        clip = b == 0 ? __ldcg(&acc->clip[0]) : b == 255 ? __ldcg(&acc->clip[1]) : 0ull;
        total = __ldcg(&acc->cnt[b]) + clip;  // clipped members sit in the sink row
    }
    __syncthreads();  // every read done before the re-zeroing
    if (b < kBuckets) {
        acc->rlo[b] = 0ull;
        acc->rhi[b] = 0ull;
        acc->cnt[b] = 0ull;
        if (b < 2) acc->clip[b] = 0ull;
        float v;
        if ((__ldcg(&st->flags) & kFlagDegenerate) != 0) v = (float)__ldcg(&st->mu);
        else if (total == 0)
            v = (float)__dadd_rn(__ldcg(&st->lo), __dmul_rn(__dadd_rn((double)b, 0.5), __ldcg(&st->width)));
        else v = codebook_entry(st, b, rl, rh, total, clip);
        for (uint32_t d = 0; d < a.ndest; ++d) a.dcb[d][(uint64_t)si.slot * kBuckets + b] = v;
    }
    if (threadIdx.x == 0)  // the ChunkMsg header of this payload, before its flag
        for (uint32_t d = 0; d < a.ndest; ++d)
            if (a.dhdr[d]) write_hdr(a.dhdr[d] + si.slot, a.hdr, si.chunk, (uint32_t)si.len, (uint8_t)a.phase_out);
    if (a.nflag) {
        // every tile of s released its stores (gpu scope) to the arrival counter this CTA
        // acquired; the system-scope fence + release extends that chain to the peers
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            const uint32_t v = raise_value(a.err, a.epoch);  // poison when this rank's round failed
            for (uint32_t f = 0; f < a.nflag; ++f) st_release_sys(a.sflag[f] + si.slot, v);
        }
    }
}

// ---------------------------------------------------------------------------
// One fused step of a CTA: a STATS tile and a BIN tile side by side. Every
// warp, per half unit: issue the STATS loads, bin its BIN half unit (pure
// compute on on-chip x) while they fly, then finish the STATS half and park
// its x. The block synchronizes twice per step (tile leaf + histogram flush).


// BIN: the segment's tables into shared memory (CTA-wide; at segment changes only)
__device__ void q2_bin_tables(const Q2Args& a, Q2Smem& sm, uint32_t s, const SegInfo& si) {
    const SegStat* st = &a.stats[si.slot];
    __syncthreads();
    const int b = threadIdx.x;
    if (b < kBuckets) {
        sm.thr[b] = b == 0 ? -INFINITY : __ldcg(&st->thr[b]);
        const uint32_t info = __ldcg(&st->binfo[b]);
        // s = high word of info (low bits zero), K = 2^52 (+ 2^41 for a wide bucket)
        sm.bsk[b] = make_double2(__hiloint2double((int)(info & ~kInfoWide), 0),
                                 __hiloint2double((int)(0x43300000u | ((info & kInfoWide) << 9)), 0));
    }
    if (b == kQThreads - 1) {  // (the last thread: 256 of them may all be busy with buckets above)
        sm.thr[kBuckets] = INFINITY;
        sm.thr[kBuckets + 1] = __ldcg(&st->lo_up);
        const float margin = __ldcg(&st->margin);
        sm.bp[0] = __ldcg(&st->c_f);
        sm.bp[1] = __ldcg(&st->inv_w_f);
        sm.bp[2] = __ldcg(&st->lo_up);
        sm.bp[3] = __ldcg(&st->hi_dn);
        sm.bp[4] = margin;
        sm.bp[5] = 1.f - margin;
        sm.degenerate = (__ldcg(&st->flags) & kFlagDegenerate) != 0;
        sm.bin_seg = (int32_t)s;
    }
    __syncthreads();
}

// STATS: the incoming codebook of segment s (hop add), after the peer flag (CTA-wide)
__device__ void q2_stats_lut(const Q2Args& a, Q2Smem& sm, uint32_t s, const SegInfo& si) {
    __syncthreads();
    if (a.in_flag) {  // peer transport: the predecessor's payload of s must have landed intact
        if (threadIdx.x == 0 &&
            spin_until_ge_sys(a.in_flag + si.in_slot, a.epoch, a.err, a.timeout_ns, a.culprit_in) && a.in_hdr)
            check_hdr(a.in_hdr + si.in_slot, a.hdr, si.chunk, (uint32_t)si.len, kPhaseRS, a.err, a.culprit_in);
        __syncthreads();
    }
    if (threadIdx.x < kBuckets) sm.lut[threadIdx.x] = __ldcg(a.in_cb + (uint64_t)si.in_slot * kBuckets + threadIdx.x);
    if (threadIdx.x == 0) sm.lut_seg = (int32_t)s;
    __syncthreads();
}

template <int SRC>
__device__ void q2_step(const Q2Args& a, Q2Smem& sm, float4* xsm, const QStep& t, QArrive (&arr)[2]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool do_s = t.s_seg != kNone, do_b = t.b_seg != kNone;
    SegInfo ss{}, sb{};
    if (do_s) ss = a.segs[t.s_seg];
    if (do_b) sb = a.segs[t.b_seg];
    if (do_b && sm.bin_seg != (int32_t)t.b_seg) q2_bin_tables(a, sm, t.b_seg, sb);
    if ((SRC & kHasIn) && do_s && sm.lut_seg != (int32_t)t.s_seg) q2_stats_lut(a, sm, t.s_seg, ss);
    uint32_t ovf_i = 0;  // overflow slot of the STATS tile: claimed now, used at the end
    if (do_s && threadIdx.x == 0 && t.s_slot == kSlotGlobal)
        ovf_i = atomicAdd(a.sync + kSyncReady + kSyPerSeg * t.s_seg + kSyOvfCount, 1u);
#ifndef EMESH_Q_NOPF
    if (do_s) {  // the NEXT STATS tile's inputs into L2 (whole 128-B lines): its loads then hit L2
        const uint64_t o0 = sm.pf_o, o1 = (uint64_t)sm.pf_o + sm.pf_no;
        const uint64_t t0 = (o0 * 32) & ~127ull, t1 = (o1 * 32 + 127) & ~127ull;
        for (uint64_t l = t0 + 128ull * threadIdx.x; l < t1; l += 128ull * kQThreads) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.a) + l));
            if (SRC & kSrcAminusB) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.b) + l));
        }
        if (SRC & kHasIn) {
            const uint64_t c0 = (o0 * 8) & ~127ull, c1 = (o1 * 8 + 127) & ~127ull;
            for (uint64_t l = c0 + 128ull * threadIdx.x; l < c1; l += 128ull * kQThreads)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(a.in_codes + l));
        }
    }
#endif
    const uint32_t us = t.s_tile * kTileUnits + warp, ub = t.b_tile * kTileUnits + warp;
    const bool vs = do_s && us < ss.nu8, vb = do_b && ub < sb.nu8;
    const uint64_t hs = ss.lo + ss.len, hb = sb.lo + sb.len;
    const uint64_t os = ss.o0 + (uint64_t)us * kUnitOct, ob = sb.o0 + (uint64_t)ub * kUnitOct;
    const bool is = vs && os * 8 >= ss.lo && (os + kUnitOct) * 8 <= hs;
    const bool ib = vb && ob * 8 >= sb.lo && (ob + kUnitOct) * 8 <= hb;
    const QSlotRef rs = q2_slot(a, sm, xsm, ss, t.s_slot), rb = q2_slot(a, sm, xsm, sb, t.b_slot);
    QMoments m{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0u, false};
    uint32_t nclip_lo = 0, nclip_hi = 0;
    uint32_t* hw = &sm.hist[warp >> 1][0][0];
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        QLoads<SRC> L;
        if (vs) q2_stats_load<SRC>(a, os, hs, is, h, L);
        if (vb) {  // bin this half while the loads fly
            float y[16];
            q2_get_half(rb, ob, h, y);
            if (sm.degenerate) {  // sigma == 0: every code is 0 (quant.hpp:49-55)
                for (int jj = 0; jj < 2; ++jj) {
                    const uint64_t o = ob + (uint64_t)(2 * h + jj) * 32 + lane;
                    for (int e = 0; e < 8; ++e)
                        if (o * 8 + e >= sb.lo && o * 8 + e < hb)
                            for (uint32_t d = 0; d < a.ndest; ++d) a.dcodes[d][o * 8 + e] = 0;
                }
#ifdef EMESH_Q_ABL_NOBIN  // ablation (timing only): the BIN pass reads x and stores codes, nothing else
            } else if (true) {
                const uint32_t p0 = __float_as_uint(y[0]) ^ __float_as_uint(y[15]);
                *reinterpret_cast<uint2*>(a.dcodes[0] + (ob + (uint64_t)(2 * h) * 32 + lane) * 8) = make_uint2(p0, p0);
#endif
            } else if (ib) {
                q2_bin_octet<true>(a, sm, &y[0], ob + (uint64_t)(2 * h) * 32 + lane, sb, hw, nclip_lo, nclip_hi);
                q2_bin_octet<true>(a, sm, &y[8], ob + (uint64_t)(2 * h + 1) * 32 + lane, sb, hw, nclip_lo, nclip_hi);
            } else {
                q2_bin_octet<false>(a, sm, &y[0], ob + (uint64_t)(2 * h) * 32 + lane, sb, hw, nclip_lo, nclip_hi);
                q2_bin_octet<false>(a, sm, &y[8], ob + (uint64_t)(2 * h + 1) * 32 + lane, sb, hw, nclip_lo, nclip_hi);
            }
        }
        if (vs) {
            q2_stats_finish<SRC>(a, sm, ss, os, is, h, L, m);
            q2_put_half(rs, os, h, L.a);
        }
    }
    if (vb && t.b_slot == kSlotGlobal && ib) {
        // consumed (read exactly once): drop the unit's scratch lines from L2 without write-back
        const uintptr_t lo_b = reinterpret_cast<uintptr_t>(rb.gp + ob * 8);
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(lo_b + (uintptr_t)lane * 128) : "memory");
    }
    if (do_s) {
        StatP p{__dadd_rn(m.s0, m.s1), __dadd_rn(m.q0, m.q1), __dadd_rn(m.d0, m.d1), m.piv, (uint64_t)m.cnt};
        p = warp_merge(p);
        if (lane == 0) {
            sm.wp[warp] = p;
            if (!isfinite(p.s) || !isfinite(p.m2)) {  // finite fp32 inputs cannot overflow an fp64 sum
                atomicOr(&a.seg_flags[t.s_seg], kFlagNonFinite);
                atomicOr(a.err, kErrNonFinite);
            }
        }
    }
    if (do_b) {
        nclip_lo = warp_sum_u(nclip_lo);
        nclip_hi = warp_sum_u(nclip_hi);
        if (lane == 0 && (nclip_lo | nclip_hi)) {
            atomicAdd(&sm.clip[0], nclip_lo);
            atomicAdd(&sm.clip[1], nclip_hi);
        }
    }
    __syncthreads();
    if (do_s && threadIdx.x == 0) {
        StatP tl = sm.wp[0];
        for (int w = 1; w < kQWarps; ++w) tl = statp_merge(tl, sm.wp[w]);
        a.leaf_stat[ss.t0 + t.s_tile] = tl;
        if (t.s_slot == kSlotGlobal) a.ovf[ss.t0 + ovf_i] = t.s_tile;  // for BIN by any CTA (published below)
        // acq_rel: publishes the leaf, the overflow entry and (bar.sync + cumulativity) the block's
        // scratch stores; the last tile to arrive finalizes the segment (deferred: QArrive)
#ifdef EMESH_Q_ABL_RELAXED
        arr[0] = QArrive{kQTaskFinStats, t.s_seg, ss.ntile - 1, atomicAdd(a.sync + kSyncReady + kSyPerSeg * t.s_seg + kSyStats, 1u)};
#else
        arr[0] = QArrive{kQTaskFinStats, t.s_seg, ss.ntile - 1,
                         atom_add_acq_rel(a.sync + kSyncReady + kSyPerSeg * t.s_seg + kSyStats, 1u)};
#endif
    }
    if (do_b) {
        if (threadIdx.x < kBuckets) {  // tile histogram (exact integers, order-free) -> segment accumulator
            const int b = threadIdx.x;
            unsigned long long r = 0;
            uint32_t cn = 0;
#pragma unroll
            for (int hh = 0; hh < kQHists; ++hh) {
                const uint32_t A = sm.hist[hh][b][0], B = sm.hist[hh][b][1], Cc = sm.hist[hh][b][2];
                r += (unsigned long long)(A & ((1u << kQCntShift) - 1u)) + ((unsigned long long)B << kQLoBits) +
                     ((unsigned long long)Cc << kQMidEnd);
                cn += A >> kQCntShift;
                sm.hist[hh][b][0] = 0u;
                sm.hist[hh][b][1] = 0u;
                sm.hist[hh][b][2] = 0u;
            }
            SegAcc* acc = &a.acc[t.b_seg];
            if (cn) {
                atomicAdd(&acc->rlo[b], r & 0xffffffffull);
                if (r >> 32) atomicAdd(&acc->rhi[b], r >> 32);
                atomicAdd(&acc->cnt[b], (unsigned long long)cn);
            }
            if (b < 2) {
                if (sm.clip[b]) atomicAdd(&acc->clip[b], (unsigned long long)sm.clip[b]);
                sm.clip[b] = 0u;
            }
        }
        if (threadIdx.x >= kQThreads - kQHists) {  // the sink rows
            const int hh = threadIdx.x - (kQThreads - kQHists);
            sm.hist[hh][kBuckets][0] = 0u;
            sm.hist[hh][kBuckets][1] = 0u;
            sm.hist[hh][kBuckets][2] = 0u;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            // acq_rel: releases the block's accumulator atomics and code stores; the last tile
            // acquires all and writes the codebook (deferred: QArrive)
#ifdef EMESH_Q_ABL_RELAXED
            arr[1] = QArrive{kQTaskFinCb, t.b_seg, sb.ntile - 1, atomicAdd(a.sync + kSyncReady + kSyPerSeg * t.b_seg + kSyBins, 1u)};
#else
            arr[1] = QArrive{kQTaskFinCb, t.b_seg, sb.ntile - 1,
                             atom_add_acq_rel(a.sync + kSyncReady + kSyPerSeg * t.b_seg + kSyBins, 1u)};
#endif
            if (t.b_slot < kQSlots) sm.freemask |= 1u << t.b_slot;
        }
    }
}

// ---------------------------------------------------------------------------
// scheduler (thread 0): the next step of this CTA

__device__ __forceinline__ bool q2_ready(const Q2Args& a, uint32_t s) {
    return ld_acquire(a.sync + kSyncReady + kSyPerSeg * s + kSyReady) != 0u;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Thread 0's scheduler state, kept in registers across steps. Every global
// access a decision needs is issued one step ahead, so a decision never
// waits on a memory round trip in the common case: the STATS claims run
// three tiles ahead (c1: next to run, its table entry loaded; c2: the one
// after, its entry in flight; c3: its claim atomic in flight) and the ready
// flag of the oldest held tile's segment is polled (relaxed) during the step.
struct QSched {
    uint32_t c1;       // claimed STATS tile to run next (>= ntiles: none left)
    uint4 ts1;         // its {segment, tile, first octet, octets}
    uint32_t c2;       // the claim after c1
    uint4 ts2;         // its table entry
    uint32_t c3;       // the claim after c2
    uint32_t ready_upto;  // segments [0, ready_upto) are known ready (published in order, mostly)
    uint32_t poll;        // relaxed read of segment ready_upto's flag (1 for an empty segment)
    uint32_t ready_seg;   // a segment found ready out of order (blocking wait)
};

// Known ready without a memory round trip: the flag polled during the last step
// (one segment per decision; flags are monotone within a launch).
__device__ __forceinline__ bool q2_known_ready(QSched& q, uint32_t s) { return s < q.ready_upto || s == q.ready_seg; }
__device__ __forceinline__ void q2_advance_ready(const Q2Args& a, QSched& q) {
    if (q.ready_upto < a.nseg && q.poll) {
        __threadfence();  // acquire: the relaxed poll saw the release of SegStat(ready_upto)
        q.ready_upto += 1;
        q.poll = 0;
    }
}

__device__ void q2_decide(const Q2Args& a, Q2Smem& sm, QSched& q, QArrive (&arr)[2], QStep& t) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
        if (arr[i].kind) {  // a tile's deferred arrival: the last tile of a segment finalizes it
            const uint32_t k = arr[i].kind;
            arr[i].kind = 0;
            if (arr[i].old == arr[i].last) {
                t.kind = k;
                t.s_seg = arr[i].seg;
                return;
            }
        }
    q2_advance_ready(a, q);
    for (;;) {
        t.kind = kQTaskStep;
        t.s_seg = t.b_seg = kNone;
        t.s_slot = t.b_slot = kSlotGlobal;
        // BIN: the oldest tile held on chip when its segment is ready, else an overflow tile of a
        // ready segment (any CTA may bin those)
        if (sm.qn > 0 && q2_known_ready(q, sm.q[sm.qh].seg)) {
            const QHeld hd = sm.q[sm.qh];
            t.b_seg = hd.seg; t.b_tile = hd.tile; t.b_slot = hd.slot;
            sm.qh = (sm.qh + 1) % kQSlots;
            sm.qn -= 1;
        } else {
            while (sm.ovf_seg < a.nseg) {
                const uint32_t s = sm.ovf_seg;
                if (__ldg(&a.segs[s].ntile) == 0) {  // empty segment (a chunk shorter than S): no tiles
                    sm.ovf_seg = s + 1;
                    continue;
                }
                if (!q2_known_ready(q, s)) break;
                uint32_t* sy = a.sync + kSyncReady + kSyPerSeg * s;
                const uint32_t cnt = __ldcg(sy + kSyOvfCount);
                if (cnt && __ldcg(sy + kSyOvfClaim) < cnt) {
                    const uint32_t i = atomicAdd(sy + kSyOvfClaim, 1u);
                    if (i < cnt) {
                        t.b_seg = s; t.b_tile = __ldcg(a.ovf + a.segs[s].t0 + i);
                        t.b_slot = kSlotGlobal;
                        break;
                    }
                }
                sm.ovf_seg = s + 1;
            }
        }
        // STATS: the claimed tile, on chip when a slot is free (the BIN tile's slot frees at the
        // end of this step), else in the overflow scratch
        if (q.c1 < a.ntiles) {
            t.s_seg = q.ts1.x; t.s_tile = q.ts1.y;
            uint32_t slot = kSlotGlobal;
            if (sm.freemask) {
                slot = __ffs(sm.freemask) - 1;
                sm.freemask &= ~(1u << slot);
                sm.q[(sm.qh + sm.qn) % kQSlots] = QHeld{q.ts1.x, q.ts1.y, slot};
                sm.qn += 1;
            }
            t.s_slot = slot;
            // advance the claim pipeline (every value used here arrived during an earlier step)
            q.c1 = q.c2;
            q.ts1 = q.ts2;
            q.c2 = q.c3;
            q.ts2 = q.c2 < a.ntiles ? __ldg(a.tile_seg + q.c2) : make_uint4(0u, 0u, 0u, 0u);  // used a step later
            q.c3 = atomicAdd(a.sync, 1u);                                                      // used a step later
            // the next STATS tile's octets, prefetched into L2 by the block during this step
            sm.pf_o = q.c1 < a.ntiles ? q.ts1.z : 0u;
            sm.pf_no = q.c1 < a.ntiles ? q.ts1.w : 0u;
        }
        if (t.s_seg != kNone || t.b_seg != kNone) return;
        if (sm.qn == 0 && sm.ovf_seg >= a.nseg) {
            t.kind = kQTaskExit;
            return;
        }
        // nothing runnable: wait for the oldest pending segment's statistics (every STATS tile
        // is claimed by a running CTA, which completes it without waiting: always progresses)
        const uint32_t s = sm.qn > 0 ? sm.q[sm.qh].seg : sm.ovf_seg;
        uint32_t ns = 32;
        while (!q2_ready(a, s)) {
            __nanosleep(ns);
            ns = ns < 1024 ? 2 * ns : ns;
        }
        q.ready_seg = s;
        if (s == q.ready_upto) {
            q.ready_upto += 1;
            q.poll = 0;
        }
    }
}

// Issued right after a decision, consumed at the next one (latency hidden by the step).
__device__ __forceinline__ void q2_prefetch(const Q2Args& a, QSched& q) {
    if (q.ready_upto < a.nseg && !q.poll)
        q.poll = __ldg(&a.segs[q.ready_upto].ntile) == 0
                     ? 1u
                     : ld_relaxed(a.sync + kSyncReady + kSyPerSeg * q.ready_upto + kSyReady);
}

template <int SRC>
__global__ void __launch_bounds__(kQThreads, kQCtasPerSm) k_quant(Q2Args a) {
    extern __shared__ __align__(16) unsigned char qraw[];
    Q2Smem& sm = *reinterpret_cast<Q2Smem*>(qraw);
    float4* xsm = reinterpret_cast<float4*>(qraw + ((sizeof(Q2Smem) + 15) & ~size_t(15)));
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {  // this CTA's share of the SM's tensor memory
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&sm.tbase)), "n"(kQTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (uint32_t i = threadIdx.x; i < kQHists * (kBuckets + 1) * 3; i += kQThreads) (&sm.hist[0][0][0])[i] = 0u;
    QSched q{};
    QArrive arr[2] = {};
    QStep t{};
    if (threadIdx.x == 0) {
        q.c1 = atomicAdd(a.sync, 1u);
        q.ts1 = q.c1 < a.ntiles ? __ldg(a.tile_seg + q.c1) : make_uint4(0u, 0u, 0u, 0u);
        q.c2 = atomicAdd(a.sync, 1u);
        q.ts2 = q.c2 < a.ntiles ? __ldg(a.tile_seg + q.c2) : make_uint4(0u, 0u, 0u, 0u);
        q.c3 = atomicAdd(a.sync, 1u);
        q.ready_upto = 0;
        q.poll = 0;
        q.ready_seg = ~0u;
        sm.ovf_seg = 0;
        sm.freemask = (1u << kQSlots) - 1u;
        sm.qh = 0;
        sm.qn = 0;
        sm.lut_seg = -1;
        sm.bin_seg = -1;
        sm.pf_no = 0;
        sm.clip[0] = sm.clip[1] = 0u;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (;;) {
        if (threadIdx.x == 0) {
            q2_decide(a, sm, q, arr, t);
            q2_prefetch(a, q);
            sm.step = t;
        }
        __syncthreads();
        const QStep st = sm.step;
        if (st.kind == kQTaskExit) break;
        if (st.kind == kQTaskStep) q2_step<SRC>(a, sm, xsm, st, arr);
        else if (st.kind == kQTaskFinStats) q2_finalize_stats(a, sm, st.s_seg, a.segs[st.s_seg]);
        else q2_finalize_codebook(a, st.s_seg, a.segs[st.s_seg]);
        __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tbase), "n"(kQTmemCols));
}

}  // namespace emesh_b200
