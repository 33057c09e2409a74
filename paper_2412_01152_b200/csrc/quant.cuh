// Segment-resident quantizer (k_quant): the reference's quantize
// (proj/include/emesh/quant.hpp:28-87) over every segment of one ring batch,
// with its producer fused in (pseudo-gradient optim.hpp:108, ring hop add
// allreduce.hpp:422, owner mean :435-439).
//
// quantize is two passes over a segment: the statistics (mu, sigma over ALL
// of the segment, quant.hpp:33-43) before any bucket can be assigned
// (:57-76). The value being quantized, x, is produced by the first pass and
// consumed by the second. At the benchmarked shapes a segment is 15.6M-16M
// elements (62.5 MB of x) — twice the GPU's shared memory — so round 1 kept x
// in an L2/HBM scratch and paid 8 B/element of DRAM for it. Here x stays ON
// CHIP: the warp that produced a unit of x parks it in its share of the SM's
// tensor memory (4 units) or shared memory (1 unit) until the segment's
// statistics are final, then bins it itself. Only units beyond a warp's
// on-chip capacity go to a global scratch (an overflow any warp may bin).
//
// Every warp is an independent worker (no block barriers in the steady
// state): it claims 4-unit quads of the batch in segment order, and per
// unit issues the STATS loads, bins one ready unit of its own while they fly
// (pure compute on on-chip x), then finishes the STATS unit. A warp only
// ever waits (for a segment's statistics) when no unit is left to claim, so
// progress never depends on co-residency (a plain launch suffices).
//
// Statistics stay deterministic under dynamic claiming: every unit writes its
// own moment leaf; the last unit of each fixed 64-unit block merges the
// block's leaves in index order, the last block of the segment merges the
// blocks in order and publishes the segment (mu, sigma, lo/hi/width,
// the exact threshold table and bucket encodings). Bucket sums are exact
// integers (order-free). Codes, codebooks and everything after them are
// therefore independent of the schedule.
//
// Element layout of a warp unit: 128 octets (8 floats = 32 B) of the arena's
// octet grid; lane l at step j (0..3) owns octet o0 + 128 u + 32 j + l, so one
// warp instruction moves 1 KB contiguous (256-bit LDG/STG, sm_100). The
// lane's 32 values x[8 j + e] are one tcgen05 32x32b row of its TMEM lane.
#pragma once

#include "kernels.cuh"

namespace emesh_b200 {

constexpr int kQWarps = 16;
constexpr int kQThreads = kQWarps * 32;  // 512: one CTA per SM
constexpr int kWTmemSlots = 4;           // units per warp in tensor memory (its 128-column share)
constexpr int kWSmemSlots = 1;           // units per warp in shared memory
constexpr int kWSlots = kWTmemSlots + kWSmemSlots;
constexpr uint32_t kSlotGlobal = 0xffu;
constexpr int kUnitOct = 128;            // octets per warp unit (1024 elements)
constexpr int kQuad = 4;                 // units per claim
constexpr int kBlkUnits = 64;            // units per leaf block (deterministic two-level merge)
constexpr int kWFlushUnits = 4;          // BIN units per histogram flush
constexpr uint32_t kNone = 0xffffffffu;

// Bin-pass limbs of a warp's histogram over <= kWFlushUnits units (4096 members):
// A = r[0:8) | 1 << 20 (count), B = r[8:28), C = r[28:42) (rare).
// 4096 * 255 < 2^20; 4096 < 2^12; 4096 * (2^20 - 1) < 2^32; 4096 * (2^14 - 1) < 2^32.
constexpr int kWLoBits = 8, kWCntShift = 20, kWMidEnd = 28;

// Per-segment sync words of one launch (zeroed per launch): base kSyncReady + 5 s; the
// leaf-block arrival counters follow at kSyncReady + 5 nseg.
enum : uint32_t { kSyReady = 0, kSyBlocks = 1, kSyBins = 2, kSyOvfCount = 3, kSyOvfClaim = 4, kSyPerSeg = 5 };

struct Q2Args {
    const SegInfo* segs;
    const uint32_t* seg_u0;    // [nseg + 1] first unit of each segment (batch-relative, segment-major)
    uint32_t nseg;
    uint32_t nunits;           // units of the batch
    const float* a;
    const float* b;
    const uint8_t* in_codes;
    const float* in_cb;
    float divisor;
    float inv_divisor;  // 1/k when k is a power of two (exact), else 0
    float* scratch;     // overflow x, octet-addressed: segment s at octets [so0, so0 + nu8 * 128)
    uint8_t* dcodes[kMaxDest];
    float* dcb[kMaxDest];
    uint32_t ndest;
    uint32_t* sflag[kMaxDest];
    uint32_t nflag;
    const uint32_t* in_flag;
    uint32_t epoch;
    unsigned long long timeout_ns;
    SegStat* stats;     // by slot
    StatP* leaf;        // by unit
    StatP* blk_leaf;    // by leaf block
    SegAcc* acc;        // by batch-local segment (self-cleaning)
    uint32_t* seg_flags;
    uint32_t* err;
    uint32_t* sync;     // [0] quad claim counter; per segment kSyPerSeg words from kSyncReady; block counters
    uint32_t* ovf;      // overflow unit lists: segment s's at [u0, u0 + nu8)
    // peer transport: ChunkMsg headers written next to every payload / checked on receipt
    ChunkHdr* dhdr[kMaxDest];
    const ChunkHdr* in_hdr;
    HdrRef hdr;
    uint32_t phase_out;  // kPhaseRS, or kPhaseAG for the owner's final payload
    uint32_t culprit_in; // rank that owes the incoming payloads (the predecessor)
};

struct QHeld {
    uint32_t seg, unit, slot;  // unit: within the segment
};

// One warp's shared memory (private: no cross-warp coordination).
struct WSm {
    double2 bsk[kBuckets];                 // BIN: per bucket {s, K}: fixed point m = x * s + K (kInfoWide)
    uint32_t hist[kBuckets + 1][3];        // BIN: limbs over <= kWFlushUnits units; row 256: sink
    float thr[kBuckets + 2];               // BIN: exact thresholds; [256] = +inf, [257] = lo_up
    float lut[kBuckets];                   // STATS: incoming codebook (hop add)
    float bp[6];                           // BIN params: c, inv_w, lo_up, hi_dn, margin, 1 - margin
    uint32_t degenerate;
    int32_t lut_seg, bin_seg, hist_seg;
    uint32_t hist_units, clip_lo, clip_hi;
    uint32_t qh, qn, freemask;
    QHeld q[kWSlots];
    float4 x[kWSmemSlots][256];            // on-chip x slot(s) in shared memory
};
constexpr uint32_t kMaxSegCache = 512;     // seg_u0 cached in shared memory when it fits
struct QCta {
    uint32_t tbase;                        // TMEM base address
    uint32_t seg_u0[kMaxSegCache + 1];
};
constexpr size_t kQ2SmemBytes = ((sizeof(QCta) + 15) & ~size_t(15)) + kQWarps * ((sizeof(WSm) + 15) & ~size_t(15));

// ---------------------------------------------------------------------------
// memory helpers

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


__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t bcast(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }

// Where a unit's x lives between its STATS and BIN passes.
struct QSlotRef {
    uint32_t slot;    // < kWTmemSlots: TMEM; < kWSlots: smem; kSlotGlobal: overflow scratch
    uint32_t taddr;   // TMEM address of the unit's 32 columns
    float4* sp;       // smem unit (256 float4: [j][lane] low half, [j][32 + lane] high half)
    float* gp;        // overflow scratch of the segment, arena-indexed by element
};

__device__ __forceinline__ QSlotRef q2_slot(const Q2Args& a, uint32_t tbase, WSm& ws, const SegInfo& si,
                                            uint32_t slot) {
    const int warp = threadIdx.x >> 5;
    QSlotRef r;
    r.slot = slot;
    r.taddr = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 128u * (uint32_t)(warp >> 2) + 32u * (slot & 3u);
    r.sp = ws.x[0];
    r.gp = a.scratch + ((int64_t)si.so0 - (int64_t)si.o0) * 8;
    return r;
}

// x of octets j = 2h, 2h + 1 (16 values per lane) into / out of the slot
__device__ __forceinline__ void q2_put_half(const QSlotRef& r, uint64_t obase, int h, const float* x) {
    const int lane = threadIdx.x & 31;
    if (r.slot < kWTmemSlots) {
        tmem_st16(r.taddr + 16u * (uint32_t)h, x);
    } else if (r.slot < kWSlots) {
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
    if (r.slot < kWTmemSlots) {
        tmem_ld16(r.taddr + 16u * (uint32_t)h, x);
    } else if (r.slot < kWSlots) {
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
// STATS: the fused producer (PG / hop add / owner mean) + per-lane moments

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
__device__ __forceinline__ void q2_stats_finish(const Q2Args& a, const WSm& sm, const SegInfo& si, uint64_t obase,
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


// ---------------------------------------------------------------------------
// BIN (exact codes + exact bucket sums into the warp's histogram)

// Bins one octet group of 8 values (codes + exact bucket sums).
template <bool INTERIOR>
__device__ __forceinline__ void q2_bin_octet(const Q2Args& a, WSm& sm, const float* xe, uint64_t o,
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
        red_shared_add_relaxed(hc, (rlo[i] & ((1u << kWLoBits) - 1u)) | (1u << kWCntShift));
        red_shared_add_relaxed(hc + 1, (rlo[i] >> kWLoBits) & ((1u << (kWMidEnd - kWLoBits)) - 1u));
        const uint32_t rc = __funnelshift_r(rlo[i], rhi[i], kWMidEnd) & ((1u << (42 - kWMidEnd)) - 1u);
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


// ---------------------------------------------------------------------------
// Segment statistics: leaves -> blocks -> segment (warp-level, fixed order)

__device__ __forceinline__ StatP ldcg_statp(const StatP* src) {
    StatP c;
    c.s = __ldcg(&src->s); c.m2 = __ldcg(&src->m2); c.d = __ldcg(&src->d);
    c.piv = __ldcg(&src->piv); c.n = __ldcg(&src->n);
    return c;
}
// Fixed-order merge of n consecutive leaves by one warp: lane l merges leaves l, l+32, ... in
// order, then the lanes merge in lane order (warp_merge). Deterministic for a given n.
__device__ StatP warp_merge_range(const StatP* src, uint32_t n) {
    const int lane = threadIdx.x & 31;
    StatP p{0.0, 0.0, 0.0, 0.0, 0};
    for (uint32_t i = lane; i < n; i += 32) p = statp_merge(p, ldcg_statp(src + i));
    return warp_merge(p);
}

// Run by the warp whose block arrival completed segment s: mu / sigma / lo / hi / width
// (quant.hpp:33-59), the exact threshold table and bucket encodings; publishes SegStat(s).
__device__ void q2_finalize_stats(const Q2Args& a, uint32_t s, const SegInfo& si) {
    const int lane = threadIdx.x & 31;
    const StatP t = warp_merge_range(a.blk_leaf + si.b0, si.nblk);
    double mu = 0.0, sigma = 0.0;
    if (lane == 0) {
        mu = __ddiv_rn(t.s, (double)si.len);
        const double dm = __dsub_rn(t.piv, mu);
        // sum (x - mu)^2 = M2 + 2 (p - mu) D + n (p - mu)^2
        double ss = __dadd_rn(t.m2, __dmul_rn(__dmul_rn(2.0, dm), t.d));
        ss = __dadd_rn(ss, __dmul_rn((double)t.n, __dmul_rn(dm, dm)));
        const double var = __ddiv_rn(ss < 0.0 ? 0.0 : ss, (double)si.len);
        sigma = __dsqrt_rn(var);
    }
    mu = __shfl_sync(0xffffffffu, mu, 0);
    sigma = __shfl_sync(0xffffffffu, sigma, 0);
    SegStat* st = &a.stats[si.slot];
    if (lane == 0) {
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
        float thr[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int b = lane + 32 * i;
            thr[i] = b == 0 ? lo_up : threshold(b, lo, hi, w);
            st->thr[b] = b == 0 ? -INFINITY : thr[i];
        }
        // bucket b spans [thr[b], thr[b + 1]): the next threshold is lane + 1's (or the next row's)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int b = lane + 32 * i;
            float nxt = __shfl_down_sync(0xffffffffu, thr[i], 1);
            const float row_next = __shfl_sync(0xffffffffu, thr[i < 7 ? i + 1 : 7], 0);
            if (lane == 31) nxt = i < 7 ? row_next : key2f(f2key(hi_dn) + 1);
            st->binfo[b] = bucket_info(thr[i], nxt);
        }
        if (lane == 0) {
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
    __syncwarp();
    if (lane == 0) {
        __threadfence();  // every lane's SegStat stores (observed through the warp barrier)
        st_release(a.sync + kSyncReady + kSyPerSeg * s + kSyReady, 1u);
    }
    __syncwarp();
}

// A finished STATS unit (its leaf stored by lane 0): arrival on its leaf block; the unit that
// completes a block merges it; the block that completes the segment finalizes the segment.
__device__ void q2_stats_arrive(const Q2Args& a, uint32_t s, const SegInfo& si, uint32_t unit) {
    const int lane = threadIdx.x & 31;
    const uint32_t blk = unit / kBlkUnits, bsize = min((uint32_t)kBlkUnits, si.nu8 - blk * kBlkUnits);
    uint32_t* blk_cnt = a.sync + kSyncReady + kSyPerSeg * a.nseg;
    uint32_t old = 0;
    if (lane == 0) old = atom_add_acq_rel(blk_cnt + si.b0 + blk, 1u);  // publishes the leaf
    old = bcast(old);
    if (old != bsize - 1) return;
    const StatP p = warp_merge_range(a.leaf + si.u0 + blk * kBlkUnits, bsize);
    uint32_t oldb = 0;
    if (lane == 0) {
        a.blk_leaf[si.b0 + blk] = p;
        oldb = atom_add_acq_rel(a.sync + kSyncReady + kSyPerSeg * s + kSyBlocks, 1u);
    }
    oldb = bcast(oldb);
    if (oldb == si.nblk - 1) q2_finalize_stats(a, s, si);
}

// ---------------------------------------------------------------------------
// BIN: the warp's tables, histogram flush, codebook

__device__ void q2_bin_tables(const Q2Args& a, WSm& ws, uint32_t s, const SegInfo& si) {
    const int lane = threadIdx.x & 31;
    const SegStat* st = &a.stats[si.slot];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int b = lane + 32 * i;
        ws.thr[b] = b == 0 ? -INFINITY : __ldcg(&st->thr[b]);
        const uint32_t info = __ldcg(&st->binfo[b]);
        // s = high word of info (low bits zero), K = 2^52 (+ 2^41 for a wide bucket)
        ws.bsk[b] = make_double2(__hiloint2double((int)(info & ~kInfoWide), 0),
                                 __hiloint2double((int)(0x43300000u | ((info & kInfoWide) << 9)), 0));
    }
    if (lane == 0) {
        ws.thr[kBuckets] = INFINITY;
        ws.thr[kBuckets + 1] = __ldcg(&st->lo_up);
        const float margin = __ldcg(&st->margin);
        ws.bp[0] = __ldcg(&st->c_f);
        ws.bp[1] = __ldcg(&st->inv_w_f);
        ws.bp[2] = __ldcg(&st->lo_up);
        ws.bp[3] = __ldcg(&st->hi_dn);
        ws.bp[4] = margin;
        ws.bp[5] = 1.f - margin;
        ws.degenerate = (__ldcg(&st->flags) & kFlagDegenerate) != 0;
        ws.bin_seg = (int32_t)s;
    }
    __syncwarp();
}

__device__ void q2_finalize_codebook(const Q2Args& a, uint32_t s, const SegInfo& si);

// The warp's histogram (units of segment hist_seg) into the segment's exact accumulator,
// then its arrival; the arrival that completes the segment writes the codebook.
__device__ void q2_flush(const Q2Args& a, WSm& ws, uint32_t& nclip_lo, uint32_t& nclip_hi) {
    const int lane = threadIdx.x & 31;
    if (ws.hist_seg < 0) return;
    const uint32_t s = (uint32_t)ws.hist_seg;
    SegAcc* acc = &a.acc[s];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int b = lane + 32 * i;
        const uint32_t A = ws.hist[b][0], B = ws.hist[b][1], Cc = ws.hist[b][2];
        const unsigned long long r = (unsigned long long)(A & ((1u << kWCntShift) - 1u)) +
                                     ((unsigned long long)B << kWLoBits) + ((unsigned long long)Cc << kWMidEnd);
        const uint32_t cn = A >> kWCntShift;
        ws.hist[b][0] = 0u;
        ws.hist[b][1] = 0u;
        ws.hist[b][2] = 0u;
        if (cn) {
            atomicAdd(&acc->rlo[b], r & 0xffffffffull);
            if (r >> 32) atomicAdd(&acc->rhi[b], r >> 32);
            atomicAdd(&acc->cnt[b], (unsigned long long)cn);
        }
    }
    const uint32_t clo = warp_sum_u(nclip_lo), chi = warp_sum_u(nclip_hi);
    nclip_lo = nclip_hi = 0;
    if (lane == 0) {
        if (clo) atomicAdd(&acc->clip[0], (unsigned long long)clo);
        if (chi) atomicAdd(&acc->clip[1], (unsigned long long)chi);
    }
    if (lane < 3) ws.hist[kBuckets][lane] = 0u;
    const uint32_t units = ws.hist_units;
    __syncwarp();
    uint32_t old = 0;
    if (lane == 0) {
        ws.hist_seg = -1;
        ws.hist_units = 0;
        // acq_rel: releases the warp's accumulator atomics and code stores (through the warp
        // barrier above); the arrival that completes the segment acquires all
        old = atom_add_acq_rel(a.sync + kSyncReady + kSyPerSeg * s + kSyBins, units);
    }
    old = bcast(old);
    __syncwarp();
    const SegInfo& si = a.segs[s];
    if (old + units == si.nu8) q2_finalize_codebook(a, s, si);
}

// Run by the warp whose flush completed segment s: the codebook from the exact bucket sums
// (quant.hpp:78-85); re-zeroes the accumulator; ChunkMsg headers; raises the arrival flags.
__device__ void q2_finalize_codebook(const Q2Args& a, uint32_t s, const SegInfo& si) {
    const int lane = threadIdx.x & 31;
    const SegStat* st = &a.stats[si.slot];
    SegAcc* acc = &a.acc[s];
    unsigned long long rl[8], rh[8], total[8];
    const unsigned long long clip_lo = __ldcg(&acc->clip[0]), clip_hi = __ldcg(&acc->clip[1]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int b = lane + 32 * i;
        rl[i] = __ldcg(&acc->rlo[b]);
        rh[i] = __ldcg(&acc->rhi[b]);
        const unsigned long long clip = b == 0 ? clip_lo : b == 255 ? clip_hi : 0ull;
        total[i] = __ldcg(&acc->cnt[b]) + clip;  // clipped members sit in the sink row
    }
    __syncwarp();  // every read done before the re-zeroing
    const bool degenerate = (__ldcg(&st->flags) & kFlagDegenerate) != 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int b = lane + 32 * i;
        acc->rlo[b] = 0ull;
        acc->rhi[b] = 0ull;
        acc->cnt[b] = 0ull;
        const unsigned long long clip = b == 0 ? clip_lo : b == 255 ? clip_hi : 0ull;
        float v;
        if (degenerate) v = (float)__ldcg(&st->mu);
        else if (total[i] == 0)
            v = (float)__dadd_rn(__ldcg(&st->lo), __dmul_rn(__dadd_rn((double)b, 0.5), __ldcg(&st->width)));
        else v = codebook_entry(st, b, rl[i], rh[i], total[i], clip);
        for (uint32_t d = 0; d < a.ndest; ++d) a.dcb[d][(uint64_t)si.slot * kBuckets + b] = v;
    }
    if (lane < 2) acc->clip[lane] = 0ull;
    __syncwarp();
    if (lane == 0) {
        for (uint32_t d = 0; d < a.ndest; ++d)  // the ChunkMsg header of this payload, before its flag
            if (a.dhdr[d]) write_hdr(a.dhdr[d] + si.slot, a.hdr, si.chunk, (uint32_t)si.len, (uint8_t)a.phase_out);
        if (a.nflag) {
            // every unit of s released its stores (gpu scope) to the arrival counter this warp
            // acquired; the system-scope fence + release extends that chain to the peers
            __threadfence_system();
            const uint32_t v = raise_value(a.err, a.epoch);  // poison when this rank's round failed
            for (uint32_t f = 0; f < a.nflag; ++f) st_release_sys(a.sflag[f] + si.slot, v);
        }
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// The warp worker

// Batch unit -> segment (binary search over seg_u0; cached in shared memory when it fits).
__device__ __forceinline__ uint32_t q2_seg_of(const Q2Args& a, const QCta& cta, uint32_t u) {
    const uint32_t* t = a.nseg <= kMaxSegCache ? cta.seg_u0 : a.seg_u0;
    uint32_t lo = 0, hi = a.nseg;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (t[mid] <= u) lo = mid; else hi = mid;
    }
    return lo;
}

// STATS: the incoming codebook of segment s (hop add), after the peer flag (warp-level)
__device__ void q2_stats_lut(const Q2Args& a, WSm& ws, uint32_t s, const SegInfo& si) {
    const int lane = threadIdx.x & 31;
    if (a.in_flag) {  // peer transport: the predecessor's payload of s must have landed intact
        if (lane == 0 && spin_until_ge_sys(a.in_flag + si.in_slot, a.epoch, a.err, a.timeout_ns, a.culprit_in) &&
            a.in_hdr)
            check_hdr(a.in_hdr + si.in_slot, a.hdr, si.chunk, (uint32_t)si.len, kPhaseRS, a.err, a.culprit_in);
        __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) ws.lut[lane + 32 * i] = __ldcg(a.in_cb + (uint64_t)si.in_slot * kBuckets + lane + 32 * i);
    if (lane == 0) ws.lut_seg = (int32_t)s;
    __syncwarp();
}

template <int SRC>
__global__ void __launch_bounds__(kQThreads, 1) k_quant(Q2Args a) {
    extern __shared__ __align__(16) unsigned char qraw[];
    QCta& cta = *reinterpret_cast<QCta*>(qraw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WSm& ws = *reinterpret_cast<WSm*>(qraw + ((sizeof(QCta) + 15) & ~size_t(15)) +
                                      (size_t)warp * ((sizeof(WSm) + 15) & ~size_t(15)));
    if (warp == 0) {  // the whole tensor memory of this SM (one CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&cta.tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (a.nseg <= kMaxSegCache)
        for (uint32_t i = threadIdx.x; i <= a.nseg; i += kQThreads) cta.seg_u0[i] = a.seg_u0[i];
    for (uint32_t i = lane; i < (kBuckets + 1) * 3; i += 32) (&ws.hist[0][0])[i] = 0u;
    if (lane == 0) {
        ws.lut_seg = ws.bin_seg = ws.hist_seg = -1;
        ws.hist_units = 0;
        ws.qh = ws.qn = 0;
        ws.freemask = (1u << kWSlots) - 1u;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = cta.tbase;

    // claims: quads of units in batch order (one atomic per 4 units), one quad ahead
    const uint32_t nquads = (a.nunits + kQuad - 1) / kQuad;
    uint32_t cq = 0, cn = 0;  // current quad's next unit and end (units)
    uint32_t nq = bcast(lane == 0 ? atomicAdd(a.sync, 1u) : 0u);  // the next claimed quad
    uint32_t ovf_seg = 0;     // lowest segment that may still hold unclaimed overflow units
    uint32_t ready_seg = kNone;
    uint32_t nclip_lo = 0, nclip_hi = 0;
    for (;;) {
        // ---- STATS unit: the next claimed unit (claim the quad after it now)
        uint32_t su = kNone;
        if (cq == cn && nq < nquads) {
            cq = nq * kQuad;
            cn = min(cq + kQuad, a.nunits);
            nq = bcast(lane == 0 ? atomicAdd(a.sync, 1u) : 0u);  // used one quad later
        }
        if (cq < cn) su = cq++;
        // ---- BIN unit: the oldest held unit whose segment is ready, else an overflow unit
        uint32_t bseg = kNone, bunit = 0, bslot = kSlotGlobal;
        if (ws.qn > 0) {
            const QHeld h = ws.q[ws.qh];
            bool rdy = h.seg == ready_seg;
            if (!rdy) {
                uint32_t v = lane == 0 ? ld_relaxed(a.sync + kSyncReady + kSyPerSeg * h.seg + kSyReady) : 0u;
                rdy = bcast(v) != 0u;
                if (rdy) { __threadfence(); ready_seg = h.seg; }
            }
            if (rdy) {
                bseg = h.seg; bunit = h.unit; bslot = h.slot;
                __syncwarp();
                if (lane == 0) { ws.qh = (ws.qh + 1) % kWSlots; ws.qn -= 1; }
            }
        }
        if (bseg == kNone && (su == kNone || ws.qn == kWSlots)) {
            // overflow units of ready segments (any warp may bin those)
            while (ovf_seg < a.nseg) {
                const SegInfo& so = a.segs[ovf_seg];
                if (so.nu8 == 0) { ++ovf_seg; continue; }
                uint32_t got = kNone, more = 0;
                if (lane == 0) {
                    uint32_t* sy = a.sync + kSyncReady + kSyPerSeg * ovf_seg;
                    if (ld_relaxed(sy + kSyReady)) {
                        __threadfence();
                        const uint32_t cnt = __ldcg(sy + kSyOvfCount);
                        more = 1;
                        if (cnt && __ldcg(sy + kSyOvfClaim) < cnt) {
                            const uint32_t i = atomicAdd(sy + kSyOvfClaim, 1u);
                            if (i < cnt) got = __ldcg(a.ovf + so.u0 + i);
                        }
                    }
                }
                got = bcast(got);
                more = bcast(more);
                if (got != kNone) { bseg = ovf_seg; bunit = got; bslot = kSlotGlobal; break; }
                if (!more) break;  // not ready yet
                ++ovf_seg;        // ready and exhausted
            }
        }
        if (su == kNone && bseg == kNone) {
            if (ws.qn == 0 && ovf_seg >= a.nseg && nq >= nquads) break;  // done
            // nothing runnable: every unit is claimed (by running warps, which complete their
            // STATS without waiting): wait for the oldest pending segment's statistics
            const uint32_t s = ws.qn > 0 ? ws.q[ws.qh].seg : ovf_seg;
            if (lane == 0) {
                uint32_t ns = 32;
                while (ld_acquire(a.sync + kSyncReady + kSyPerSeg * s + kSyReady) == 0u) {
                    __nanosleep(ns);
                    ns = ns < 1024 ? 2 * ns : ns;
                }
            }
            __syncwarp();
            ready_seg = s;
            continue;
        }
        // ---- STATS setup (segment, slot, LUT)
        uint32_t sseg = kNone, sunit = 0, sslot = kSlotGlobal, ovf_i = 0;
        SegInfo ss{}, sb{};
        if (su != kNone) {
            sseg = q2_seg_of(a, cta, su);
            ss = a.segs[sseg];
            sunit = su - ss.u0;
            if ((SRC & kHasIn) && ws.lut_seg != (int32_t)sseg) q2_stats_lut(a, ws, sseg, ss);
            if (ws.freemask) {
                sslot = __ffs(ws.freemask) - 1;
                __syncwarp();
                if (lane == 0) {
                    ws.freemask &= ~(1u << sslot);
                    ws.q[(ws.qh + ws.qn) % kWSlots] = QHeld{sseg, sunit, sslot};
                    ws.qn += 1;
                }
            } else if (lane == 0) {
                ovf_i = atomicAdd(a.sync + kSyncReady + kSyPerSeg * sseg + kSyOvfCount, 1u);  // used at the end
            }
        }
        // ---- BIN setup (tables, histogram segment)
        if (bseg != kNone) {
            sb = a.segs[bseg];
            if (ws.hist_seg != (int32_t)bseg) {  // a histogram holds one segment: flush the previous one
                q2_flush(a, ws, nclip_lo, nclip_hi);
                if (lane == 0) ws.hist_seg = (int32_t)bseg;
                __syncwarp();
            }
            if (ws.bin_seg != (int32_t)bseg) q2_bin_tables(a, ws, bseg, sb);
        }
        // ---- the fused unit: STATS loads in flight while the BIN half is computed
        const bool vs = sseg != kNone, vb = bseg != kNone;
        const uint64_t hs = ss.lo + ss.len, hb = sb.lo + sb.len;
        const uint64_t os = ss.o0 + (uint64_t)sunit * kUnitOct, ob = sb.o0 + (uint64_t)bunit * kUnitOct;
        const bool is = vs && os * 8 >= ss.lo && (os + kUnitOct) * 8 <= hs;
        const bool ib = vb && ob * 8 >= sb.lo && (ob + kUnitOct) * 8 <= hb;
        const QSlotRef rs = q2_slot(a, tbase, ws, ss, sslot), rb = q2_slot(a, tbase, ws, sb, bslot);
        QMoments m{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0u, false};
        uint32_t* hw = &ws.hist[0][0];
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            QLoads<SRC> L;
            if (vs) q2_stats_load<SRC>(a, os, hs, is, h, L);
            if (vb) {  // bin this half while the loads fly
                float y[16];
                q2_get_half(rb, ob, h, y);
                if (ws.degenerate) {  // sigma == 0: every code is 0 (quant.hpp:49-55)
                    for (int jj = 0; jj < 2; ++jj) {
                        const uint64_t o = ob + (uint64_t)(2 * h + jj) * 32 + lane;
                        for (int e = 0; e < 8; ++e)
                            if (o * 8 + e >= sb.lo && o * 8 + e < hb)
                                for (uint32_t d = 0; d < a.ndest; ++d) a.dcodes[d][o * 8 + e] = 0;
                    }
                } else if (ib) {
                    q2_bin_octet<true>(a, ws, &y[0], ob + (uint64_t)(2 * h) * 32 + lane, sb, hw, nclip_lo, nclip_hi);
                    q2_bin_octet<true>(a, ws, &y[8], ob + (uint64_t)(2 * h + 1) * 32 + lane, sb, hw, nclip_lo, nclip_hi);
                } else {
                    q2_bin_octet<false>(a, ws, &y[0], ob + (uint64_t)(2 * h) * 32 + lane, sb, hw, nclip_lo, nclip_hi);
                    q2_bin_octet<false>(a, ws, &y[8], ob + (uint64_t)(2 * h + 1) * 32 + lane, sb, hw, nclip_lo, nclip_hi);
                }
            }
            if (vs) {
                q2_stats_finish<SRC>(a, ws, ss, os, is, h, L, m);
                q2_put_half(rs, os, h, L.a);
            }
        }
        // ---- BIN epilogue: slot free, scratch discard, histogram accounting
        if (vb) {
            if (bslot == kSlotGlobal && ib) {
                // consumed (read exactly once): drop the unit's scratch lines from L2 without write-back
                const uintptr_t lo_b = reinterpret_cast<uintptr_t>(rb.gp + ob * 8);
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(lo_b + (uintptr_t)lane * 128) : "memory");
            }
            __syncwarp();
            if (lane == 0) {
                if (bslot < kWSlots) ws.freemask |= 1u << bslot;
                ws.hist_units += 1;
            }
            __syncwarp();
            if (ws.hist_units == kWFlushUnits) q2_flush(a, ws, nclip_lo, nclip_hi);
        }
        // ---- STATS epilogue: the unit's leaf, overflow registration, arrival
        if (vs) {
            StatP p{__dadd_rn(m.s0, m.s1), __dadd_rn(m.q0, m.q1), __dadd_rn(m.d0, m.d1), m.piv, (uint64_t)m.cnt};
            p = warp_merge(p);
            if (lane == 0) {
                a.leaf[ss.u0 + sunit] = p;
                if (sslot == kSlotGlobal) a.ovf[ss.u0 + ovf_i] = sunit;  // for BIN by any warp (published below)
                if (!isfinite(p.s) || !isfinite(p.m2)) {  // finite fp32 inputs cannot overflow an fp64 sum
                    atomicOr(&a.seg_flags[sseg], kFlagNonFinite);
                    atomicOr(a.err, kErrNonFinite);
                }
            }
            __syncwarp();  // the lanes' scratch stores, then lane 0's release (cumulative)
            q2_stats_arrive(a, sseg, ss, sunit);
        }
    }
    q2_flush(a, ws, nclip_lo, nclip_hi);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

}  // namespace emesh_b200

