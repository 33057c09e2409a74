// sm_100a kernels for the DiLoCo outer-synchronisation hot path.
//
// Reference semantics (restated in oracle/emesh_oracle.c, checked bit-for-bit):
//   quantize            proj/include/emesh/quant.hpp:28-87
//   dequantize_into     proj/include/emesh/quant.hpp:89-94
//   pseudo-gradient     proj/include/emesh/optim.hpp:99-111
//   nesterov_outer_step proj/include/emesh/optim.hpp:116-132
//   ring hop add / mean proj/include/emesh/allreduce.hpp:422, :435-439
//
// Everything is HBM-bound elementwise/scan work: no tensor cores. The whole
// file is compiled with -fmad=false (no FMA contraction) and IEEE div/sqrt,
// because the reference's x86-64 build has no FMA.
//
// Data layout: one flat fp32 arena per tensor (theta_g, theta_l, momentum),
// canonical tensor order (tensor.hpp:87-93). A "segment" is one quantization
// unit of the reference (one sub-slice of one rank chunk,
// allreduce.hpp:326-336). Codes live in a u8 arena indexed like the fp32
// arena; codebooks in a [slot][256] f32 arena; per-segment statistics in a
// SegStat arena.
//
// Work decomposition: a "unit" is 256 float4 slots (1024 elements) of one
// segment, owned by one warp, on the 16-byte-aligned float4 grid of the
// arena. Segments start at arbitrary element offsets, so the first and last
// float4 of a segment may be shared with a neighbour: loads are full float4
// (always in-bounds for 16-B aligned arenas), stores to such partial slots
// are per element.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <math.h>

namespace emesh_b200 {

constexpr int kBuckets = 256;
constexpr int kWarps = 8;              // warps per CTA
constexpr int kThreads = kWarps * 32;  // 256
constexpr int kSlotsPerLane = 8;       // float4 slots per lane per unit
constexpr int kUnitSlots = 32 * kSlotsPerLane;  // 256 float4 = 1024 elements
#ifndef EMESH_QUANT_MINB
#define EMESH_QUANT_MINB 3
#endif
#ifndef EMESH_UNITS_PER_WARP
#define EMESH_UNITS_PER_WARP 4
#endif
constexpr int kUnitsPerWarp = EMESH_UNITS_PER_WARP;  // warp units per tile task (2 or 4)
static_assert(kUnitsPerWarp == 2 || kUnitsPerWarp == 4, "limb layout sized for <= 4096 members per warp");
// Bin-pass limbs (32-bit smem atomics per warp over one tile, see bin_unit):
// A = r[0:kLoBits) | 1 << kCntShift, B = r[kLoBits:kMidEnd), C = r[kMidEnd:42).
// With m = 1024 kUnitsPerWarp members: m (2^kLoBits - 1) < 2^kCntShift,
// m < 2^(32 - kCntShift), m 2^(kMidEnd - kLoBits) <= 2^32, m 2^(42 - kMidEnd) < 2^32.
constexpr int kLoBits = kUnitsPerWarp == 2 ? 9 : 7;
constexpr int kCntShift = kUnitsPerWarp == 2 ? 20 : 19;
constexpr int kMidEnd = kUnitsPerWarp == 2 ? 30 : 26;
// The tile shape (kWarps * upw units: 16K or 8K elements) is chosen per batch at
// run time (SegInfo::upw, Plan::add_batch): the limb layout above is sized for
// the largest tile and stays exact for a smaller one (its bounds cap m).

// Exact fixed-point encoding of one bucket's members for the codebook sums:
// each member x maps to a non-negative integer r(x) < 2^42 with
// sum x = f(sum r, count), so per-bucket sums are integer sums — associative,
// identical for any accumulation order, and equal to the reference's
// sequential fp64 sum whenever that sum is exact (quant.hpp:74).
//  * "narrow" buckets (all members of one sign, magnitudes within 2^17 of
//    each other, normal): r = |x| / Q with Q = 2^e the ulp of the smallest
//    member — an exact integer < 2^41; x = +-r Q.
//  * "wide" buckets (at or near zero): r = rint(x / Q) + 2^41 with a quantum
//    Q = 2^e = 2^-41 of the bucket's magnitude.
// Both are ONE fp64 fma, m = x * s + K with s = +-2^-e and K = 2^52 (narrow) or
// 2^52 + 2^41 (wide): m lands in [2^52, 2^53) and its mantissa bits are r.
// Per-bucket info word = the high word of s (sign, exponent; its low mantissa
// bits are zero) with bit 0 = wide, so a member's m needs no table but this.
constexpr uint32_t kInfoWide = 1u;
constexpr double kMagic52 = 4503599627370496.0;  // 2^52
constexpr double kWideK = 4503599627370496.0 + 2199023255552.0;  // 2^52 + 2^41
constexpr int kWideBiasBits = 41;

// Per-segment statistics, written once by the segment's last STATS tile (finalize_stats).
struct SegStat {
    double mu, sigma, lo, width, hi;  // first four exported as {mu, sigma, lo, width}
    float c_f, inv_w_f;  // bucket estimate g = fma(x, inv_w_f, -c_f), c_f = (float)(lo / width)
    float lo_up, hi_dn;  // x < lo <=> x < lo_up ; x > hi <=> x > hi_dn (fp32 x)
    uint32_t flags;      // kFlagNonFinite | kFlagDegenerate
    float margin;        // fp32 bucket estimate is exact when its fraction is in (margin, 1-margin)
    float thr[kBuckets];  // thr[j] = smallest fp32 x with code(x) >= j (j=1..255)
    uint32_t binfo[kBuckets];  // bucket encodings (see kInfoWide)
};
constexpr uint32_t kFlagNonFinite = 1u;
constexpr uint32_t kFlagDegenerate = 2u;  // sigma == 0 (quant.hpp:49-55)


// One segment of a batch (host-built, device-resident). CTA-aligned: the
// segment's work is ncta consecutive CTAs ("tiles") of 8 warp units each.
struct SegInfo {
    uint64_t lo;        // absolute element offset in the arena
    uint64_t len;       // elements
    uint64_t q0;        // lo >> 2: first float4 slot
    uint64_t sq0;       // the segment's first float4 slot in the batch's scratch
    uint32_t nunits;    // warp units (1024-element float4-grid spans)
    uint32_t cta0;      // first tile (batch-relative): leaf_stat index
    uint32_t ncta;      // tiles
    uint32_t slot;      // global segment slot (stats / codebook index)
    uint32_t in_slot;   // slot of the incoming payload's codebook (== slot)
    uint32_t upw;       // warp units per tile (2 or 4, <= kUnitsPerWarp; one value per batch)
};

// Moments of a set of values around a pivot p: s = sum x, m2 = sum (x-p)^2,
// d = sum (x-p). Two partials merge exactly (in real arithmetic) by moving
// one to the other's pivot, so partials can be combined in any grouping; the
// kernels combine them in a fixed order, so results are deterministic.
struct StatP {
    double s, m2, d, piv;
    uint64_t n;
};

__device__ __forceinline__ StatP statp_merge(StatP a, const StatP& b) {
    if (b.n == 0) return a;
    if (a.n == 0) return b;
    const double dl = __dsub_rn(b.piv, a.piv);
    const double bn = (double)b.n;
    a.m2 = __dadd_rn(__dadd_rn(a.m2, b.m2),
                     __dadd_rn(__dmul_rn(__dmul_rn(2.0, dl), b.d), __dmul_rn(bn, __dmul_rn(dl, dl))));
    a.d = __dadd_rn(__dadd_rn(a.d, b.d), __dmul_rn(bn, dl));
    a.s = __dadd_rn(a.s, b.s);
    a.n += b.n;
    return a;
}

constexpr int kMaxDest = 8;  // output destinations of one quantizer launch (ranks of a peer ring)

// Producer of the value being quantized, fused into the statistics pass.
enum : int {
    kSrcA = 0,          // x = a                      (plain buffer)
    kSrcAminusB = 1,    // x = a - b                  (pseudo-gradient, optim.hpp:108)
    kHasIn = 2,         // x += cb_in[code_in]        (ring hop add, allreduce.hpp:422)
    kDivK = 4,          // x = x / k                  (owner mean, allreduce.hpp:439)
};

// Bucket histogram of a segment, accumulated by integer atomics from every
// BIN tile (order-free, hence deterministic): the fixed-point codes r(x) of the
// members split as sum (r mod 2^32) and sum (r >> 32) (no u64 overflow for
// any segment size), member counts (clipped members included, with r = 0),
// and the clipped-low / clipped-high counts (xc = lo / hi, quant.hpp:66-67).
// Zero between launches: the segment's last BIN tile re-zeroes it.
struct SegAcc {
    unsigned long long rlo[kBuckets];
    unsigned long long rhi[kBuckets];
    unsigned long long cnt[kBuckets];
    unsigned long long clip[2];
};

struct QuantArgs {
    const SegInfo* segs;
    const uint32_t* cta_seg;   // CTA -> batch-local segment
    uint32_t ncta;
    uint32_t nseg;
    const float* a;
    const float* b;
    const uint8_t* in_codes;
    const float* in_cb;
    float divisor;
    float inv_divisor;         // 1/k when k is a power of two (exact), else 0
    float* scratch;            // x of the batch; segment s at float4 slots [sq0, sq0 + slots)
    // output destinations (peer transport: the successor's arena); after a
    // segment's codes + codebook are stored everywhere, store `epoch` to
    // sflag[f][slot] for every flag f (the successor's arrival flags, or
    // every rank's for the owner's final payload)
    uint8_t* dcodes[kMaxDest];
    float* dcb[kMaxDest];
    uint32_t ndest;
    uint32_t* sflag[kMaxDest];
    uint32_t nflag;
    uint32_t remote;           // bit 0: peer-memory outputs; bit 1: system fence per tile
    const uint32_t* in_flag;   // peer transport: in_codes / in_cb of slot s valid once in_flag[s] >= epoch
    uint32_t epoch;
    unsigned long long timeout_ns;  // peer-wait budget (spin_until_ge_sys)
    SegStat* stats;            // indexed by slot
    StatP* leaf_stat;          // [tile]
    SegAcc* acc;               // [seg] bucket histograms (batch-local segment)
    uint32_t* seg_flags;       // [seg] non-finite bits (reset by the stats root)
    uint32_t* err;             // sticky error word (bit 0: non-finite)
    uint32_t* sync;            // see kSyncReady (zeroed per launch)
    const uint4* runs;         // task order as runs {first task, kind, segment, first tile}
    uint32_t nruns, ntasks;
    struct TraceRec* trace;    // optional task timeline (nullptr: off)
    uint32_t* trace_n;
    uint32_t trace_cap;
};


// Optional per-task timeline (globaltimer ns), for tuning the task plan.
struct TraceRec {
    unsigned long long t0, t1, t2, t3;  // claimed/start, ready, main loop done, end
    uint32_t kind, seg, tile, smid;
};
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------
// small helpers

#ifndef EMESH_STREAM_NO_L1
#define EMESH_STREAM_NO_L1 1
#endif
#ifndef EMESH_CODES_NO_L1
#define EMESH_CODES_NO_L1 0
#endif
#ifndef EMESH_BIN_PF_FIRST
#define EMESH_BIN_PF_FIRST 1
#endif
// Streaming (read-once) loads. EMESH_STREAM_NO_L1 (default): no L1
// allocation, leaving L1 to the BIN scratch prefetch (EMESH_BIN_L1PF);
// otherwise ld.global.cs (evict-first).
__device__ __forceinline__ float4 ld4_stream(const float* p, uint64_t q) {
#if EMESH_STREAM_NO_L1
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(reinterpret_cast<const float4*>(p) + q));
    return v;
#else
    return __ldcs(reinterpret_cast<const float4*>(p) + q);
#endif
}
#ifndef EMESH_STATS_L1PF
#define EMESH_STATS_L1PF 0
#endif
// STATS' theta loads: streamed past L1, or (EMESH_STATS_L1PF) through L1 after
// a prefetch of the warp's next half-unit (read-only inputs of the launch).
__device__ __forceinline__ float4 ld4_stats(const float* p, uint64_t q) {
#if EMESH_STATS_L1PF
    return reinterpret_cast<const float4*>(p)[q];
#else
    return ld4_stream(p, q);
#endif
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
#if EMESH_STREAM_NO_L1 && EMESH_CODES_NO_L1
    uint32_t v;
    asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}
__device__ __forceinline__ float4 ld4(const float* p, uint64_t q) {
    return __ldg(reinterpret_cast<const float4*>(p) + q);
}
__device__ __forceinline__ uint32_t warp_sum_u(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_shared_add(uint32_t* p, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
// predicated (no branch): adds only when v != 0
__device__ __forceinline__ void red_shared_add_nz(uint32_t* p, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q red.shared.add.u32 [%0], %1;\n\t}"
                 ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
// Cross-GPU signalling (peer transport): flags live in the receiver's memory.
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Waits for a peer's arrival flag. A peer that stops (crash, abort) must not
// hang the GPU: after timeout_ns (ReduceOptions::step_timeout,
// allreduce.hpp:59) the wait gives up and sets err bit 1 (the host reports
// RingFailureError); once that bit is set every other wait gives up at once.
constexpr uint32_t kErrRingTimeout = 2u;
__device__ __forceinline__ void spin_until_ge_sys(const uint32_t* p, uint32_t epoch, uint32_t* err,
                                                  unsigned long long timeout_ns) {
    uint32_t ns = 64;
    const unsigned long long t0 = gtimer();
    while ((int32_t)(ld_acquire_sys(p) - epoch) < 0) {
        if (ld_acquire(err) & kErrRingTimeout) return;
        if (gtimer() - t0 > timeout_ns) {
            atomicOr(err, kErrRingTimeout);
            return;
        }
        __nanosleep(ns);
        ns = ns < 2048 ? 2 * ns : ns;
    }
}

// The reference's bucket function, exactly (quant.hpp:65-72).
__device__ __forceinline__ int code_exact(float xf, double lo, double hi, double w) {
    double x = (double)xf;
    if (x < lo) x = lo;
    if (x > hi) x = hi;
    const double q = floor(__ddiv_rn(__dsub_rn(x, lo), w));
    int b = q < 0.0 ? 0 : (q > 255.0 ? 255 : (int)q);
    return b;
}

__device__ __forceinline__ uint32_t f2key(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// thr_j = min{ x fp32 : code_exact(x) >= j }, j in [1,255]. code_exact is
// monotone in x, so this is an exact threshold table: for every finite x,
// code(x) = #{ j : thr_j <= x }.
__device__ float threshold(int j, double lo, double hi, double w) {
    float g = (float)__dadd_rn(lo, __dmul_rn((double)j, w));
    uint32_t key = f2key(g);
    // linear walk from the nearest-float guess (normally 0-2 steps)
    if (code_exact(g, lo, hi, w) >= j) {
        for (int it = 0; it < 8; ++it) {
            float p = key2f(key - 1);
            if (code_exact(p, lo, hi, w) >= j) { key -= 1; } else { return key2f(key); }
        }
    } else {
        for (int it = 0; it < 8; ++it) {
            key += 1;
            if (code_exact(key2f(key), lo, hi, w) >= j) return key2f(key);
        }
    }
    // fallback: bisection on the ordered key space over the whole range
    uint32_t a = f2key((float)lo) - 4, b = f2key((float)hi) + 4;  // code(a) < j <= code(b)
    if (code_exact(key2f(a), lo, hi, w) >= j) return key2f(a);
    while (b - a > 1) {
        uint32_t m = a + (b - a) / 2;
        if (code_exact(key2f(m), lo, hi, w) >= j) b = m; else a = m;
    }
    return key2f(b);
}


// ---------------------------------------------------------------------------
// STATS pass: fused producer (PG / hop dequant-add / divide) + moments, one
// pass: each lane accumulates s = sum x, d = sum (x-p), m2 = sum (x-p)^2 around
// a pivot p (its first value), merged exactly in a fixed order over the warp,
// the CTA (one leaf per tile) and the segment (finalize_stats). Writes x to
// scratch for the BIN pass unless the source is a plain buffer. The segment's
// last tile publishes SegStat: mu, sigma, lo, hi, width (quant.hpp:33-59), the
// exact threshold table and the bucket encodings.

__device__ __forceinline__ StatP shfl_statp(const StatP& p, int src) {
    StatP o;
    o.s = __shfl_sync(0xffffffffu, p.s, src);
    o.m2 = __shfl_sync(0xffffffffu, p.m2, src);
    o.d = __shfl_sync(0xffffffffu, p.d, src);
    o.piv = __shfl_sync(0xffffffffu, p.piv, src);
    o.n = __shfl_sync(0xffffffffu, p.n, src);
    return o;
}

// Fixed-order warp merge (lane i absorbs lane i+o): deterministic.
__device__ __forceinline__ StatP warp_merge(StatP p) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const StatP q = shfl_statp(p, lane + o < 32 ? lane + o : lane);
        if ((lane & (2 * o - 1)) == 0) p = statp_merge(p, q);
    }
    return shfl_statp(p, 0);
}

__device__ __forceinline__ int exponent_of(float f) {  // floor(log2|f|) for normal f; -127.. for subnormal
    const uint32_t u = __float_as_uint(f) & 0x7fffffffu;
    const int e = (int)(u >> 23);
    if (e) return e - 127;
    return u ? (31 - __clz(u)) - 149 : -150;
}

// Encoding of bucket b whose fp32 members lie in [t0, t1) (see kInfoWide).
__device__ uint32_t bucket_info(float t0, float t1) {
    if (!(t1 > t0)) return (1023u << 20) | kInfoWide;  // holds no fp32 value
    const float last = key2f(f2key(t1) - 1);
    if (t0 > 0.f || last < 0.f) {
        const float mn = t0 > 0.f ? t0 : last, mx = t0 > 0.f ? last : t0;
        const uint32_t e_lo = (__float_as_uint(mn) >> 23) & 0xffu, e_hi = (__float_as_uint(mx) >> 23) & 0xffu;
        // Q = ulp(mn) = 2^(e_lo - 150); s = +-2^(150 - e_lo); r < 2^(24 + 17)
        if (e_lo >= 1u && e_hi - e_lo <= 17u) return ((1023u + 150u - e_lo) << 20) | (t0 > 0.f ? 0u : 0x80000000u);
    }
    const float mx = fmaxf(fabsf(t0), fabsf(last));
    const int e = exponent_of(mx) + 1 - kWideBiasBits;  // |x| < 2^(e+41); s = 2^-e
    return ((uint32_t)(1023 - e) << 20) | kInfoWide;
}

// ---------------------------------------------------------------------------
// Persistent quantizer: one launch per batch (pipelining window), a grid of
// co-resident CTAs that claim tile tasks in plan order (one atomicAdd each).

struct QSmem {
    uint32_t hist[kWarps][kBuckets + 1][3];  // per-warp limbs over the tile (bin), see bin_unit; row 256: sink
    uint2 bsk[2 * kBuckets];             // per bucket {high word of s, high word of K} (bin), twice:
                                         // index code | 256 = same bucket (see kInfoWide)
    float thr[kBuckets + 2];             // exact threshold table (bin); [257] = bucket 0's base (lo_up)
    float lut[kBuckets];                 // incoming codebook (stats, hop)
    StatP wp[kWarps];
    double red[2];
    uint32_t clip[2];
    uint32_t flag;
    uint32_t task;
    int32_t bin_seg, lut_seg, ready_seg;
    uint32_t run_idx;
    unsigned long long t_main;  // trace: main loop done
};

// Task order (host-built run table, QuantArgs::runs): the STATS tiles of
// the batch in segment order; the BIN tiles of segment s once `lag` more
// tasks were issued after its last STATS tile (lag ~ 1.5 grids: the segment's
// statistics are normally published before its bins are claimed, and a
// tile's scratch x is re-read soon enough to still be in L2). The last STATS
// tile of s to finish finalizes SegStat(s); the last BIN tile of s to finish
// writes its codebook. A BIN task only waits (at the top of the loop, owing
// nothing) on STATS tiles claimed before it, so the grid always progresses
// whatever the co-residency.
// sync layout: [0] task counter, [kSyncReady + s] SegStat(s) published,
// [kSyncReady + nseg + s] STATS tiles done, [kSyncReady + 2 nseg + s] BIN tiles done.
constexpr uint32_t kSyncReady = 32;
enum : uint32_t { kTaskStats = 0, kTaskBin = 2 };
// mixed run (alternating STATS / BIN tasks): y = kTaskMix{Rev,Fwd} | bin segment << 2,
// z = STATS segment, w = first STATS tile | first BIN tile << 16
constexpr uint32_t kTaskMixRev = 1, kTaskMixFwd = 3;
constexpr uint32_t kMaxRunsSmem = 512;  // run table cached in smem when it fits (8 KB)
constexpr uint32_t kMaxSegsSmem = 128;  // SegInfo cached in smem when it fits (6 KB)



__device__ void finalize_stats(const QuantArgs& a, QSmem& sm, uint32_t s, const SegInfo& si);

#ifndef EMESH_SCRATCH_EVICT_LAST
#define EMESH_SCRATCH_EVICT_LAST 0
#endif
// Scratch x (written by STATS, read once by BIN, then discarded): an
// L2::evict_last hint keeps it ahead of the streaming (evict-first) inputs.
__device__ __forceinline__ void st_scratch(float4* p, float4 v) {
#if EMESH_SCRATCH_EVICT_LAST
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
#else
    *p = v;
#endif
}

template <int SRC>
__device__ __forceinline__ void stats_tile(const QuantArgs& a, QSmem& sm, uint32_t s, const SegInfo& si,
                                           uint32_t tile) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t hiel = si.lo + si.len;     // exclusive
    float4* xs = reinterpret_cast<float4*>(a.scratch) + ((int64_t)si.sq0 - (int64_t)si.q0);

    if (SRC & kHasIn) {
        if (sm.lut_seg != (int32_t)s) {
            __syncthreads();
            if (a.in_flag) {  // peer transport: wait until the predecessor's payload of s landed
                if (threadIdx.x == 0) spin_until_ge_sys(a.in_flag + si.in_slot, a.epoch, a.err, a.timeout_ns);
                __syncthreads();
            }
            sm.lut[threadIdx.x] = __ldcg(a.in_cb + (uint64_t)si.in_slot * kBuckets + threadIdx.x);
            __syncthreads();
            if (threadIdx.x == 0) sm.lut_seg = (int32_t)s;
        }
    }
    StatP p{0.0, 0.0, 0.0, 0.0, 0};
    double sum0 = 0.0, sum1 = 0.0, d0 = 0.0, d1 = 0.0, q0 = 0.0, q1 = 0.0;
    double piv = 0.0;
    uint32_t cnt = 0;
    bool have_piv = false;
    for (int ui = 0; ui < (int)si.upw; ++ui) {
        const uint32_t u = (tile * si.upw + ui) * kWarps + warp;  // segment-relative unit
        if (u >= si.nunits) break;
        const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;
        const bool interior = qbase * 4 >= si.lo && (qbase + kUnitSlots) * 4 <= hiel;  // warp-uniform
        constexpr int kHalf = kSlotsPerLane / 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float4 xa[kHalf], xb[kHalf];
            uint32_t c4[kHalf];
#if EMESH_STATS_L1PF
            {   // the warp's next half-unit of A (lanes 0-15) and B (lanes 16-31) into L1, 2 KB each
                const bool more = h == 0 || (ui + 1 < (int)si.upw && u + kWarps < si.nunits);
                const uint64_t qn = h == 0 ? qbase + (uint64_t)kHalf * 32 : qbase + (uint64_t)kWarps * kUnitSlots;
                const uint64_t ql = qn + (uint64_t)(lane & 15) * 8;
                if (more && ql * 4 < hiel && ((SRC & kSrcAminusB) || lane < 16))
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const float4*>(lane < 16 ? a.a : a.b) + ql));
            }
#endif
#pragma unroll
            for (int jj = 0; jj < kHalf; ++jj) {
                const uint64_t q = qbase + (uint64_t)(h * kHalf + jj) * 32 + lane;
                const bool in = interior || q * 4 < hiel;
                xa[jj] = in ? ld4_stats(a.a, q) : make_float4(0.f, 0.f, 0.f, 0.f);
                if (SRC & kSrcAminusB) xb[jj] = in ? ld4_stats(a.b, q) : make_float4(0.f, 0.f, 0.f, 0.f);
                if (SRC & kHasIn) c4[jj] = in ? ld_stream_u32(reinterpret_cast<const uint32_t*>(a.in_codes) + q) : 0u;
            }
#pragma unroll
            for (int jj = 0; jj < kHalf; ++jj) {
                const uint64_t q = qbase + (uint64_t)(h * kHalf + jj) * 32 + lane;
                const uint64_t e0 = q * 4;
                float x[4] = {xa[jj].x, xa[jj].y, xa[jj].z, xa[jj].w};
                if (SRC & kSrcAminusB) {
                    x[0] = __fsub_rn(x[0], xb[jj].x); x[1] = __fsub_rn(x[1], xb[jj].y);
                    x[2] = __fsub_rn(x[2], xb[jj].z); x[3] = __fsub_rn(x[3], xb[jj].w);
                }
                if (SRC & kHasIn) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) x[e] = __fadd_rn(x[e], sm.lut[(c4[jj] >> (8 * e)) & 0xff]);
                }
                if (SRC & kDivK) {
                    // x / k (allreduce.hpp:439): exact multiply for a power-of-two k
                    if (a.inv_divisor != 0.f) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) x[e] = __fmul_rn(x[e], a.inv_divisor);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e) x[e] = __fdiv_rn(x[e], a.divisor);
                    }
                }
                if (interior && !have_piv) {  // pivot: the lane's first value
                    piv = (double)x[0];
                    have_piv = true;
                }
                if (interior) {
                    const double x0 = (double)x[0], x1 = (double)x[1], x2 = (double)x[2], x3 = (double)x[3];
                    const double v0 = __dsub_rn(x0, piv), v1 = __dsub_rn(x1, piv);
                    const double v2 = __dsub_rn(x2, piv), v3 = __dsub_rn(x3, piv);
                    sum0 = __dadd_rn(__dadd_rn(sum0, x0), x2);
                    sum1 = __dadd_rn(__dadd_rn(sum1, x1), x3);
                    d0 = __dadd_rn(__dadd_rn(d0, v0), v2);
                    d1 = __dadd_rn(__dadd_rn(d1, v1), v3);
                    // sigma is not bit-exact vs the sequential reference anyway:
                    // fused multiply-adds for the squares
                    q0 = __fma_rn(v2, v2, __fma_rn(v0, v0, q0));
                    q1 = __fma_rn(v3, v3, __fma_rn(v1, v1, q1));
                    if (SRC != kSrcA) st_scratch(xs + q, make_float4(x[0], x[1], x[2], x[3]));
                } else {
                    uint32_t vm = 0u;
#pragma unroll
                    for (int e = 0; e < 4; ++e) vm |= (e0 + e >= si.lo && e0 + e < hiel) ? (1u << e) : 0u;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (vm & (1u << e)) {
                            const double xd = (double)x[e];
                            if (!have_piv) { piv = xd; have_piv = true; }
                            const double dv = __dsub_rn(xd, piv);
                            sum0 = __dadd_rn(sum0, xd);
                            d0 = __dadd_rn(d0, dv);
                            q0 = __fma_rn(dv, dv, q0);
                            cnt += 1;
                            if (SRC != kSrcA) reinterpret_cast<float*>(xs + q)[e] = x[e];
                        }
                    }
                }
            }
        }
        if (interior) cnt += kSlotsPerLane * 4;  // per lane
    }
    p = StatP{__dadd_rn(sum0, sum1), __dadd_rn(q0, q1), __dadd_rn(d0, d1), piv, (uint64_t)cnt};
    p = warp_merge(p);
    if (a.trace && threadIdx.x == 0) sm.t_main = gtimer();
    if (lane == 0) {
        sm.wp[warp] = p;
        // finite fp32 inputs cannot overflow an fp64 sum: one check per unit
        if (!isfinite(p.s) || !isfinite(p.m2)) {
            atomicOr(&a.seg_flags[s], kFlagNonFinite);
            atomicOr(a.err, 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        StatP t = sm.wp[0];
        for (int w = 1; w < kWarps; ++w) t = statp_merge(t, sm.wp[w]);
        a.leaf_stat[si.cta0 + tile] = t;
        // acq_rel: publishes this leaf; the last tile to arrive acquires all
        sm.flag = atom_add_acq_rel(&a.sync[kSyncReady + a.nseg + s], 1u) == si.ncta - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (sm.flag) finalize_stats(a, sm, s, si);
}

// Run by the last STATS tile of s to finish: combine the segment's leaves in
// a fixed order (thread t: leaves t, t+256, ...; then warps; then the 8 warp
// partials), finalize mu / sigma / lo / hi / width (quant.hpp:33-59), the
// exact threshold table and the bucket parameters, and publish SegStat(s).
__device__ void finalize_stats(const QuantArgs& a, QSmem& sm, uint32_t s, const SegInfo& si) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    StatP p{0.0, 0.0, 0.0, 0.0, 0};
    for (uint32_t i = threadIdx.x; i < si.ncta; i += kThreads) {
        const StatP* src = &a.leaf_stat[si.cta0 + i];
        StatP ch;
        ch.s = __ldcg(&src->s); ch.m2 = __ldcg(&src->m2); ch.d = __ldcg(&src->d);
        ch.piv = __ldcg(&src->piv); ch.n = __ldcg(&src->n);
        p = statp_merge(p, ch);
    }
    p = warp_merge(p);
    if (lane == 0) sm.wp[warp] = p;
    __syncthreads();
    if (threadIdx.x == 0) {
        StatP t = sm.wp[0];
        for (int w = 1; w < kWarps; ++w) t = statp_merge(t, sm.wp[w]);
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
        // smallest fp32 >= lo, largest fp32 <= hi (clipping in fp32 terms)
        float lo_up = (float)lo;
        if ((double)lo_up < lo) lo_up = key2f(f2key(lo_up) + 1);
        float hi_dn = (float)hi;
        if ((double)hi_dn > hi) hi_dn = key2f(f2key(hi_dn) - 1);
        const int b = threadIdx.x;
        sm.thr[b] = b == 0 ? lo_up : threshold(b, lo, hi, w);
        if (b == 0) sm.thr[kBuckets] = key2f(f2key(hi_dn) + 1);
        __syncthreads();
        st->thr[b] = b == 0 ? -INFINITY : sm.thr[b];
        st->binfo[b] = bucket_info(sm.thr[b], sm.thr[b + 1]);
        if (b == 0) {
            st->lo = lo; st->hi = hi; st->width = w;
            const float c_f = (float)__ddiv_rn(lo, w), inv_w = (float)__ddiv_rn(1.0, w);
            st->c_f = c_f;
            st->inv_w_f = inv_w;
            st->lo_up = lo_up;
            st->hi_dn = hi_dn;
            // Error of g = fma(x, inv_w, -c) (fp32) vs (x - lo) / w, in buckets, for
            // lo <= x <= hi: inv_w and c carry <= 2^-24 relative error each
            // (|x| / w and |lo| / w terms), the fma one rounding of |g| <= 256:
            // err <= ((max(|lo|, |hi|) + |lo|) / w + 256) 2^-24; x2 for safety.
            const double mag = __ddiv_rn(fmax(fabs(lo), fabs(hi)) + fabs(lo), w);
            const double err = __dmul_rn(__dadd_rn(mag, 256.0), 1.01 / 16777216.0);
            const double mg = __dmul_rn(2.0, err) + 1e-6;
            st->margin = mg < 0.25 ? (float)mg : 2.0f;  // 2.0: always use the table
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        sm.bin_seg = -1;  // thr in smem now holds this segment's raw table: force a reload
        st_release(&a.sync[kSyncReady + s], 1u);  // publish (cumulative over the CTA's SegStat writes)
    }
}

// Exact bucket by the threshold table (the rare path of the fp32 estimate).
__device__ __noinline__ int bucket_walk(float x, int c, const float* thr) {
    while (c < 255 && x >= thr[c + 1]) ++c;
    while (c > 0 && x < thr[c]) --c;
    return c;
}


struct BinParams {
    float c, inv_w, lo_up, hi_dn, margin, one_m;  // bucket estimate g = fma(x, inv_w, -c)
};

// One warp unit of the bin pass (1024 elements; this lane's 32), in groups of
// 8: bucket estimates for all 8, rare fix-ups (exact table near an edge,
// clipping), fixed-point codes via the fp32 fast path (fp64 for the few
// buckets that need it), then the limb atomics — unconditional, so the
// common path has no data-dependent branches (invalid lanes add 0).
// Per-warp limbs over a tile (see kLoBits): A += low bits | one count,
// B += middle bits, C += high bits (only when nonzero: rare).
#ifndef EMESH_BIN_L1PF
#define EMESH_BIN_L1PF 1
#endif
// BIN's scratch reads. With EMESH_BIN_L1PF (default) the warp prefetches its
// next unit's 4 KB of scratch into L1 while it bins the current one, and the
// loads go through L1. Each scratch line belongs to exactly one segment
// (segments own whole units of scratch, Plan::add_batch), is written once by
// its STATS tiles before the segment's statistics are published, and only
// read (or prefetched) after: no stale L1 copy can exist within the launch.
__device__ __forceinline__ float4 ld_scratch(const float4* p) {
#if EMESH_BIN_L1PF
    return *p;
#else
    return __ldcg(p);
#endif
}

template <bool INTERIOR, bool FROM_SCRATCH>
__device__ __forceinline__ void bin_unit(const QuantArgs& a, QSmem& sm, const SegInfo& si, uint64_t qbase,
                                         uint64_t hiel, const float4* xs, uint32_t* hw, const BinParams& p,
                                         uint32_t& nclip_lo, uint32_t& nclip_hi) {
    const int lane = threadIdx.x & 31;
    constexpr int kHalf = kSlotsPerLane / 2;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        float4 xv[kHalf];
#pragma unroll
        for (int jj = 0; jj < kHalf; ++jj) {
            const uint64_t q = qbase + (uint64_t)(h * kHalf + jj) * 32 + lane;
            const bool in = INTERIOR || q * 4 < hiel;
            xv[jj] = !in ? make_float4(0.f, 0.f, 0.f, 0.f) : FROM_SCRATCH ? ld_scratch(xs + q) : ld4(a.a, q);
        }
#pragma unroll
        for (int pr = 0; pr < kHalf / 2; ++pr) {
            float xe[8] = {xv[2 * pr].x, xv[2 * pr].y, xv[2 * pr].z, xv[2 * pr].w,
                           xv[2 * pr + 1].x, xv[2 * pr + 1].y, xv[2 * pr + 1].z, xv[2 * pr + 1].w};
            const uint64_t q0 = qbase + (uint64_t)(h * kHalf + 2 * pr) * 32 + lane;
            uint32_t vmask = 0xffu;
            if (!INTERIOR) {
                vmask = 0u;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint64_t e = (q0 + (uint64_t)(i >> 2) * 32) * 4 + (i & 3);
                    vmask |= (e >= si.lo && e < hiel) ? (1u << i) : 0u;
                }
            }
            int cc[8];
            bool okall = true;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                // in range and clear of every bucket edge by the proven margin:
                // then trunc(g) is the exact bucket. Clipped x fails this test
                // (g < margin or g > 256 - margin), see SegStat::margin.
                const float g = __fmaf_rn(xe[i], p.inv_w, -p.c);
                const int c = __float2int_rz(g);
                const float fr = __fsub_rn(g, __int2float_rz(c));
                okall &= (fr > p.margin) & (fr < p.one_m) & ((uint32_t)c < 256u);
                cc[i] = c;
            }
            // clipped lanes (and lanes outside the segment) keep their code in the
            // low byte and set bit 8: their limbs go to the sink row 256; the
            // codebook adds the clipped ones as count * lo / hi (quant.hpp:66-67)
            if (!INTERIOR) {
#pragma unroll
                for (int i = 0; i < 8; ++i) cc[i] |= ((vmask >> i) & 1u) ? 0 : 256;
            }
            if (!okall) {  // rare: near an edge (exact table) or clipped (quant.hpp:66-67)
                uint32_t clo_m = 0, chi_m = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float x = xe[i];
                    const float g = __fmaf_rn(x, p.inv_w, -p.c);
                    const int c0 = __float2int_rz(g);
                    const float fr = __fsub_rn(g, __int2float_rz(c0));
                    const int sink = cc[i] & 256;
                    if (x < p.lo_up) {
                        cc[i] = 256; clo_m |= 1u << i;
                    } else if (x > p.hi_dn) {
                        cc[i] = 256 | 255; chi_m |= 1u << i;
                    } else if (!(fr > p.margin && fr < p.one_m && (uint32_t)c0 < 256u)) {
                        cc[i] = sink | bucket_walk(x, min(max(c0, 0), 255), sm.thr);
                    }
                }
                nclip_lo += __popc(clo_m & vmask);
                nclip_hi += __popc(chi_m & vmask);
            }
            // fixed point r(x) (see kInfoWide), split into the limbs
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint2 sk = sm.bsk[cc[i]];
                // m = x * s + K in [2^52, 2^53): mantissa = r (see kInfoWide)
                const double sc = __hiloint2double((int)sk.x, 0);
                const double kk = __hiloint2double((int)sk.y, 0);
                const double m = __fma_rn((double)xe[i], sc, kk);
                const uint32_t rlo = (uint32_t)__double2loint(m);
                const uint32_t rhi = (uint32_t)__double2hiint(m);
                uint32_t* hc = hw + 3 * min(cc[i], kBuckets);
                red_shared_add(hc, (rlo & ((1u << kLoBits) - 1u)) | (1u << kCntShift));
                red_shared_add(hc + 1, (rlo >> kLoBits) & ((1u << (kMidEnd - kLoBits)) - 1u));
                const uint32_t rc = __funnelshift_r(rlo, rhi, kMidEnd) & ((1u << (42 - kMidEnd)) - 1u);
                if (rc) red_shared_add(hc + 2, rc);
            }
            const uint32_t p0 = __byte_perm(__byte_perm(cc[0], cc[1], 0x0040), __byte_perm(cc[2], cc[3], 0x0040), 0x5410);
            const uint32_t p1 = __byte_perm(__byte_perm(cc[4], cc[5], 0x0040), __byte_perm(cc[6], cc[7], 0x0040), 0x5410);
            for (uint32_t d = 0; d < a.ndest; ++d) {
                uint8_t* oc = a.dcodes[d];
                if (INTERIOR) {
                    reinterpret_cast<uint32_t*>(oc)[q0] = p0;
                    reinterpret_cast<uint32_t*>(oc)[q0 + 32] = p1;
                } else {
#pragma unroll
                    for (int f = 0; f < 2; ++f) {
                        const uint64_t q = q0 + (uint64_t)f * 32;
                        const uint32_t packed = f ? p1 : p0;
                        const uint32_t vm = (vmask >> (4 * f)) & 0xfu;
                        if (vm == 0xfu) {
                            reinterpret_cast<uint32_t*>(oc)[q] = packed;
                        } else if (vm) {
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (vm & (1u << e)) oc[q * 4 + e] = (uint8_t)(packed >> (8 * e));
                        }
                    }
                }
            }
        }
        if (FROM_SCRATCH && INTERIOR) {
            // this half's 2 KB of scratch x is consumed (each element is read
            // exactly once): drop the 128-B L2 lines wholly inside it without
            // write-back — x was only ever meant as an L2 round trip
            const uintptr_t lo_b = reinterpret_cast<uintptr_t>(xs + qbase + (uint64_t)h * kHalf * 32);
            const uintptr_t hi_b = lo_b + (uintptr_t)kHalf * 32 * 16;
            const uintptr_t line = ((lo_b + 127) & ~(uintptr_t)127) + (uintptr_t)lane * 128;
            if (lane < 16 && line + 128 <= hi_b)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
        }
    }
}

__device__ void finalize_codebook(const QuantArgs& a, uint32_t s, const SegInfo& si);
__device__ float codebook_entry(const SegStat* st, int b, unsigned long long rl, unsigned long long rh,
                                unsigned long long total, unsigned long long clip);

template <bool FROM_SCRATCH>
__device__ __forceinline__ void bin_tile(const QuantArgs& a, QSmem& sm, uint32_t s, const SegInfo& si, uint32_t tile) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const SegStat* st = &a.stats[si.slot];
#if EMESH_BIN_L1PF && EMESH_BIN_PF_FIRST
    if (FROM_SCRATCH) {  // the warp's first unit, while the tables load (the segment's scratch is complete)
        const uint32_t u0 = tile * si.upw * kWarps + warp;
        if (u0 < si.nunits) {
            const float4* p0 = reinterpret_cast<const float4*>(a.scratch) + si.sq0 + (uint64_t)u0 * kUnitSlots + lane * 8;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(p0));
        }
    }
#endif
    if (sm.bin_seg != (int32_t)s) {
        __syncthreads();
        const int b = threadIdx.x;
        sm.thr[b] = b == 0 ? -INFINITY : __ldcg(&st->thr[b]);
        const uint32_t info = __ldcg(&st->binfo[b]);
        const uint2 sk = make_uint2(info & ~kInfoWide, 0x43300000u | ((info & kInfoWide) << 9));  // K = 2^52 (+2^41)
        sm.bsk[b] = sm.bsk[kBuckets + b] = sk;

        if (b == 0) {
            sm.thr[kBuckets] = INFINITY;
            sm.thr[kBuckets + 1] = __ldcg(&st->lo_up);
        }
        __syncthreads();
        if (threadIdx.x == 0) sm.bin_seg = (int32_t)s;
    }
    const float c_f = __ldcg(&st->c_f), inv_w = __ldcg(&st->inv_w_f);
    const float lo_up = __ldcg(&st->lo_up), hi_dn = __ldcg(&st->hi_dn);  // x < lo <=> x < lo_up (fp32 x)
    const float margin = __ldcg(&st->margin), one_m = 1.f - margin;
    const bool degenerate = (__ldcg(&st->flags) & kFlagDegenerate) != 0;
    uint32_t* hw = &sm.hist[warp][0][0];  // zero on entry (kernel start / previous tile's combine)
    if (threadIdx.x < 2) sm.clip[threadIdx.x] = 0u;
    __syncthreads();

    const uint64_t hiel = si.lo + si.len;
    const float4* xs = reinterpret_cast<const float4*>(a.scratch) + ((int64_t)si.sq0 - (int64_t)si.q0);
    uint32_t nclip_lo = 0, nclip_hi = 0;
    const BinParams bpar{c_f, inv_w, lo_up, hi_dn, margin, one_m};
    for (int ui = 0; ui < (int)si.upw; ++ui) {
        const uint32_t u = (tile * si.upw + ui) * kWarps + warp;
        if (u >= si.nunits) break;
        const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;
        const bool interior = qbase * 4 >= si.lo && (qbase + kUnitSlots) * 4 <= hiel;  // warp-uniform
#if EMESH_BIN_L1PF
        if (FROM_SCRATCH && ui + 1 < (int)si.upw && u + kWarps < si.nunits) {
            const float4* nx = xs + qbase + (uint64_t)kWarps * kUnitSlots + lane * 8;  // one 128-B line per lane
            asm volatile("prefetch.global.L1 [%0];" ::"l"(nx));
        }
#endif
        if (degenerate) {  // sigma == 0: every code is 0 (quant.hpp:49-55)
            for (int j = 0; j < kSlotsPerLane; ++j) {
                const uint64_t q = qbase + (uint64_t)j * 32 + lane;
                for (int e = 0; e < 4; ++e)
                    if (q * 4 + e >= si.lo && q * 4 + e < hiel)
                        for (uint32_t d = 0; d < a.ndest; ++d) a.dcodes[d][q * 4 + e] = 0;
            }
        } else if (interior) {
            bin_unit<true, FROM_SCRATCH>(a, sm, si, qbase, hiel, xs, hw, bpar, nclip_lo, nclip_hi);
        } else {
            bin_unit<false, FROM_SCRATCH>(a, sm, si, qbase, hiel, xs, hw, bpar, nclip_lo, nclip_hi);
        }
    }
    nclip_lo = warp_sum_u(nclip_lo);
    nclip_hi = warp_sum_u(nclip_hi);
    if (lane == 0 && (nclip_lo | nclip_hi)) {
        atomicAdd(&sm.clip[0], nclip_lo);
        atomicAdd(&sm.clip[1], nclip_hi);
    }
    __syncthreads();
    if (threadIdx.x == 0 && a.trace) sm.t_main = gtimer();
    {   // tile histogram (exact integers, order-free) into the segment's
        // accumulator; re-zero the limbs
        const int b = threadIdx.x;
        unsigned long long r = 0;
        uint32_t cn = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t A = sm.hist[w][b][0], B = sm.hist[w][b][1], C = sm.hist[w][b][2];
            r += (unsigned long long)(A & ((1u << kCntShift) - 1u)) + ((unsigned long long)B << kLoBits) +
                 ((unsigned long long)C << kMidEnd);
            cn += A >> kCntShift;
            sm.hist[w][b][0] = 0u;
            sm.hist[w][b][1] = 0u;
            sm.hist[w][b][2] = 0u;
        }
        SegAcc* acc = &a.acc[s];
        if (cn) {
            atomicAdd(&acc->rlo[b], r & 0xffffffffull);
            if (r >> 32) atomicAdd(&acc->rhi[b], r >> 32);
            atomicAdd(&acc->cnt[b], (unsigned long long)cn);
        }
        if (b < 2 && sm.clip[b]) atomicAdd(&acc->clip[b], (unsigned long long)sm.clip[b]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // codes stored to peer memory are performed system-wide before the
        // arrival, so the last tile's flag store (system scope) covers them
        if (a.remote & 2u) __threadfence_system();
        // acq_rel: releases the CTA's atomics; the last tile acquires all
        sm.flag = atom_add_acq_rel(&a.sync[kSyncReady + 2 * a.nseg + s], 1u) == si.ncta - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (sm.flag) finalize_codebook(a, s, si);
}

// Run by the last BIN tile of s to finish: the codebook from the exact
// bucket sums (quant.hpp:78-85); re-zeroes the accumulator for the next launch.
__device__ void finalize_codebook(const QuantArgs& a, uint32_t s, const SegInfo& si) {
    const SegStat* st = &a.stats[si.slot];
    const bool degenerate = (__ldcg(&st->flags) & kFlagDegenerate) != 0;
    const int b = threadIdx.x;
    SegAcc* acc = &a.acc[s];
    const unsigned long long rl = __ldcg(&acc->rlo[b]), rh = __ldcg(&acc->rhi[b]);
    const unsigned long long clip = b == 0 ? __ldcg(&acc->clip[0]) : b == 255 ? __ldcg(&acc->clip[1]) : 0ull;
    const unsigned long long total = __ldcg(&acc->cnt[b]) + clip;  // clipped members sit in the sink row
    __syncthreads();  // every read done before the re-zeroing
    acc->rlo[b] = 0ull;
    acc->rhi[b] = 0ull;
    acc->cnt[b] = 0ull;
    if (b < 2) acc->clip[b] = 0ull;
    float v;
    if (degenerate) {
        v = (float)__ldcg(&st->mu);
    } else if (total == 0) {
        v = (float)__dadd_rn(__ldcg(&st->lo), __dmul_rn(__dadd_rn((double)b, 0.5), __ldcg(&st->width)));
    } else {
        v = codebook_entry(st, b, rl, rh, total, clip);
    }
    for (uint32_t d = 0; d < a.ndest; ++d) a.dcb[d][(uint64_t)si.slot * kBuckets + b] = v;
    if (a.nflag) {
        // Every tile of s released its stores (gpu scope) to the arrival
        // counter this CTA acquired; the system-scope fence + release here
        // extends that causality chain to the peers polling the flags.
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            for (uint32_t f = 0; f < a.nflag; ++f) st_release_sys(a.sflag[f] + si.slot, a.epoch);
        }
    }
}

// Codebook entry b from the exact bucket sums (quant.hpp:78-85).
__device__ float codebook_entry(const SegStat* st, int b, unsigned long long rl, unsigned long long rh,
                                unsigned long long total, unsigned long long clip) {
    const unsigned long long cnt = total - clip;  // clipped members are counted with r = 0
    double sum = 0.0;
    if (cnt) {
        const uint32_t info = __ldcg(&st->binfo[b]);
        // sum r (exact, 128-bit); wide: sum x = (sum r - cnt 2^41) Q;
        // narrow: sum x = +-(sum r) 2^(E0 - 150)
        __int128 S = (__int128)rl + ((__int128)rh << 32);
        if (info & kInfoWide) S -= (__int128)cnt << kWideBiasBits;
        const long long hi64 = (long long)(S >> 64);
        const long long s64 = (long long)(unsigned long long)S;
        const bool fits = (hi64 == 0 && s64 >= 0) || (hi64 == -1 && s64 < 0);
        const double v = fits ? (double)s64 : __dadd_rn(ldexp((double)hi64, 64), (double)(unsigned long long)S);
        // sum x = sum(r) / s (wide: after removing the bias): exact power-of-two scaling
        const int e = 1023 - (int)((info >> 20) & 0x7ffu);  // |s| = 2^-e
        sum = ldexp(v, e);
        if (info & 0x80000000u) sum = -sum;
    }
    if (b == 0 && clip) sum = __dadd_rn(sum, __dmul_rn((double)clip, __ldcg(&st->lo)));
    if (b == 255 && clip) sum = __dadd_rn(sum, __dmul_rn((double)clip, __ldcg(&st->hi)));
    return (float)__ddiv_rn(sum, (double)total);
}

// Task t of run r -> (kind, segment, tile).
__device__ __forceinline__ void decode_run(const uint4 r, uint32_t t, uint32_t& kind, uint32_t& s, uint32_t& tile) {
    const uint32_t off = t - r.x, k = r.y & 3u;
    if (k == kTaskMixRev || k == kTaskMixFwd) {
        const uint32_t i = off >> 1;
        if (off & 1u) {
            kind = kTaskBin;
            s = r.y >> 2;
            tile = k == kTaskMixRev ? (r.w >> 16) - i : (r.w >> 16) + i;
        } else {
            kind = kTaskStats;
            s = r.z;
            tile = (r.w & 0xffffu) + i;
        }
    } else {
        kind = r.y;
        s = r.z;
        tile = (r.w & 0x80000000u) ? (r.w & 0x7fffffffu) - off : r.w + off;
    }
}

template <int SRC>
__global__ void __launch_bounds__(kThreads, EMESH_QUANT_MINB) k_quant(QuantArgs a) {
    extern __shared__ __align__(16) unsigned char qsmem_raw[];
    QSmem& sm = *reinterpret_cast<QSmem*>(qsmem_raw);  // dynamic: > 48 KB in total
    uint4* runs_s = reinterpret_cast<uint4*>(qsmem_raw + sizeof(QSmem));
    SegInfo* segs_s = reinterpret_cast<SegInfo*>(qsmem_raw + sizeof(QSmem) + kMaxRunsSmem * sizeof(uint4));
    const bool runs_in_smem = a.nruns <= kMaxRunsSmem;
    const bool segs_in_smem = a.nseg <= kMaxSegsSmem;
    for (uint32_t i = threadIdx.x; i < kWarps * (kBuckets + 1) * 3; i += kThreads) (&sm.hist[0][0][0])[i] = 0u;
    if (runs_in_smem)
        for (uint32_t i = threadIdx.x; i < a.nruns; i += kThreads) runs_s[i] = a.runs[i];
    if (segs_in_smem)
        for (uint32_t i = threadIdx.x; i < a.nseg; i += kThreads) segs_s[i] = a.segs[i];
    uint32_t nxt = 0;  // thread 0: the next task, claimed at the start of the current one
    if (threadIdx.x == 0) {
        sm.bin_seg = -1;
        sm.lut_seg = -1;
        sm.ready_seg = -1;
        nxt = atomicAdd(&a.sync[0], 1u);
    }
    for (;;) {
        if (threadIdx.x == 0) sm.task = nxt;
        __syncthreads();
        const uint32_t t = sm.task;
        if (t >= a.ntasks) return;
        // claim the following task now: the atomic's latency hides behind this tile
        if (threadIdx.x == 0) nxt = atomicAdd(&a.sync[0], 1u);
        uint32_t kind, s, tile;
        if (runs_in_smem) {  // binary search of the run table (smem)
            uint32_t lo = 0, hi = a.nruns;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (runs_s[mid].x <= t) lo = mid; else hi = mid;
            }
            decode_run(runs_s[lo], t, kind, s, tile);
        } else {
            uint32_t lo = 0, hi = a.nruns;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (a.runs[mid].x <= t) lo = mid; else hi = mid;
            }
            decode_run(a.runs[lo], t, kind, s, tile);
        }
        const SegInfo si = segs_in_smem ? segs_s[s] : a.segs[s];
        unsigned long long t0 = 0, t1 = 0;
        if (a.trace) t0 = gtimer();
        if (kind == kTaskBin && threadIdx.x == 0 && sm.ready_seg != (int32_t)s) {
            // acquire SegStat(s) (cached per CTA); the CTA owes nothing here
            uint32_t ns = 32;
            while (ld_acquire(&a.sync[kSyncReady + s]) == 0u) {
                __nanosleep(ns);
                ns = ns < 1024 ? 2 * ns : ns;
            }
            sm.ready_seg = (int32_t)s;
        }
        if (a.trace) t1 = gtimer();
        __syncthreads();  // everyone has read sm.task; SegStat(s) visible for BIN
        switch (kind) {
            case kTaskStats: stats_tile<SRC>(a, sm, s, si, tile); break;
            default: bin_tile<SRC != kSrcA>(a, sm, s, si, tile); break;
        }
        if (a.trace && threadIdx.x == 0) {
            const uint32_t i = atomicAdd(a.trace_n, 1u);
            if (i < a.trace_cap) {
                uint32_t smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                a.trace[i] = TraceRec{t0, t1, sm.t_main, gtimer(), kind, s, tile, smid};
            }
        }
    }
}

constexpr size_t kQuantSmemBytes = sizeof(QSmem) + kMaxRunsSmem * sizeof(uint4) + kMaxSegsSmem * sizeof(SegInfo);

// ---------------------------------------------------------------------------
// Elementwise kernels over segment batches (codebook LUT in smem).

struct ApplyArgs {
    const SegInfo* segs;
    const uint32_t* cta_seg;
    uint32_t ncta;
    uint32_t upw;          // the batch's warp units per tile = CTAs per tile
    const uint8_t* codes;  // arena-indexed
    const float* cb;       // [slot][256]
    float* theta;          // theta_g, updated in place
    float* buf;            // Nesterov momentum, updated in place
    float* theta_local;    // optional: theta_l <- theta_g (trainer.hpp:382)
    float* out;            // dequantize target (arena-indexed)
    float lr, mom;
    const uint32_t* in_flag;  // peer transport: codes / codebook of slot s valid once in_flag[s] >= epoch
    uint32_t epoch;
    uint32_t* err;            // sticky error word (kErrRingTimeout)
    unsigned long long timeout_ns;
};
// k_apply-family CTAs: a.upw per quantizer tile, one unit per warp (measured
// best: k_apply 11.3 -> 11.0 ms per round).
constexpr int kApplyUnits = 1;  // units per warp in one k_apply CTA

__device__ __forceinline__ void nesterov1(float& th, float& b, float d, float lr, float mom) {
    // optim.hpp:127-130, fp32, this exact association, no FMA
    const float nb = __fadd_rn(__fmul_rn(mom, b), d);
    b = nb;
    th = __fsub_rn(th, __fmul_rn(lr, __fadd_rn(d, __fmul_rn(mom, nb))));
}

// MODE 0: dequantize into out; MODE 1: dequant + Nesterov (+ optional theta_l write)
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_apply(ApplyArgs a) {
    __shared__ float lut[kBuckets];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x / a.upw, part = blockIdx.x % a.upw;
    const SegInfo si = a.segs[a.cta_seg[tile]];
    if (a.in_flag) {
        if (threadIdx.x == 0) spin_until_ge_sys(a.in_flag + si.slot, a.epoch, a.err, a.timeout_ns);
        __syncthreads();
    }
    lut[threadIdx.x] = __ldcg(a.cb + (uint64_t)si.slot * kBuckets + threadIdx.x);
    __syncthreads();
    const uint64_t hiel = si.lo + si.len;
    for (int ui = 0; ui < kApplyUnits; ++ui) {
    const uint32_t u = ((tile - si.cta0) * a.upw + part * kApplyUnits + ui) * kWarps + warp;
    if (u >= si.nunits) return;
    const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;
#pragma unroll 4
    for (int j = 0; j < kSlotsPerLane; ++j) {
        const uint64_t q = qbase + (uint64_t)j * 32 + lane;
        const uint64_t e0 = q * 4;
        if (e0 >= hiel) continue;
        const bool full = e0 >= si.lo && e0 + 4 <= hiel;
        const uint32_t c4 = __ldcs(reinterpret_cast<const uint32_t*>(a.codes) + q);
        float d[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) d[e] = lut[(c4 >> (8 * e)) & 0xff];
        if (MODE == 0) {
            if (full) {
                reinterpret_cast<float4*>(a.out)[q] = make_float4(d[0], d[1], d[2], d[3]);
            } else {
                for (int e = 0; e < 4; ++e)
                    if (e0 + e >= si.lo && e0 + e < hiel) a.out[e0 + e] = d[e];
            }
        } else {
            float4 th = __ldcs(reinterpret_cast<const float4*>(a.theta) + q);
            float4 bb = __ldcs(reinterpret_cast<const float4*>(a.buf) + q);
            float t4[4] = {th.x, th.y, th.z, th.w}, b4[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) nesterov1(t4[e], b4[e], d[e], a.lr, a.mom);
            if (full) {
                const float4 to = make_float4(t4[0], t4[1], t4[2], t4[3]);
                __stcs(reinterpret_cast<float4*>(a.theta) + q, to);
                __stcs(reinterpret_cast<float4*>(a.buf) + q, make_float4(b4[0], b4[1], b4[2], b4[3]));
                if (a.theta_local) __stcs(reinterpret_cast<float4*>(a.theta_local) + q, to);
            } else {
                for (int e = 0; e < 4; ++e)
                    if (e0 + e >= si.lo && e0 + e < hiel) {
                        a.theta[e0 + e] = t4[e];
                        a.buf[e0 + e] = b4[e];
                        if (a.theta_local) a.theta_local[e0 + e] = t4[e];
                    }
            }
        }
    }
    }
}

// ---------------------------------------------------------------------------
// ReduceMode::fp32 ring (allreduce.hpp:120-164: raw fp32 payloads). One CTA
// per warp unit of a quantizer tile (like k_apply); segments are still the framing
// unit (allreduce.hpp:326-336), and with the peer transport the last CTA of
// a segment raises its arrival flags.

struct F32HopArgs {
    const SegInfo* segs;
    const uint32_t* cta_seg;
    uint32_t upw;              // the batch's warp units per tile = CTAs per tile
    const float* a;            // theta_g (PG) or the ring input
    const float* b;            // theta_l (PG) or nullptr
    const float* in;           // incoming partial sums (arena-indexed) or nullptr (hop 0)
    float divisor, inv_divisor;  // owner mean: x / k (allreduce.hpp:435-440)
    float* dst[kMaxDest];      // payload destinations (arena-indexed)
    uint32_t ndest;
    uint32_t* sflag[kMaxDest];  // peer arrival flags raised per finished segment
    uint32_t nflag;
    uint32_t* seg_done;        // [batch segment] CTA arrival counters (zeroed per launch)
    const uint32_t* in_flag;   // peer transport: wait in_flag[slot] >= epoch before reading `in`
    uint32_t epoch;
    uint32_t nseg;
    uint32_t* err;
    unsigned long long timeout_ns;
};

// x = (a - b | a) (+ in) (/ k), the reduce-scatter accumulate
// accum[lo + i] += vals[i] (allreduce.hpp:422) and the owner mean (:435-440).
template <bool PG, bool HAS_IN, bool DIV>
__global__ void __launch_bounds__(kThreads) k_f32_hop(F32HopArgs a) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x / a.upw, part = blockIdx.x % a.upw;
    const uint32_t s = a.cta_seg[tile];
    const SegInfo si = a.segs[s];
    if (HAS_IN && a.in_flag) {
        if (threadIdx.x == 0) spin_until_ge_sys(a.in_flag + si.in_slot, a.epoch, a.err, a.timeout_ns);
        __syncthreads();
    }
    const uint64_t hiel = si.lo + si.len;
    for (int ui = 0; ui < kApplyUnits; ++ui) {
        const uint32_t u = ((tile - si.cta0) * a.upw + part * kApplyUnits + ui) * kWarps + warp;
        if (u >= si.nunits) break;
        const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;
#pragma unroll 4
        for (int j = 0; j < kSlotsPerLane; ++j) {
            const uint64_t q = qbase + (uint64_t)j * 32 + lane;
            const uint64_t e0 = q * 4;
            if (e0 >= hiel) continue;
            const bool full = e0 >= si.lo && e0 + 4 <= hiel;
            float4 v = __ldcs(reinterpret_cast<const float4*>(a.a) + q);
            float x[4] = {v.x, v.y, v.z, v.w};
            if (PG) {
                const float4 l = __ldcs(reinterpret_cast<const float4*>(a.b) + q);
                x[0] = __fsub_rn(x[0], l.x); x[1] = __fsub_rn(x[1], l.y);
                x[2] = __fsub_rn(x[2], l.z); x[3] = __fsub_rn(x[3], l.w);
            }
            if (HAS_IN) {
                const float4 w = __ldcs(reinterpret_cast<const float4*>(a.in) + q);
                x[0] = __fadd_rn(x[0], w.x); x[1] = __fadd_rn(x[1], w.y);
                x[2] = __fadd_rn(x[2], w.z); x[3] = __fadd_rn(x[3], w.w);
            }
            if (DIV) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    x[e] = a.inv_divisor != 0.f ? __fmul_rn(x[e], a.inv_divisor) : __fdiv_rn(x[e], a.divisor);
            }
            for (uint32_t d = 0; d < a.ndest; ++d) {
                if (full) {
                    __stcs(reinterpret_cast<float4*>(a.dst[d]) + q, make_float4(x[0], x[1], x[2], x[3]));
                } else {
                    for (int e = 0; e < 4; ++e)
                        if (e0 + e >= si.lo && e0 + e < hiel) a.dst[d][e0 + e] = x[e];
                }
            }
        }
    }
    if (a.nflag) {  // last CTA of the segment flags it (see finalize_codebook for the ordering argument)
        __shared__ uint32_t last;
        __syncthreads();
        if (threadIdx.x == 0)
            last = atom_add_acq_rel(a.seg_done + s, 1u) == si.ncta * a.upw - 1 ? 1u : 0u;
        __syncthreads();
        if (last && threadIdx.x == 0) {
            __threadfence_system();
            for (uint32_t f = 0; f < a.nflag; ++f) st_release_sys(a.sflag[f] + si.slot, a.epoch);
        }
    }
}

// Decode of an fp32 final payload: MODE 0 copy into `out`, MODE 1 Nesterov
// (optim.hpp:116-132) with avg = payload (+ optional theta_l write).
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_f32_apply(ApplyArgs a, const float* pay) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x / a.upw, part = blockIdx.x % a.upw;
    const SegInfo si = a.segs[a.cta_seg[tile]];
    if (a.in_flag) {
        if (threadIdx.x == 0) spin_until_ge_sys(a.in_flag + si.slot, a.epoch, a.err, a.timeout_ns);
        __syncthreads();
    }
    const uint64_t hiel = si.lo + si.len;
    for (int ui = 0; ui < kApplyUnits; ++ui) {
        const uint32_t u = ((tile - si.cta0) * a.upw + part * kApplyUnits + ui) * kWarps + warp;
        if (u >= si.nunits) return;
        const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;
#pragma unroll 4
        for (int j = 0; j < kSlotsPerLane; ++j) {
            const uint64_t q = qbase + (uint64_t)j * 32 + lane;
            const uint64_t e0 = q * 4;
            if (e0 >= hiel) continue;
            const bool full = e0 >= si.lo && e0 + 4 <= hiel;
            const float4 dv = __ldcs(reinterpret_cast<const float4*>(pay) + q);
            const float d[4] = {dv.x, dv.y, dv.z, dv.w};
            if (MODE == 0) {
                if (full) {
                    reinterpret_cast<float4*>(a.out)[q] = dv;
                } else {
                    for (int e = 0; e < 4; ++e)
                        if (e0 + e >= si.lo && e0 + e < hiel) a.out[e0 + e] = d[e];
                }
            } else {
                float4 th = __ldcs(reinterpret_cast<const float4*>(a.theta) + q);
                float4 bb = __ldcs(reinterpret_cast<const float4*>(a.buf) + q);
                float t4[4] = {th.x, th.y, th.z, th.w}, b4[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) nesterov1(t4[e], b4[e], d[e], a.lr, a.mom);
                if (full) {
                    const float4 to = make_float4(t4[0], t4[1], t4[2], t4[3]);
                    __stcs(reinterpret_cast<float4*>(a.theta) + q, to);
                    __stcs(reinterpret_cast<float4*>(a.buf) + q, make_float4(b4[0], b4[1], b4[2], b4[3]));
                    if (a.theta_local) __stcs(reinterpret_cast<float4*>(a.theta_local) + q, to);
                } else {
                    for (int e = 0; e < 4; ++e)
                        if (e0 + e >= si.lo && e0 + e < hiel) {
                            a.theta[e0 + e] = t4[e];
                            a.buf[e0 + e] = b4[e];
                            if (a.theta_local) a.theta_local[e0 + e] = t4[e];
                        }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// AdamW inner step (optim.hpp:63-94), the producer of theta_l: decoupled
// weight decay on p, bias-corrected moments, every fp32 operation rounded in
// the reference's order (no FMA). bc1 / bc2 come from the host (std::pow in
// double, optim.hpp:73-76). A non-finite gradient leaves its element
// untouched and sets err bit 0 (the host raises NumericError, optim.hpp:84-85).
struct AdamWArgs {
    float lr, lrwd, b1, omb1, b2, omb2, bc1, bc2, eps;
};

__device__ __forceinline__ void adamw1(float& p, float g, float& m, float& v, const AdamWArgs& h) {
    p = __fsub_rn(p, __fmul_rn(h.lrwd, p));
    m = __fadd_rn(__fmul_rn(h.b1, m), __fmul_rn(h.omb1, g));
    v = __fadd_rn(__fmul_rn(h.b2, v), __fmul_rn(__fmul_rn(h.omb2, g), g));
    const float mhat = __fdiv_rn(m, h.bc1), vhat = __fdiv_rn(v, h.bc2);
    p = __fsub_rn(p, __fdiv_rn(__fmul_rn(h.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), h.eps)));
}

__global__ void __launch_bounds__(kThreads) k_adamw(float* p, const float* g, float* m, float* v, uint64_t n,
                                                    AdamWArgs h, uint32_t* err) {
    const uint64_t n4 = n / 4, stride = (uint64_t)gridDim.x * blockDim.x;
    bool bad = false;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
        const float4 gv = __ldcs(reinterpret_cast<const float4*>(g) + q);
        float4 pv = __ldcs(reinterpret_cast<const float4*>(p) + q);
        float4 mv = __ldcs(reinterpret_cast<const float4*>(m) + q);
        float4 vv = __ldcs(reinterpret_cast<const float4*>(v) + q);
        float gg[4] = {gv.x, gv.y, gv.z, gv.w}, pp[4] = {pv.x, pv.y, pv.z, pv.w};
        float mm[4] = {mv.x, mv.y, mv.z, mv.w}, vw[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (isfinite(gg[e])) adamw1(pp[e], gg[e], mm[e], vw[e], h);
            else bad = true;
        }
        __stcs(reinterpret_cast<float4*>(p) + q, make_float4(pp[0], pp[1], pp[2], pp[3]));
        __stcs(reinterpret_cast<float4*>(m) + q, make_float4(mm[0], mm[1], mm[2], mm[3]));
        __stcs(reinterpret_cast<float4*>(v) + q, make_float4(vw[0], vw[1], vw[2], vw[3]));
    }
    for (uint64_t i = n4 * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (isfinite(g[i])) adamw1(p[i], g[i], m[i], v[i], h);
        else bad = true;
    }
    if (bad && err) atomicOr(err, 1u);
}

// ---------------------------------------------------------------------------
// Flat elementwise kernels (no segments).

// K1: delta = prev - local (optim.hpp:108), 128-bit loads/stores.
__global__ void __launch_bounds__(kThreads) k_pseudo_gradient(const float* __restrict__ prev,
                                                              const float* __restrict__ local,
                                                              float* __restrict__ delta, uint64_t n) {
    const uint64_t n4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
        const float4 p = __ldcs(reinterpret_cast<const float4*>(prev) + q);
        const float4 l = __ldcs(reinterpret_cast<const float4*>(local) + q);
        __stcs(reinterpret_cast<float4*>(delta) + q,
               make_float4(__fsub_rn(p.x, l.x), __fsub_rn(p.y, l.y), __fsub_rn(p.z, l.z), __fsub_rn(p.w, l.w)));
    }
    for (uint64_t i = n4 * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        delta[i] = __fsub_rn(prev[i], local[i]);
}

// Nesterov from an fp32 average (optim.hpp:116-132). With local != nullptr
// the average is the pseudo-gradient itself (k == 1: ring is the identity,
// allreduce.hpp:319), fused: avg = theta - local.
// local and local_out may alias (theta_l read, then overwritten with theta_g).
__global__ void __launch_bounds__(kThreads) k_nesterov_f32(float* theta, const float* avg, const float* local,
                                                           float* buf, float* local_out, uint64_t n, float lr,
                                                           float mom) {
    const uint64_t n4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
        const float4 th = __ldcs(reinterpret_cast<const float4*>(theta) + q);
        const float4 bb = __ldcs(reinterpret_cast<const float4*>(buf) + q);
        float4 d;
        if (local) {
            const float4 l = __ldcs(reinterpret_cast<const float4*>(local) + q);
            d = make_float4(__fsub_rn(th.x, l.x), __fsub_rn(th.y, l.y), __fsub_rn(th.z, l.z), __fsub_rn(th.w, l.w));
        } else {
            d = __ldcs(reinterpret_cast<const float4*>(avg) + q);
        }
        float t4[4] = {th.x, th.y, th.z, th.w}, b4[4] = {bb.x, bb.y, bb.z, bb.w};
        float d4[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) nesterov1(t4[e], b4[e], d4[e], lr, mom);
        const float4 to = make_float4(t4[0], t4[1], t4[2], t4[3]);
        __stcs(reinterpret_cast<float4*>(theta) + q, to);
        __stcs(reinterpret_cast<float4*>(buf) + q, make_float4(b4[0], b4[1], b4[2], b4[3]));
        if (local_out) __stcs(reinterpret_cast<float4*>(local_out) + q, to);
    }
    for (uint64_t i = n4 * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        float th = theta[i], b = buf[i];
        const float d = local ? __fsub_rn(th, local[i]) : avg[i];
        nesterov1(th, b, d, lr, mom);
        theta[i] = th;
        buf[i] = b;
        if (local_out) local_out[i] = th;
    }
}

}  // namespace emesh_b200
