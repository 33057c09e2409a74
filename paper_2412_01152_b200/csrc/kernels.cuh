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
// segment's work is ncta consecutive tiles of kWarps * upw warp units; a
// warp unit is 256 float4 slots (1024 elements) of the arena's float4 grid.
struct SegInfo {
    uint64_t lo;        // absolute element offset in the arena
    uint64_t len;       // elements
    uint64_t q0;        // lo >> 2: first float4 slot
    uint64_t sq0;       // the segment's first float4 slot in the batch's scratch (whole units)
    uint32_t nunits;    // warp units (1024-element float4-grid spans)
    uint32_t cta0;      // first tile (batch-relative): leaf_stat index
    uint32_t ncta;      // tiles
    uint32_t slot;      // global segment slot (stats / codebook index)
    uint32_t in_slot;   // slot of the incoming payload's codebook (== slot)
    uint32_t upw;       // warp units per tile (1, 2 or 4; one value per batch)
    uint32_t chunk;     // ring chunk of the segment (ChunkMsg header)
    uint32_t pad_;
};
constexpr uint32_t kSyncReady = 32;  // first per-segment word of a launch's sync array

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

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------
// small helpers

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
// Cross-GPU signalling (peer transport): flags live in the receiver's memory.
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// ---- ring failure model of the peer transport (allreduce.hpp:247-305, :341-359)
//
// Arrival flags hold the round (job) number. A rank whose round failed raises
// kPoison | culprit instead of the round number on every flag it still owes,
// so the failure sweeps the ring the way the reference's abort frames do
// (abort_both_ways, allreduce.hpp:341-359): every rank waits on its
// predecessor for every reduce-scatter segment and on every owner's final
// payload, so no rank can complete a round another rank failed. err[0] holds
// sticky bits, err[1] the culprit rank + 1 (first failure wins; 0 = none).
constexpr uint32_t kPoison = 0x80000000u;
constexpr uint32_t kNoCulprit = 0xffu;
constexpr uint32_t kErrNonFinite = 1u;
constexpr uint32_t kErrRingTimeout = 2u;  // RingFailureError: a peer stalled or failed
constexpr uint32_t kErrStale = 4u;        // StalePlanError: a peer runs a newer plan epoch
constexpr uint32_t kErrProto = 8u;        // Error: ring protocol violation (header mismatch)
constexpr uint32_t kErrRing = kErrRingTimeout | kErrStale | kErrProto;

__device__ __forceinline__ void ring_fail(uint32_t* err, uint32_t bits, uint32_t culprit) {
    atomicCAS(err + 1, 0u, (culprit & 0xffu) + 1u);
    atomicOr(err, bits);
}
// The value this rank raises on a flag: the round, or poison naming the culprit.
__device__ __forceinline__ uint32_t raise_value(const uint32_t* err, uint32_t epoch) {
    if (ld_acquire(err) & kErrRing) {
        const uint32_t c = ld_acquire(err + 1);
        return kPoison | (c ? (c - 1u) & 0xffu : kNoCulprit);
    }
    return epoch;
}
// Waits for a peer's arrival flag. A peer that stops (crash, abort) must not
// hang the GPU: after timeout_ns (ReduceOptions::step_timeout,
// allreduce.hpp:59) the wait gives up naming `culprit` (the rank that owes
// the flag: the predecessor for reduce-scatter payloads, the owner for final
// ones); a poisoned flag fails at once with the culprit it carries; once
// this rank failed, every other wait gives up at once. Returns true when the
// flag arrived for this round.
//
// Attribution past k = 2 (reduce-scatter waits, wait_self / wait_pred set):
// a waiter publishes the round it waits in (its "waiting" word, mapped by its
// successor). When the budget expires and the predecessor is itself waiting
// in this round, the predecessor is blocked on a rank further up, not dead:
// the waiter grants it one more budget for its poisoned flag (which names
// the real culprit) before blaming it. A dead or stalled predecessor is not
// waiting in this round and is named at once.
__device__ __forceinline__ bool spin_until_ge_sys(const uint32_t* p, uint32_t epoch, uint32_t* err,
                                                  unsigned long long timeout_ns, uint32_t culprit,
                                                  uint32_t* wait_self = nullptr,
                                                  const uint32_t* wait_pred = nullptr) {
    uint32_t ns = 64;
    unsigned long long t0 = gtimer();
    bool extended = false;
    if (wait_self) *reinterpret_cast<volatile uint32_t*>(wait_self) = epoch;
    for (;;) {
        const uint32_t v = ld_acquire_sys(p);
        if (v & kPoison) {
            ring_fail(err, kErrRingTimeout, v & 0xffu);
            return false;
        }
        if ((int32_t)(v - epoch) >= 0) return true;
        if (ld_acquire(err) & kErrRing) return false;
        if (gtimer() - t0 > timeout_ns) {
            if (wait_pred && !extended && *reinterpret_cast<const volatile uint32_t*>(wait_pred) == epoch) {
                extended = true;  // the predecessor is blocked too: wait for its verdict
                t0 = gtimer();
                continue;
            }
            ring_fail(err, kErrRingTimeout, culprit);
            return false;
        }
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : ns;  // short cap: a hop's flag latency is on the small-round critical path
    }
}
constexpr uint32_t kSyncExit = 1;   // sync[] word counting the quantizer CTAs that ran out of tasks
constexpr uint32_t kWaitSlot = 63;  // the "waiting" word's index in each rank's mapped done[] array

// ChunkMsg header (allreduce.hpp:66-103) of one segment payload in a peer
// arena, written by the producer before it raises the segment's flag and
// validated by the consumer after (AttemptRx::expect, allreduce.hpp:252-283):
// a newer plan epoch -> StalePlanError; another job, phase, chunk, mode or
// element count (the wire format's u32 count, quant.hpp:102-109) -> ring
// protocol violation.
struct ChunkHdr {
    unsigned long long job;  // ReduceJob id
    uint32_t epoch;          // plan epoch
    uint32_t chunk;          // ring chunk the segment belongs to
    uint32_t count;          // elements of the segment
    uint8_t phase, mode;     // Phase (0 reduce_scatter, 1 all_gather), ReduceMode (0 fp32, 1 int8)
    uint16_t pad;
};
enum : uint8_t { kPhaseRS = 0, kPhaseAG = 1 };
struct HdrRef {  // what a consumer expects
    unsigned long long job;
    uint32_t epoch;
    uint8_t mode;
};
// Validates the header a flag published (the caller acquired the flag).
__device__ __forceinline__ bool check_hdr(const ChunkHdr* h, const HdrRef& want, uint32_t chunk, uint32_t count,
                                          uint8_t phase, uint32_t* err, uint32_t culprit) {
    const unsigned long long job = __ldcg(&h->job);
    const uint32_t epoch = __ldcg(&h->epoch), ch = __ldcg(&h->chunk), cnt = __ldcg(&h->count);
    const uint32_t pm = __ldcg(reinterpret_cast<const uint32_t*>(&h->phase));
    if (epoch > want.epoch) {
        ring_fail(err, kErrStale, culprit);
        return false;
    }
    if (epoch != want.epoch || job != want.job || ch != chunk || cnt != count || (pm & 0xffu) != phase ||
        ((pm >> 8) & 0xffu) != want.mode) {
        ring_fail(err, kErrProto, culprit);
        return false;
    }
    return true;
}
__device__ __forceinline__ void write_hdr(ChunkHdr* h, const HdrRef& me, uint32_t chunk, uint32_t count,
                                          uint8_t phase) {
    h->job = me.job;
    h->epoch = me.epoch;
    h->chunk = chunk;
    h->count = count;
    *reinterpret_cast<uint32_t*>(&h->phase) = (uint32_t)phase | ((uint32_t)me.mode << 8);
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

// Exact bucket by the threshold table (the rare path of the fp32 estimate).
__device__ __noinline__ int bucket_walk(float x, int c, const float* thr) {
    while (c < 255 && x >= thr[c + 1]) ++c;
    while (c > 0 && x < thr[c]) --c;
    return c;
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
    // atomic commit (peer / NCCL transports): the round's gate word; every CTA
    // writes only when it holds `epoch` (k_round_gate: every final payload of
    // the round arrived intact), so a failed round leaves theta / momentum
    // untouched and allreduce_with_retry can restart from them
    const volatile uint32_t* gate;
    uint32_t epoch;
    // k_apply<1>: the workers whose replicas decode this payload (several on one GPU: the virtual
    // ring decodes each final payload once for all of them); [0] = theta / buf / theta_local
    uint32_t nw;
    float* thetas[kMaxDest];
    float* bufs[kMaxDest];
    float* locals[kMaxDest];
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
    if (a.gate && *a.gate != a.epoch) return;  // the round failed somewhere: commit nothing
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
        } else if (MODE == 1) {  // one replica
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
        } else {  // MODE 2: several local replicas of one payload (virtual ring)
            // every replica's loads first (independent streams in flight), then the updates
            constexpr int kW = 4;  // replicas handled per pass
            for (uint32_t w0 = 0; w0 < a.nw; w0 += kW) {
            float4 thv[kW], bbv[kW];
#pragma unroll
            for (int i = 0; i < kW; ++i)
                if (w0 + i < a.nw) {
                    thv[i] = __ldcs(reinterpret_cast<const float4*>(a.thetas[w0 + i]) + q);
                    bbv[i] = __ldcs(reinterpret_cast<const float4*>(a.bufs[w0 + i]) + q);
                }
#pragma unroll
            for (int i = 0; i < kW; ++i) {
                if (w0 + i >= a.nw) break;
                float* const theta = a.thetas[w0 + i];
                float* const buf = a.bufs[w0 + i];
                float* const tloc = a.locals[w0 + i];
                const float4 th = thv[i], bb = bbv[i];
                float t4[4] = {th.x, th.y, th.z, th.w}, b4[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) nesterov1(t4[e], b4[e], d[e], a.lr, a.mom);
                if (full) {
                    const float4 to = make_float4(t4[0], t4[1], t4[2], t4[3]);
                    __stcs(reinterpret_cast<float4*>(theta) + q, to);
                    __stcs(reinterpret_cast<float4*>(buf) + q, make_float4(b4[0], b4[1], b4[2], b4[3]));
                    if (tloc) __stcs(reinterpret_cast<float4*>(tloc) + q, to);
                } else {
                    for (int e = 0; e < 4; ++e)
                        if (e0 + e >= si.lo && e0 + e < hiel) {
                            theta[e0 + e] = t4[e];
                            buf[e0 + e] = b4[e];
                            if (tloc) tloc[e0 + e] = t4[e];
                        }
                }
            }
            }
        }
    }
    }
}

// ---------------------------------------------------------------------------
// Round commit (peer transport). Each owner's final quantizer stores its
// payload into every rank (ag_flag per segment) and then, from its last CTA,
// a "done" word into every rank's done[q]: the round number, or poison
// naming a culprit when q's round failed. k_round_gate (one small
// CTA, after this rank's last quantizer) waits for every other owner's done
// word, validates the final payloads' ChunkMsg headers and then publishes
// the gate word the decode kernels check: the round number to commit, 0 to
// leave theta / momentum untouched (the reference applies Nesterov only to
// a completed all-reduce, trainer.hpp:375-381).
struct GateArgs {
    const uint32_t* done;  // [k] owner q's done word (this rank's memory)
    uint32_t* gate;        // this rank's gate word
    uint32_t* err;
    const ChunkHdr* hdr;   // final-payload headers by slot (this rank's arena)
    const uint2* meta;     // by slot: {ring chunk, elements}
    const uint32_t* ag_flag;  // by slot, when the owners' quantizers stored the final payloads themselves
    HdrRef want;
    uint32_t k, rank, own_chunk, nslots, epoch;
    unsigned long long timeout_ns;
};
__global__ void __launch_bounds__(kThreads) k_round_gate(GateArgs a) {
    const uint32_t t = threadIdx.x;
    if (t < 32 && t < a.k && t != a.rank) spin_until_ge_sys(a.done + t, a.epoch, a.err, a.timeout_ns, t);
    __syncthreads();
    if (a.hdr && !(ld_acquire(a.err) & kErrRing)) {
        for (uint32_t s = t; s < a.nslots; s += blockDim.x) {
            const uint2 m = a.meta[s];
            if (m.x == a.own_chunk || m.y == 0) continue;
            const uint32_t owner = (m.x + a.k - 1) % a.k;
            // the owner's quantizer stored this payload itself: its per-segment flag (system-scope
            // release after the stores) makes the bytes visible here
            if (a.ag_flag && !spin_until_ge_sys(a.ag_flag + s, a.epoch, a.err, a.timeout_ns, owner)) continue;
            check_hdr(a.hdr + s, a.want, m.x, m.y, kPhaseAG, a.err, owner);
        }
    }
    __syncthreads();
    if (t == 0) *a.gate = (ld_acquire(a.err) & kErrRing) ? 0u : a.epoch;
}
// The word this rank, as an owner, sends to every peer after its final payload.
__global__ void k_done_value(const uint32_t* err, uint32_t epoch, uint32_t* out) {
    if (threadIdx.x == 0) *out = raise_value(err, epoch);
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
    uint32_t ndest_fail;       // destinations still written once this rank's round failed (QuantArgs)
    uint32_t* sflag[kMaxDest];  // peer arrival flags raised per finished segment
    uint32_t nflag;
    uint32_t* seg_done;        // [batch segment] CTA arrival counters (zeroed per launch)
    const uint32_t* in_flag;   // peer transport: wait in_flag[slot] >= epoch before reading `in`
    uint32_t epoch;
    uint32_t nseg;
    uint32_t* err;
    unsigned long long timeout_ns;
    // ChunkMsg headers (peer transport): written next to every payload, checked on receipt
    ChunkHdr* dhdr[kMaxDest];
    const ChunkHdr* in_hdr;
    HdrRef hdr;
    uint8_t phase_out;
    uint32_t culprit_in;       // rank that owes the incoming payload (the predecessor)
    uint32_t* wait_self;       // this rank's / the predecessor's "waiting" words (spin_until_ge_sys)
    const uint32_t* wait_pred;
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
        if (threadIdx.x == 0 &&
            spin_until_ge_sys(a.in_flag + si.in_slot, a.epoch, a.err, a.timeout_ns, a.culprit_in, a.wait_self,
                              a.wait_pred) &&
            a.in_hdr)
            check_hdr(a.in_hdr + si.in_slot, a.hdr, si.chunk, (uint32_t)si.len, kPhaseRS, a.err, a.culprit_in);
        __syncthreads();
    }
    const uint64_t hiel = si.lo + si.len;
    const uint32_t nd = (ld_acquire(a.err) & kErrRing) ? a.ndest_fail : a.ndest;
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
            for (uint32_t d = 0; d < nd; ++d) {
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
            const uint32_t ndh = (ld_acquire(a.err) & kErrRing) ? a.ndest_fail : a.ndest;
            for (uint32_t d = 0; d < ndh; ++d)
                if (a.dhdr[d]) write_hdr(a.dhdr[d] + si.slot, a.hdr, si.chunk, (uint32_t)si.len, a.phase_out);
            __threadfence_system();
            const uint32_t v = raise_value(a.err, a.epoch);
            for (uint32_t f = 0; f < a.nflag; ++f) st_release_sys(a.sflag[f] + si.slot, v);
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
    if (a.gate && *a.gate != a.epoch) return;  // the round failed somewhere: commit nothing
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
