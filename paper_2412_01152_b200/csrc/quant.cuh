// Persistent two-pass quantizer (k_quant): the reference's quantize
// (proj/include/emesh/quant.hpp:28-87) over every segment of one ring batch,
// with its producer fused in (pseudo-gradient optim.hpp:108, ring hop add
// allreduce.hpp:422, owner mean :435-439). STATS tiles compute the value x
// and its moments and park x in a per-batch scratch; once a segment's
// statistics are published, BIN tiles re-read x and assign codes + exact
// bucket sums. See DESIGN.md §3 for the numerics and §7 for the on-chip
// (tensor-memory) variants measured in round 2.
#pragma once

#include "kernels.cuh"

namespace emesh_b200 {

constexpr int kQuantMinBlocks = 3;  // co-resident quantizer CTAs per SM (80 registers)
constexpr int kUnitsPerWarp = 6;    // warp units per tile task (large batches; SegInfo::upw):
                                    // 6 vs 4 measured -1.5 % per launch (fewer per-tile tables,
                                    // barriers and accumulator atomics)
// Bin-pass limbs (32-bit smem atomics per warp over one tile, see bin_unit):
// A = r[0:kLoBits) | 1 << kCntShift, B = r[kLoBits:kMidEnd), C = r[kMidEnd:42).
// With m = 1024 kUnitsPerWarp members: m (2^kLoBits - 1) < 2^kCntShift,
// m < 2^(32 - kCntShift), m 2^(kMidEnd - kLoBits) <= 2^32, m 2^(42 - kMidEnd) < 2^32.
constexpr int kLoBits = 6;
constexpr int kCntShift = 19;
constexpr int kMidEnd = 25;
static_assert(1024LL * kUnitsPerWarp * ((1LL << kLoBits) - 1) < (1LL << kCntShift), "A limb");
static_assert(1024LL * kUnitsPerWarp < (1LL << (32 - kCntShift)), "count");
static_assert(1024LL * kUnitsPerWarp * (1LL << (kMidEnd - kLoBits)) <= (1LL << 32), "B limb");
static_assert(1024LL * kUnitsPerWarp * (1LL << (42 - kMidEnd)) < (1LL << 32), "C limb");
// The tile shape (kWarps * upw units: 48K, 16K or 8K elements) is chosen per
// batch at run time (SegInfo::upw, Plan::add_batch): the limb layout above is
// sized for the largest tile and stays exact for a smaller one (its bounds cap m).

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
    uint32_t ndest_fail;       // destinations still written once this rank's round failed: a failed
                               // owner must not overwrite the peers' arenas with a garbage final payload
                               // (a late peer may still read its reduce-scatter input from those slots)
    uint32_t* sflag[kMaxDest];
    uint32_t nflag;
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
    // peer transport: ChunkMsg headers written next to every payload / checked on receipt
    ChunkHdr* dhdr[kMaxDest];
    const ChunkHdr* in_hdr;
    HdrRef hdr;
    uint32_t phase_out;        // kPhaseRS, or kPhaseAG for the owner's final payload
    uint32_t culprit_in;       // rank that owes the incoming payloads (the predecessor)
    uint32_t* wait_self;       // this rank's / the predecessor's "waiting" words (spin_until_ge_sys)
    const uint32_t* wait_pred;
    // the owner's final quantizer: once every CTA is done, the last one stores this rank's done
    // value (the round, or poison naming the culprit) into every peer's done word (p2p_commit)
    uint32_t* done_dst[kMaxDest];
    uint32_t ndone;
};



// Streaming (read-once) loads: no L1 allocation, leaving L1 to the BIN
// pass's scratch prefetch.
__device__ __forceinline__ float4 ld4_stream(const float* p, uint64_t q) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(reinterpret_cast<const float4*>(p) + q));
    return v;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) { return __ldcs(p); }
__device__ __forceinline__ float4 ld4(const float* p, uint64_t q) {
    return __ldg(reinterpret_cast<const float4*>(p) + q);
}

// ---------------------------------------------------------------------------
// Persistent quantizer: one launch per batch (pipelining window), a grid of
// co-resident CTAs that claim tile tasks in plan order (one atomicAdd each).

struct __align__(16) QSmem {
    uint32_t hist[kWarps][kBuckets + 1][3];  // per-warp limbs over the tile (bin), see bin_unit; row 256: sink
    uint32_t binfo[kBuckets];            // bucket encodings (bin, see kInfoWide): one 32-bit lookup per
                                         // element (a 64/128-bit table measured slower: more smem wavefronts)
    float lut[kBuckets];                 // incoming codebook (stats, hop)
    float thr[kBuckets + 2];             // exact threshold table (bin); [257] = bucket 0's base (lo_up)
    StatP wp[kWarps];
    double red[2];
    uint32_t clip[2];
    uint32_t flag;
    uint32_t task;
    int32_t bin_seg, lut_seg, ready_seg;
    uint32_t run_idx;
    uint32_t cnt_one;  // 1 << kCntShift, read back from smem (an opaque register for lop3_and_or)
    uint32_t nd;       // destinations this BIN tile writes (QuantArgs::ndest_fail)
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
enum : uint32_t { kTaskStats = 0, kTaskBin = 2 };
// mixed run (alternating STATS / BIN tasks): y = kTaskMix{Rev,Fwd} | bin segment << 2,
// z = STATS segment, w = first STATS tile | first BIN tile << 16
constexpr uint32_t kTaskMixRev = 1, kTaskMixFwd = 3;
constexpr uint32_t kMaxRunsSmem = 256;  // run table cached in smem when it fits (4 KB)
constexpr uint32_t kMaxSegsSmem = 128;  // SegInfo cached in smem when it fits



__device__ void finalize_stats(const QuantArgs& a, QSmem& sm, uint32_t s, const SegInfo& si);

// Where BIN gets x: the STATS pass's scratch, the input itself (plain
// quantize), or theta_g - theta_l recomputed (the PG payload: the same 8
// bytes of DRAM reads as the scratch round trip, without its 4-byte write)
// (the hops' x = (theta_g - theta_l) + cb_in[code] recomputed in BIN was 12-25 % slower than the scratch:
// one more byte per element and a second lookup table)
enum : int { kBinScratch = 0, kBinA = 1, kBinRecompute = 2 };
template <int SRC> constexpr int kBinSource = SRC == kSrcA ? kBinA : SRC == kSrcAminusB ? kBinRecompute : kBinScratch;
template <int SRC> constexpr bool kStatsWritesScratch = kBinSource<SRC> == kBinScratch;

// Scratch x (written by STATS, read once by BIN, then discarded).
__device__ __forceinline__ void st_scratch(float4* p, float4 v) { *p = v; }

template <int SRC>
__device__ __forceinline__ void stats_tile(const QuantArgs& a, QSmem& sm, uint32_t s, const SegInfo& si,
                                           uint32_t tile) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t hiel = si.lo + si.len;     // exclusive
    float4* xs = reinterpret_cast<float4*>(a.scratch) + ((int64_t)si.sq0 - (int64_t)si.q0);

    if (SRC & kHasIn) {
        if (sm.lut_seg != (int32_t)s) {
            __syncthreads();
            if (a.in_flag) {  // peer transport: the predecessor's payload of s must have landed intact
                if (threadIdx.x == 0 &&
                    spin_until_ge_sys(a.in_flag + si.in_slot, a.epoch, a.err, a.timeout_ns, a.culprit_in,
                                      a.wait_self, a.wait_pred) &&
                    a.in_hdr)
                    check_hdr(a.in_hdr + si.in_slot, a.hdr, si.chunk, (uint32_t)si.len, kPhaseRS, a.err,
                              a.culprit_in);
                __syncthreads();
            }
            sm.lut[threadIdx.x] = __ldcg(a.in_cb + (uint64_t)si.in_slot * kBuckets + threadIdx.x);
            __syncthreads();
            if (threadIdx.x == 0) sm.lut_seg = (int32_t)s;
        }
    }
    StatP p{0.0, 0.0, 0.0, 0.0, 0};
    double sum0 = 0.0, sum1 = 0.0, q0 = 0.0, q1 = 0.0;
    double piv = 0.0;
    uint32_t cnt = 0;
    bool have_piv = false;
    for (int ui = 0; ui < (int)si.upw; ++ui) {
        const uint32_t u = (tile * si.upw + ui) * kWarps + warp;  // segment-relative unit
        if (u >= si.nunits) break;
        const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;
        const bool interior = qbase * 4 >= si.lo && (qbase + kUnitSlots) * 4 <= hiel;  // warp-uniform
        constexpr int kHalf = kSlotsPerLane / 2;
#pragma unroll 1  // a smaller kernel (fewer instruction-cache misses): -1.4 % per launch
        for (int h = 0; h < 2; ++h) {
            float4 xa[kHalf], xb[kHalf];
            uint32_t c4[kHalf];
#pragma unroll
            for (int jj = 0; jj < kHalf; ++jj) {
                const uint64_t q = qbase + (uint64_t)(h * kHalf + jj) * 32 + lane;
                const bool in = interior || q * 4 < hiel;
                xa[jj] = in ? ld4_stream(a.a, q) : make_float4(0.f, 0.f, 0.f, 0.f);
                if (SRC & kSrcAminusB) xb[jj] = in ? ld4_stream(a.b, q) : make_float4(0.f, 0.f, 0.f, 0.f);
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
                    // sigma is not bit-exact vs the sequential reference anyway:
                    // fused multiply-adds for the squares
                    q0 = __fma_rn(v2, v2, __fma_rn(v0, v0, q0));
                    q1 = __fma_rn(v3, v3, __fma_rn(v1, v1, q1));
                    if (kStatsWritesScratch<SRC>) st_scratch(xs + q, make_float4(x[0], x[1], x[2], x[3]));
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
                            q0 = __fma_rn(dv, dv, q0);
                            cnt += 1;
                            if (kStatsWritesScratch<SRC>) reinterpret_cast<float*>(xs + q)[e] = x[e];
                        }
                    }
                }
            }
        }
        if (interior) cnt += kSlotsPerLane * 4;  // per lane
    }
    // D = sum (x - p) of the lane, as sum x - n p (sigma's pivot correction, see finalize_stats;
    // sigma is not reproduced bit-for-bit either way)
    const double sx = __dadd_rn(sum0, sum1);
    p = StatP{sx, __dadd_rn(q0, q1), __dsub_rn(sx, __dmul_rn((double)cnt, piv)), piv, (uint64_t)cnt};
    p = warp_merge(p);
    if (lane == 0) {
        sm.wp[warp] = p;
        // finite fp32 inputs cannot overflow an fp64 sum: one check per unit
        if (!isfinite(p.s) || !isfinite(p.m2)) {
            atomicOr(&a.seg_flags[s], kFlagNonFinite);
            atomicOr(a.err, kErrNonFinite);
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



struct BinParams {
    float c, inv_w, lo_up, hi_dn, margin, one_m;  // bucket estimate g = fma(x, inv_w, -c)
    uint32_t cnt_one;                              // 1 << kCntShift, in a register (see lop3_and_or)
};
// (a & b) | c in one LOP3: c comes from a register, so ptxas cannot split the
// two immediates into two instructions.
template <uint32_t B>
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(B), "r"(c));
    return d;
}

// One warp unit of the bin pass (1024 elements; this lane's 32), in groups of
// 8: bucket estimates for all 8, rare fix-ups (exact table near an edge,
// clipping), fixed-point codes via the fp32 fast path (fp64 for the few
// buckets that need it), then the limb atomics — unconditional, so the
// common path has no data-dependent branches (invalid lanes add 0).
// Per-warp limbs over a tile (see kLoBits): A += low bits | one count,
// B += middle bits, C += high bits (only when nonzero: rare).
// BIN's scratch reads. The warp prefetches its
// next unit's 4 KB of scratch into L1 while it bins the current one, and the
// loads go through L1. Each scratch line belongs to exactly one segment
// (segments own whole units of scratch, Plan::add_batch), is written once by
// its STATS tiles before the segment's statistics are published, and only
// read (or prefetched) after: no stale L1 copy can exist within the launch.
__device__ __forceinline__ float4 ld_scratch(const float4* p) { return *p; }

template <bool INTERIOR, int BSRC, int SRC>
__device__ __forceinline__ void bin_unit(const QuantArgs& a, QSmem& sm, const SegInfo& si, uint64_t qbase,
                                         uint64_t hiel, const float4* xs, uint32_t* hw, const BinParams& p,
                                         uint32_t nd, uint32_t& nclip_lo, uint32_t& nclip_hi) {
    const int lane = threadIdx.x & 31;
    constexpr int kHalf = kSlotsPerLane / 2;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        float4 xv[kHalf];
#pragma unroll
        for (int jj = 0; jj < kHalf; ++jj) {
            const uint64_t q = qbase + (uint64_t)(h * kHalf + jj) * 32 + lane;
            const bool in = INTERIOR || q * 4 < hiel;
            if (!in) {
                xv[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
            } else if (BSRC == kBinScratch) {
                xv[jj] = ld_scratch(xs + q);
            } else if (BSRC == kBinA) {
                xv[jj] = ld4(a.a, q);
            } else {  // kBinRecompute (PG payload): x = theta_g - theta_l again, STATS' rounding
                static_assert(BSRC != kBinRecompute || SRC == kSrcAminusB, "BIN recomputes only the PG payload");
                const float4 u = ld4_stream(a.a, q), w = ld4_stream(a.b, q);
                xv[jj] = make_float4(__fsub_rn(u.x, w.x), __fsub_rn(u.y, w.y), __fsub_rn(u.z, w.z), __fsub_rn(u.w, w.w));
            }
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
                const uint32_t info = sm.binfo[cc[i] & 0xff];  // sink members: their bucket's entry
                // m = x * s + K in [2^52, 2^53): mantissa = r (see kInfoWide); s = the entry's
                // high word, K = 2^52 (+ 2^41 for the wide bucket)
                const double sc = __hiloint2double((int)(info & ~kInfoWide), 0);
                const double kk = __hiloint2double((int)(0x43300000u | ((info & kInfoWide) << 9)), 0);
                const double m = __fma_rn((double)xe[i], sc, kk);
                const uint32_t rlo = (uint32_t)__double2loint(m);
                const uint32_t rhi = (uint32_t)__double2hiint(m);
                uint32_t* hc = hw + 3 * min(cc[i], kBuckets);
                red_shared_add(hc, lop3_and_or<(1u << kLoBits) - 1u>(rlo, p.cnt_one));
                red_shared_add(hc + 1, (rlo >> kLoBits) & ((1u << (kMidEnd - kLoBits)) - 1u));
                const uint32_t rc = __funnelshift_r(rlo, rhi, kMidEnd) & ((1u << (42 - kMidEnd)) - 1u);
                if (rc) red_shared_add(hc + 2, rc);  // nonzero mostly in the wide bucket (an unconditional
                                                     // third atomic measured 1.3 % slower)
            }
            const uint32_t p0 = __byte_perm(__byte_perm(cc[0], cc[1], 0x0040), __byte_perm(cc[2], cc[3], 0x0040), 0x5410);
            const uint32_t p1 = __byte_perm(__byte_perm(cc[4], cc[5], 0x0040), __byte_perm(cc[6], cc[7], 0x0040), 0x5410);
            for (uint32_t d = 0; d < nd; ++d) {
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
    }
}

__device__ void finalize_codebook(const QuantArgs& a, uint32_t s, const SegInfo& si);
__device__ float codebook_entry(const SegStat* st, int b, unsigned long long rl, unsigned long long rh,
                                unsigned long long total, unsigned long long clip);

template <int BSRC, int SRC>
__device__ __forceinline__ void bin_tile(const QuantArgs& a, QSmem& sm, uint32_t s, const SegInfo& si, uint32_t tile) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const SegStat* st = &a.stats[si.slot];
    if (BSRC == kBinScratch) {  // the warp's first unit, while the tables load (the segment's scratch is complete)
        const uint32_t u0 = tile * si.upw * kWarps + warp;
        if (u0 < si.nunits) {
            const float4* p0 = reinterpret_cast<const float4*>(a.scratch) + si.sq0 + (uint64_t)u0 * kUnitSlots + lane * 8;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(p0));
        }
    }
    if (sm.bin_seg != (int32_t)s) {
        __syncthreads();
        const int b = threadIdx.x;
        sm.thr[b] = b == 0 ? -INFINITY : __ldcg(&st->thr[b]);
        const uint32_t info = __ldcg(&st->binfo[b]);
        sm.binfo[b] = info;

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
    if (threadIdx.x == 0) sm.nd = (ld_acquire(a.err) & kErrRing) ? a.ndest_fail : a.ndest;
    __syncthreads();
    const uint32_t nd = sm.nd;

    const uint64_t hiel = si.lo + si.len;
    const float4* xs = reinterpret_cast<const float4*>(a.scratch) + ((int64_t)si.sq0 - (int64_t)si.q0);
    uint32_t nclip_lo = 0, nclip_hi = 0;
    const BinParams bpar{c_f, inv_w, lo_up, hi_dn, margin, one_m, sm.cnt_one};
    for (int ui = 0; ui < (int)si.upw; ++ui) {
        const uint32_t u = (tile * si.upw + ui) * kWarps + warp;
        if (u >= si.nunits) break;
        const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;
        const bool interior = qbase * 4 >= si.lo && (qbase + kUnitSlots) * 4 <= hiel;  // warp-uniform
        if (BSRC == kBinScratch && ui + 1 < (int)si.upw && u + kWarps < si.nunits) {
            const float4* nx = xs + qbase + (uint64_t)kWarps * kUnitSlots + lane * 8;  // one 128-B line per lane
            asm volatile("prefetch.global.L1 [%0];" ::"l"(nx));
        }
        if (degenerate) {  // sigma == 0: every code is 0 (quant.hpp:49-55)
            for (int j = 0; j < kSlotsPerLane; ++j) {
                const uint64_t q = qbase + (uint64_t)j * 32 + lane;
                for (int e = 0; e < 4; ++e)
                    if (q * 4 + e >= si.lo && q * 4 + e < hiel)
                        for (uint32_t d = 0; d < nd; ++d) a.dcodes[d][q * 4 + e] = 0;
            }
        } else if (interior) {
            bin_unit<true, BSRC, SRC>(a, sm, si, qbase, hiel, xs, hw, bpar, nd, nclip_lo, nclip_hi);
        } else {
            bin_unit<false, BSRC, SRC>(a, sm, si, qbase, hiel, xs, hw, bpar, nd, nclip_lo, nclip_hi);
        }
    }
    nclip_lo = warp_sum_u(nclip_lo);
    nclip_hi = warp_sum_u(nclip_hi);
    if (lane == 0 && (nclip_lo | nclip_hi)) {
        atomicAdd(&sm.clip[0], nclip_lo);
        atomicAdd(&sm.clip[1], nclip_hi);
    }
    __syncthreads();
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
    const uint32_t nd = (ld_acquire(a.err) & kErrRing) ? a.ndest_fail : a.ndest;
    for (uint32_t d = 0; d < nd; ++d) a.dcb[d][(uint64_t)si.slot * kBuckets + b] = v;
    if (threadIdx.x == 0)  // the ChunkMsg header of this payload, before its flag
        for (uint32_t d = 0; d < nd; ++d)
            if (a.dhdr[d]) write_hdr(a.dhdr[d] + si.slot, a.hdr, si.chunk, (uint32_t)si.len, (uint8_t)a.phase_out);
    if (a.nflag) {
        // Every tile of s released its stores (gpu scope) to the arrival
        // counter this CTA acquired; the system-scope fence + release here
        // extends that causality chain to the peers polling the flags.
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            const uint32_t v = raise_value(a.err, a.epoch);  // poison when this rank's round failed
            for (uint32_t f = 0; f < a.nflag; ++f) st_release_sys(a.sflag[f] + si.slot, v);
        }
    }
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
__global__ void __launch_bounds__(kThreads, kQuantMinBlocks) k_quant(QuantArgs a) {
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
        sm.cnt_one = 1u << kCntShift;
        sm.bin_seg = -1;
        sm.lut_seg = -1;
        sm.ready_seg = -1;
        nxt = atomicAdd(&a.sync[0], 1u);
    }
    for (;;) {
        if (threadIdx.x == 0) sm.task = nxt;
        __syncthreads();
        const uint32_t t = sm.task;
        if (t >= a.ntasks) {
            if (a.ndone && threadIdx.x == 0 &&
                atom_add_acq_rel(&a.sync[kSyncExit], 1u) == gridDim.x - 1) {  // the last CTA out
                __threadfence_system();
                const uint32_t v = raise_value(a.err, a.epoch);
                for (uint32_t d = 0; d < a.ndone; ++d) st_release_sys(a.done_dst[d], v);
            }
            return;
        }
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
        if (kind == kTaskBin && threadIdx.x == 0 && sm.ready_seg != (int32_t)s) {
            // acquire SegStat(s) (cached per CTA); the CTA owes nothing here
            uint32_t ns = 32;
            while (ld_acquire(&a.sync[kSyncReady + s]) == 0u) {
                __nanosleep(ns);
                ns = ns < 128 ? 2 * ns : ns;
            }
            sm.ready_seg = (int32_t)s;
        }
        __syncthreads();  // everyone has read sm.task; SegStat(s) visible for BIN
        switch (kind) {
            case kTaskStats: stats_tile<SRC>(a, sm, s, si, tile); break;
            default: bin_tile<kBinSource<SRC>, SRC>(a, sm, s, si, tile); break;
        }
    }
}

constexpr size_t kQuantSmemBytes = sizeof(QSmem) + kMaxRunsSmem * sizeof(uint4) + kMaxSegsSmem * sizeof(SegInfo);

}  // namespace emesh_b200
