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

#include <cstdint>
#include <cuda_runtime.h>
#include <math.h>

namespace emesh_b200 {

constexpr int kBuckets = 256;
constexpr int kWarps = 8;              // warps per CTA
constexpr int kThreads = kWarps * 32;  // 256
constexpr int kSlotsPerLane = 8;       // float4 slots per lane per unit
constexpr int kUnitSlots = 32 * kSlotsPerLane;  // 256 float4 = 1024 elements

// Per-segment statistics, written once by the finalizing warp of k_stats.
struct SegStat {
    double mu, sigma, lo, width, hi;  // first four exported as {mu, sigma, lo, width}
    float lo_f, inv_w_f;
    uint32_t flags;  // kFlagNonFinite | kFlagDegenerate
    uint32_t pad;
    float thr[kBuckets];  // thr[j] = smallest fp32 x with code(x) >= j (j=1..255)
};
constexpr uint32_t kFlagNonFinite = 1u;
constexpr uint32_t kFlagDegenerate = 2u;  // sigma == 0 (quant.hpp:49-55)


// One segment of a batch (host-built, device-resident). CTA-aligned: the
// segment's work is ncta consecutive CTAs ("tiles") of 8 warp units each.
struct SegInfo {
    uint64_t lo;        // absolute element offset in the arena
    uint64_t len;       // elements
    uint64_t q0;        // lo >> 2: first float4 slot
    uint32_t nunits;    // warp units (1024-element float4-grid spans)
    uint32_t cta0;      // first CTA (batch-relative)
    uint32_t ncta;      // tiles = leaves of the combine tree
    uint32_t slot;      // global segment slot (stats / codebook index)
    uint32_t in_slot;   // slot of the incoming payload's codebook (== slot)
    uint32_t node_base; // internal tree nodes + counters of this segment
};

// Moments of a set of values around a pivot p: s = sum x, m2 = sum (x-p)^2,
// d = sum (x-p). Two partials merge exactly (in real arithmetic) by moving
// one to the other's pivot, so the combine tree can run in any shape; it
// runs in a fixed order, so results are deterministic.
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

// Producer of the value being quantized, fused into the statistics pass.
enum : int {
    kSrcA = 0,          // x = a                      (plain buffer)
    kSrcAminusB = 1,    // x = a - b                  (pseudo-gradient, optim.hpp:108)
    kHasIn = 2,         // x += cb_in[code_in]        (ring hop add, allreduce.hpp:422)
    kDivK = 4,          // x = x / k                  (owner mean, allreduce.hpp:439)
};

constexpr int kFan = 16;  // combine-tree fan-in

struct QuantArgs {
    const SegInfo* segs;
    const uint32_t* cta_seg;   // CTA -> batch-local segment
    uint32_t ncta;
    uint32_t nseg;
    uint64_t scratch_q0;       // first float4 slot covered by scratch
    const float* a;
    const float* b;
    const uint8_t* in_codes;
    const float* in_cb;
    float divisor;
    float* scratch;            // x, float4-slot indexed from scratch_q0
    uint8_t* out_codes;
    float* out_cb;
    SegStat* stats;            // indexed by slot
    StatP* leaf_stat;          // [cta]
    StatP* node_stat;          // [node]
    double* leaf_sum;          // [cta][256]
    uint32_t* leaf_cnt;        // [cta][256]
    double* node_sum;          // [node][256]
    uint32_t* node_cnt;        // [node][256]
    uint32_t* tree_cnt;        // [2][node]: k_stats, k_bin arrival counters
    uint32_t nnodes;
    uint32_t* seg_flags;       // [seg] non-finite bits (reset by the stats root)
    uint32_t* err;             // sticky error word (bit 0: non-finite)
};

// ---------------------------------------------------------------------------
// small helpers

__device__ __forceinline__ float4 ld4_stream(const float* p, uint64_t q) {
    return __ldcs(reinterpret_cast<const float4*>(p) + q);
}
__device__ __forceinline__ float4 ld4(const float* p, uint64_t q) {
    return __ldg(reinterpret_cast<const float4*>(p) + q);
}
__device__ __forceinline__ float f4get(const float4& v, int e) {
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint32_t warp_sum_u(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
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
// Deterministic last-arriver combine tree over a segment's tiles. Level 0 =
// leaves (one per CTA), level l+1 node i = children [16i, 16i+16) of level l.
// The CTA that completes a node's last child combines the children in index
// order, so the result is independent of scheduling. Returns false when the
// calling CTA is not the one to continue upward.
struct TreeCursor {
    uint32_t level, idx, n, off;  // off: node offset of this level (level >= 1)
};

__device__ __forceinline__ bool tree_arrive(TreeCursor& c, uint32_t* counters, uint32_t node_base, uint32_t* s_flag) {
    const uint32_t parent = c.idx / kFan;
    const uint32_t first = parent * kFan;
    const uint32_t nch = min((uint32_t)kFan, c.n - first);
    const uint32_t poff = c.level == 0 ? 0u : c.off + c.n;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t* ctr = counters + node_base + poff + parent;
        const bool last = atomicAdd(ctr, 1u) == nch - 1;
        if (last) *ctr = 0;  // re-arm for the next launch (no other arrivals remain)
        *s_flag = last ? 1u : 0u;
    }
    __syncthreads();
    if (!*s_flag) return false;
    __threadfence();
    c.idx = parent;  // caller combines children [first, first+nch) of the old level
    return true;
}

// ---------------------------------------------------------------------------
// K_stats: fused producer (PG / hop dequant-add / divide) + moments. Writes x
// to scratch (for k_bin) unless the source is a plain buffer. The combine
// tree's root publishes SegStat (mu, sigma, lo, hi, width, threshold table).

template <int SRC>
__global__ void __launch_bounds__(kThreads, 3) k_stats(QuantArgs a) {
    __shared__ float lut[kBuckets];
    __shared__ StatP wp[kWarps];
    __shared__ uint32_t s_flag;
    __shared__ double s_red[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t s = a.cta_seg[blockIdx.x];
    const SegInfo si = a.segs[s];
    const uint32_t tile = blockIdx.x - si.cta0;
    const uint32_t u = tile * kWarps + warp;  // segment-relative unit
    const uint64_t hiel = si.lo + si.len;     // exclusive
    const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;

    if (SRC & kHasIn) {
        lut[threadIdx.x] = a.in_cb[(uint64_t)si.in_slot * kBuckets + threadIdx.x];
        __syncthreads();
    }

    float v[kSlotsPerLane][4];
    double sum = 0.0;
    uint32_t cnt = 0;
    bool bad = false;
    if (u < si.nunits) {
#pragma unroll
        for (int j = 0; j < kSlotsPerLane; ++j) {
            const uint64_t q = qbase + (uint64_t)j * 32 + lane;
            const uint64_t e0 = q * 4;
#pragma unroll
            for (int e = 0; e < 4; ++e) v[j][e] = 0.f;
            if (e0 >= hiel) continue;
            float4 xa = ld4_stream(a.a, q);
            float x[4] = {xa.x, xa.y, xa.z, xa.w};
            if (SRC & kSrcAminusB) {
                float4 xb = ld4_stream(a.b, q);
                x[0] = __fsub_rn(x[0], xb.x); x[1] = __fsub_rn(x[1], xb.y);
                x[2] = __fsub_rn(x[2], xb.z); x[3] = __fsub_rn(x[3], xb.w);
            }
            if (SRC & kHasIn) {
                uint32_t c4 = __ldcs(reinterpret_cast<const uint32_t*>(a.in_codes) + q);
#pragma unroll
                for (int e = 0; e < 4; ++e) x[e] = __fadd_rn(x[e], lut[(c4 >> (8 * e)) & 0xff]);
            }
            if (SRC & kDivK) {
#pragma unroll
                for (int e = 0; e < 4; ++e) x[e] = __fdiv_rn(x[e], a.divisor);
            }
            const bool full = e0 >= si.lo && e0 + 4 <= hiel;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const bool valid = full || (e0 + e >= si.lo && e0 + e < hiel);
                if (valid) {
                    v[j][e] = x[e];
                    sum = __dadd_rn(sum, (double)x[e]);
                    cnt += 1;
                    bad |= !isfinite(x[e]);
                }
            }
            if (SRC != kSrcA) {
                float4* dst = reinterpret_cast<float4*>(a.scratch) + (q - a.scratch_q0);
                if (full) {
                    *dst = make_float4(x[0], x[1], x[2], x[3]);
                } else {
                    float* d1 = reinterpret_cast<float*>(dst);
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (e0 + e >= si.lo && e0 + e < hiel) d1[e] = x[e];
                }
            }
        }
    }
    const double S = warp_sum_d(sum);
    const uint32_t n = warp_sum_u(cnt);
    const double m = n ? __ddiv_rn(S, (double)n) : 0.0;
    double m2 = 0.0, dd = 0.0;
    if (u < si.nunits) {
#pragma unroll
        for (int j = 0; j < kSlotsPerLane; ++j) {
            const uint64_t e0 = (qbase + (uint64_t)j * 32 + lane) * 4;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (e0 + e >= si.lo && e0 + e < hiel) {
                    const double dv = __dsub_rn((double)v[j][e], m);
                    m2 = __dadd_rn(m2, __dmul_rn(dv, dv));
                    dd = __dadd_rn(dd, dv);
                }
            }
        }
    }
    m2 = warp_sum_d(m2);
    dd = warp_sum_d(dd);
    const bool anybad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        wp[warp] = StatP{S, m2, dd, m, (uint64_t)n};
        if (anybad) {
            atomicOr(&a.seg_flags[s], kFlagNonFinite);
            atomicOr(a.err, 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        StatP t = wp[0];
        for (int w = 1; w < kWarps; ++w) t = statp_merge(t, wp[w]);
        a.leaf_stat[blockIdx.x] = t;
    }
    // ---- combine tree over this segment's tiles
    TreeCursor c{0, tile, si.ncta, 0};
    while (c.n > 1) {
        const uint32_t lvl = c.level, n_old = c.n, off_old = c.off;
        if (!tree_arrive(c, a.tree_cnt, si.node_base, &s_flag)) return;
        const uint32_t first = c.idx * kFan, nch = min((uint32_t)kFan, n_old - first);
        const uint32_t poff = lvl == 0 ? 0u : off_old + n_old;
        if (threadIdx.x == 0) {
            StatP t{0, 0, 0, 0, 0};
            for (uint32_t i = 0; i < nch; ++i) {
                const StatP* src = lvl == 0 ? &a.leaf_stat[si.cta0 + first + i] : &a.node_stat[si.node_base + off_old + first + i];
                StatP ch;
                ch.s = __ldcg(&src->s); ch.m2 = __ldcg(&src->m2); ch.d = __ldcg(&src->d);
                ch.piv = __ldcg(&src->piv); ch.n = __ldcg(&src->n);
                t = statp_merge(t, ch);
            }
            a.node_stat[si.node_base + poff + c.idx] = t;
        }
        c.level = lvl + 1;
        c.n = (n_old + kFan - 1) / kFan;
        c.off = poff;
    }
    // ---- root: finalize segment statistics (quant.hpp:33-59)
    __syncthreads();
    __threadfence();
    if (threadIdx.x == 0) {
        const StatP* src = c.level == 0 ? &a.leaf_stat[blockIdx.x] : &a.node_stat[si.node_base + c.off];
        StatP t;
        t.s = __ldcg(&src->s); t.m2 = __ldcg(&src->m2); t.d = __ldcg(&src->d); t.piv = __ldcg(&src->piv);
        t.n = __ldcg(&src->n);
        const double mu = __ddiv_rn(t.s, (double)si.len);
        const double dm = __dsub_rn(t.piv, mu);
        // sum (x - mu)^2 = M2 + 2 (p - mu) D + n (p - mu)^2
        double ss = __dadd_rn(t.m2, __dmul_rn(__dmul_rn(2.0, dm), t.d));
        ss = __dadd_rn(ss, __dmul_rn((double)t.n, __dmul_rn(dm, dm)));
        const double var = __ddiv_rn(ss < 0.0 ? 0.0 : ss, (double)si.len);
        s_red[0] = mu;
        s_red[1] = __dsqrt_rn(var);
    }
    __syncthreads();
    const double mu = s_red[0], sigma = s_red[1];
    SegStat* st = &a.stats[si.slot];
    if (threadIdx.x == 0) {
        st->mu = mu;
        st->sigma = sigma;
        st->flags = __ldcg(&a.seg_flags[s]) | (sigma == 0.0 ? kFlagDegenerate : 0u);
        a.seg_flags[s] = 0;
        if (sigma == 0.0) {
            st->lo = mu; st->hi = mu; st->width = 0.0;
            st->lo_f = (float)mu; st->inv_w_f = 0.f;
        }
    }
    if (sigma != 0.0) {
        const double six = __dmul_rn(6.0, sigma);
        const double lo = __dsub_rn(mu, six);
        const double hi = __dadd_rn(mu, six);
        const double w = __ddiv_rn(__dsub_rn(hi, lo), 256.0);
        if (threadIdx.x == 0) {
            st->lo = lo; st->hi = hi; st->width = w;
            st->lo_f = (float)lo;
            st->inv_w_f = (float)__ddiv_rn(1.0, w);
            st->thr[0] = -INFINITY;
        } else {
            st->thr[threadIdx.x] = threshold(threadIdx.x, lo, hi, w);
        }
    }
}

// ---------------------------------------------------------------------------
// Deterministic per-warp histogram update: lanes holding the same bucket are
// combined in lane order by the group's lowest lane, which alone touches the
// warp-private smem row (no fp64 smem atomics — they are CAS loops on sm_100
// and their order is nondeterministic).
__device__ __forceinline__ void warp_hist_add(double* wsum, uint32_t* wcnt, int key, double xc, bool valid) {
    const int lane = threadIdx.x & 31;
    const int k = valid ? key : (kBuckets + lane);  // invalid lanes: unique dummy keys
    const uint32_t peers = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(peers) - 1;
    double acc = xc;
    uint32_t rem = (lane == leader) ? (peers & (peers - 1)) : 0u;  // others, ascending
    while (__any_sync(0xffffffffu, rem != 0u)) {
        const int src = rem ? (__ffs(rem) - 1) : lane;
        const double o = __shfl_sync(0xffffffffu, xc, src);
        if (rem) { acc = __dadd_rn(acc, o); rem &= rem - 1; }
    }
    if (valid && lane == leader) {
        wsum[key] = __dadd_rn(wsum[key], acc);
        wcnt[key] += __popc(peers);
    }
    __syncwarp();
}

// K_bin: codes + per-tile 256-bucket (sum of clipped x, count) histogram;
// the combine tree's root turns the segment histogram into the codebook
// (quant.hpp:78-85).
template <bool FROM_SCRATCH>
__global__ void __launch_bounds__(kThreads) k_bin(QuantArgs a) {
    __shared__ double wsum[kWarps][kBuckets];
    __shared__ uint32_t wcnt[kWarps][kBuckets];
    __shared__ float thr[kBuckets + 1];
    __shared__ uint32_t s_flag;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t s = a.cta_seg[blockIdx.x];
    const SegInfo si = a.segs[s];
    const uint32_t tile = blockIdx.x - si.cta0;
    const SegStat* st = &a.stats[si.slot];
    const double lo = st->lo, hi = st->hi;
    const float lo_f = st->lo_f, inv_w = st->inv_w_f;
    const bool degenerate = (st->flags & kFlagDegenerate) != 0;
    thr[threadIdx.x] = st->thr[threadIdx.x];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) { wsum[w][threadIdx.x] = 0.0; wcnt[w][threadIdx.x] = 0u; }
    if (threadIdx.x == 0) { thr[0] = -INFINITY; thr[kBuckets] = INFINITY; }
    __syncthreads();

    const uint64_t hiel = si.lo + si.len;
    const uint32_t u = tile * kWarps + warp;
    if (u < si.nunits) {
        const uint64_t qbase = si.q0 + (uint64_t)u * kUnitSlots;
#pragma unroll 2
        for (int j = 0; j < kSlotsPerLane; ++j) {
            const uint64_t q = qbase + (uint64_t)j * 32 + lane;
            const uint64_t e0 = q * 4;
            const bool any = e0 < hiel;
            float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (any) xv = FROM_SCRATCH ? *(reinterpret_cast<const float4*>(a.scratch) + (q - a.scratch_q0))
                                       : ld4(a.a, q);
            const bool full = any && e0 >= si.lo && e0 + 4 <= hiel;
            uint32_t packed = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const bool valid = any && (full || (e0 + e >= si.lo && e0 + e < hiel));
                const float x = f4get(xv, e);
                int c = 0;
                double xc = 0.0;
                if (!degenerate) {
                    float g = __fmul_rn(__fsub_rn(x, lo_f), inv_w);
                    c = g < 0.f ? 0 : (g > 255.f ? 255 : (int)g);
                    if (!(c >= 0 && c <= 255)) c = 0;  // NaN guard
                    while (c < 255 && x >= thr[c + 1]) ++c;
                    while (c > 0 && x < thr[c]) --c;
                    xc = (double)x;
                    if (xc < lo) xc = lo;
                    if (xc > hi) xc = hi;
                }
                packed |= (uint32_t)c << (8 * e);
                if (!degenerate) warp_hist_add(wsum[warp], wcnt[warp], c, xc, valid);
            }
            if (full) {
                reinterpret_cast<uint32_t*>(a.out_codes)[q] = packed;
            } else if (any) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (e0 + e >= si.lo && e0 + e < hiel) a.out_codes[e0 + e] = (uint8_t)(packed >> (8 * e));
            }
        }
    }
    __syncthreads();
    {   // tile histogram, fixed warp order
        const int b = threadIdx.x;
        double sm = 0.0;
        uint32_t cn = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) { sm = __dadd_rn(sm, wsum[w][b]); cn += wcnt[w][b]; }
        a.leaf_sum[(uint64_t)blockIdx.x * kBuckets + b] = sm;
        a.leaf_cnt[(uint64_t)blockIdx.x * kBuckets + b] = cn;
    }
    // ---- combine tree (16 independent loads per thread per level)
    uint32_t* ctr = a.tree_cnt + a.nnodes;
    TreeCursor c{0, tile, si.ncta, 0};
    double rs = 0.0;
    uint64_t rc = 0;
    bool have = false;
    while (c.n > 1) {
        const uint32_t lvl = c.level, n_old = c.n, off_old = c.off;
        if (!tree_arrive(c, ctr, si.node_base, &s_flag)) return;
        const uint32_t first = c.idx * kFan, nch = min((uint32_t)kFan, n_old - first);
        const uint32_t poff = lvl == 0 ? 0u : off_old + n_old;
        const int b = threadIdx.x;
        double ps[kFan];
        uint32_t pc[kFan];
#pragma unroll
        for (int i = 0; i < kFan; ++i) {
            if ((uint32_t)i < nch) {
                const uint64_t ix = (lvl == 0 ? (uint64_t)(si.cta0 + first + i) : (uint64_t)(si.node_base + off_old + first + i)) * kBuckets + b;
                ps[i] = __ldcg((lvl == 0 ? a.leaf_sum : a.node_sum) + ix);
                pc[i] = __ldcg((lvl == 0 ? a.leaf_cnt : a.node_cnt) + ix);
            } else { ps[i] = 0.0; pc[i] = 0u; }
        }
        rs = 0.0;
        rc = 0;
#pragma unroll
        for (int i = 0; i < kFan; ++i) { rs = __dadd_rn(rs, ps[i]); rc += pc[i]; }
        have = true;
        if ((n_old + kFan - 1) / kFan > 1) {  // not the root yet: publish the node
            a.node_sum[(uint64_t)(si.node_base + poff + c.idx) * kBuckets + b] = rs;
            a.node_cnt[(uint64_t)(si.node_base + poff + c.idx) * kBuckets + b] = (uint32_t)rc;
        }
        c.level = lvl + 1;
        c.n = (n_old + kFan - 1) / kFan;
        c.off = poff;
    }
    if (!have) {  // single-tile segment: this CTA's own histogram is the root
        __syncthreads();
        double sm = 0.0;
        uint32_t cn = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) { sm = __dadd_rn(sm, wsum[w][threadIdx.x]); cn += wcnt[w][threadIdx.x]; }
        rs = sm;
        rc = cn;
    }
    const int b = threadIdx.x;
    float* cb = a.out_cb + (uint64_t)si.slot * kBuckets;
    if (degenerate) cb[b] = (float)st->mu;
    else if (rc) cb[b] = (float)__ddiv_rn(rs, (double)rc);
    else cb[b] = (float)__dadd_rn(lo, __dmul_rn(__dadd_rn((double)b, 0.5), st->width));
}

// ---------------------------------------------------------------------------
// Elementwise kernels over segment batches (codebook LUT in smem).

struct ApplyArgs {
    const SegInfo* segs;
    const uint32_t* cta_seg;
    uint32_t ncta;
    const uint8_t* codes;  // arena-indexed
    const float* cb;       // [slot][256]
    float* theta;          // theta_g, updated in place
    float* buf;            // Nesterov momentum, updated in place
    float* theta_local;    // optional: theta_l <- theta_g (trainer.hpp:382)
    float* out;            // dequantize target (arena-indexed)
    float lr, mom;
};

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
    const SegInfo si = a.segs[a.cta_seg[blockIdx.x]];
    lut[threadIdx.x] = a.cb[(uint64_t)si.slot * kBuckets + threadIdx.x];
    __syncthreads();
    const uint32_t u = (blockIdx.x - si.cta0) * kWarps + warp;
    if (u >= si.nunits) return;
    const uint64_t hiel = si.lo + si.len;
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
