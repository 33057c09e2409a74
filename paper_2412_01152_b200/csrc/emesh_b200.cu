// C-ABI, segment planning and the ring engine (NCCL over NVLink, or k
// virtual workers on one GPU) for the outer-synchronisation hot path.
// See include/emesh_b200.h for the reference interface each entry replaces.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <functional>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "emesh_b200.h"
#include "kernels.cuh"
#include "quant.cuh"

using namespace emesh_b200;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

}  // namespace

namespace emesh_b200 {
int set_error(int code, const std::string& msg) {  // for the other translation units (checkpoint.cu)
    g_err = msg;
    return code;
}
}  // namespace emesh_b200

namespace {

#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(EMESH_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)
#define NC(call)                                                                          \
    do {                                                                                  \
        ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess)                                                            \
            return fail(EMESH_ENCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, __LINE__); \
    } while (0)
#define TRY(expr)                   \
    do {                            \
        int rc_ = (expr);           \
        if (rc_ != EMESH_OK) return rc_; \
    } while (0)

// ---------------------------------------------------------------------------
// Segment plan: allreduce.hpp:107-118 (split) and :326-336 (subs_of).

void split_piece(uint64_t total, uint64_t parts, uint64_t i, uint64_t* lo, uint64_t* len) {
    const uint64_t base = parts ? total / parts : 0, rem = parts ? total % parts : 0;
    *len = base + (i < rem ? 1 : 0);
    *lo = i * base + (i < rem ? i : rem);
}

struct Seg {
    uint64_t lo, len;
};

uint32_t quant_lag_tiles();
bool bin_reverse();
bool quant_mix();

// One pipelining window: consecutive segments of one rank chunk.
struct Batch {
    uint32_t chunk = 0, window = 0;
    uint32_t slot0 = 0, nseg = 0;
    uint64_t el_lo = 0, el_hi = 0;  // element span [el_lo, el_hi) (contiguous for a flat arena)
    uint64_t elems = 0;             // elements in the batch
    std::vector<std::pair<uint64_t, uint64_t>> eruns;  // contiguous element runs {lo, len} (transfers)
    uint32_t ncta = 0, nruns = 0, ntasks = 0;
    uint32_t upw = kUnitsPerWarp;   // warp units per tile (tile_units_per_warp)
    size_t off_segs = 0, off_cta = 0, off_runs = 0;  // byte offsets into the table arena
    const SegInfo* d_segs = nullptr;
    const uint32_t* d_cta_seg = nullptr;
    const uint4* d_runs = nullptr;

    void bind(void* base) {
        d_segs = reinterpret_cast<const SegInfo*>((char*)base + off_segs);
        d_cta_seg = reinterpret_cast<const uint32_t*>((char*)base + off_cta);
        d_runs = reinterpret_cast<const uint4*>((char*)base + off_runs);
    }
};

// Tile shape per batch: 4 warp units (16K elements) per tile for large batches,
// 2 (8K) for small ones and 1 for tiny ones, where more CTAs per segment shorten
// the serial STATS -> thresholds -> BIN chain. Measured at 2 GPUs
// (profiles/r01_u2_ab/): 2-unit tiles take 0.101 vs 0.122 ms per round at 1 MB,
// 0.171 vs 0.183 ms at 64 MB (8M-element batches), but are 2-4 % slower from
// 32M-element batches up; 1-unit tiles (profiles/r01_tile1/) a further -8..-14 %
// on <= 2M-element batches at 2 and 4 GPUs, mixed at 4M-8M.
uint32_t tile_units_per_warp(uint64_t batch_elems) {
    constexpr uint64_t kTinyBatchElems = 2ull << 20, kSmallBatchElems = 16ull << 20;
    if (batch_elems <= kTinyBatchElems) return 1u;
    return batch_elems <= kSmallBatchElems ? (uint32_t)std::min(2, kUnitsPerWarp) : (uint32_t)kUnitsPerWarp;
}

struct Plan {
    uint64_t n = 0;
    uint32_t k = 1, S = 4;
    std::vector<Seg> segs;                      // global slot order (chunk-major)
    std::vector<std::vector<Batch>> batches;    // [chunk][window]
    std::vector<uint8_t> host_tables;
    void* d_tables = nullptr;
    size_t max_cta = 0, max_segs = 0, max_slots = 0;

    // Appends the device tables for one batch over segments [s0, s1).
    // One batch over every segment (the peer transport's single decode launch
    // per round); built after the ring batches, not sized into the quantizer's
    // workspace (it never quantizes).
    Batch all;
    bool has_all = false;
    void add_all() {
        const size_t mc = max_cta, ms = max_segs, mx = max_slots;
        add_batch(0, 0, 0, (uint32_t)segs.size());
        all = batches[0].back();
        batches[0].pop_back();
        max_cta = mc; max_segs = ms; max_slots = mx;
        has_all = true;
    }

    void add_batch(uint32_t chunk, uint32_t window, uint32_t s0, uint32_t s1) {
        Batch b;
        b.chunk = chunk;
        b.window = window;
        b.slot0 = s0;
        b.nseg = s1 - s0;
        {
            uint64_t tot = 0;
            for (uint32_t s = s0; s < s1; ++s) tot += segs[s].len;
            b.upw = tile_units_per_warp(tot);
        }
        std::vector<SegInfo> infos;
        std::vector<uint32_t> cseg;
        bool first = true;
        uint64_t sq = 0;  // scratch float4 slots so far
        for (uint32_t s = s0; s < s1; ++s) {
            const Seg& g = segs[s];
            SegInfo si{};
            si.lo = g.lo;
            si.len = g.len;
            si.q0 = g.lo >> 2;
            si.sq0 = sq;
            si.cta0 = (uint32_t)cseg.size();
            si.slot = s;
            si.in_slot = s;
            si.upw = b.upw;
            si.chunk = chunk;
            if (g.len > 0) {
                const uint64_t q_last = (g.lo + g.len - 1) >> 2;
                const uint64_t nq = q_last - si.q0 + 1;
                si.nunits = (uint32_t)((nq + kUnitSlots - 1) / kUnitSlots);
                si.ncta = (si.nunits + kWarps * b.upw - 1) / (kWarps * b.upw);
                // whole units: no 128-B scratch line (and no prefetched unit) is
                // shared with another segment, whose STATS may not have run yet
                sq += (nq + kUnitSlots - 1) / kUnitSlots * kUnitSlots;
                if (first) { b.el_lo = g.lo; first = false; }
                b.el_lo = std::min(b.el_lo, g.lo);
                b.el_hi = std::max(b.el_hi, g.lo + g.len);
                b.elems += g.len;
                if (!b.eruns.empty() && b.eruns.back().first + b.eruns.back().second == g.lo)
                    b.eruns.back().second += g.len;
                else
                    b.eruns.push_back({g.lo, g.len});
            }
            for (uint32_t t = 0; t < si.ncta; ++t) cseg.push_back((uint32_t)infos.size());
            infos.push_back(si);
        }
        b.ncta = (uint32_t)cseg.size();
        // persistent-kernel task order (see kernels.cuh): STATS tiles in
        // segment order; the BIN tiles of s (in reverse tile order: the most
        // recently written scratch is re-read first, while still in L2) become
        // available `lag` tasks after its last STATS tile and are then
        // interleaved 1:1 with the following STATS tiles, so every SM always
        // runs a mix of the HBM-bound STATS and the issue-bound BIN work.
        // Compressed into runs {first task, kind | bin segment << 2, segment,
        // first tile}: plain runs (one kind) and mixed runs (S, B, S, B, ...).
        std::vector<uint4> runs;
        {
            const uint32_t lag = quant_lag_tiles();
            struct Task { uint32_t kind, seg, tile; };
            std::vector<Task> order;
            order.reserve(2 * (size_t)b.ncta);
            struct Pending { uint32_t seg, next, left, at; };
            std::vector<Pending> bq;
            size_t hb = 0;
            const bool mix = quant_mix();
            auto bin_ready = [&]() { return hb < bq.size() && order.size() >= bq[hb].at; };
            auto pop_bin = [&]() {
                Pending& pb = bq[hb];
                order.push_back({kTaskBin, pb.seg, pb.next});
                if (bin_reverse()) --pb.next; else ++pb.next;
                if (--pb.left == 0) ++hb;
            };
            for (uint32_t i = 0; i < infos.size(); ++i) {
                for (uint32_t t = 0; t < infos[i].ncta; ++t) {
                    order.push_back({kTaskStats, i, t});
                    if (mix) {
                        if (bin_ready()) pop_bin();
                    } else {  // whole-segment BIN blocks (no interleaving)
                        while (bin_ready()) pop_bin();
                    }
                }
                if (infos[i].ncta)
                    bq.push_back({i, bin_reverse() ? infos[i].ncta - 1 : 0u, infos[i].ncta,
                                  (uint32_t)order.size() + lag});
            }
            while (hb < bq.size()) pop_bin();
            b.ntasks = (uint32_t)order.size();
            const int dir = bin_reverse() ? -1 : 1;
            size_t p0 = 0;
            while (p0 < order.size()) {
                const Task& t0 = order[p0];
                // mixed run: S(a, i), B(b, j), S(a, i+1), B(b, j+dir), ...
                size_t q = p0;
                if (t0.kind == kTaskStats && p0 + 1 < order.size() && order[p0 + 1].kind == kTaskBin) {
                    const Task& t1 = order[p0 + 1];
                    while (q + 1 < order.size()) {
                        const uint32_t i = (uint32_t)((q - p0) / 2);
                        const Task& s0 = order[q];
                        const Task& s1 = order[q + 1];
                        if (s0.kind != kTaskStats || s0.seg != t0.seg || s0.tile != t0.tile + i) break;
                        if (s1.kind != kTaskBin || s1.seg != t1.seg || (int64_t)s1.tile != (int64_t)t1.tile + dir * (int64_t)i) break;
                        q += 2;
                    }
                    if (q - p0 >= 4 && t0.tile < 0x10000u && t1.tile < 0x10000u) {
                        runs.push_back(make_uint4((uint32_t)p0, (dir < 0 ? kTaskMixRev : kTaskMixFwd) | (t1.seg << 2), t0.seg,
                                                  t0.tile | (t1.tile << 16)));
                        p0 = q;
                        continue;
                    }
                    q = p0;
                }
                // plain run of one kind and segment, tiles +1 (STATS) / +dir (BIN)
                const int step = t0.kind == kTaskBin ? dir : 1;
                q = p0 + 1;
                while (q < order.size() && order[q].kind == t0.kind && order[q].seg == t0.seg &&
                       (int64_t)order[q].tile == (int64_t)t0.tile + step * (int64_t)(q - p0))
                    ++q;
                runs.push_back(make_uint4((uint32_t)p0, t0.kind, t0.seg,
                                          step < 0 ? 0x80000000u | t0.tile : t0.tile));
                p0 = q;
            }
        }
        b.nruns = (uint32_t)runs.size();

        auto append = [&](const void* p, size_t bytes) {
            size_t off = (host_tables.size() + 15) & ~size_t(15);
            host_tables.resize(off + bytes);
            if (bytes) std::memcpy(host_tables.data() + off, p, bytes);
            return off;
        };
        b.off_segs = append(infos.data(), infos.size() * sizeof(SegInfo));
        b.off_cta = append(cseg.data(), cseg.size() * sizeof(uint32_t));
        b.off_runs = append(runs.data(), runs.size() * sizeof(uint4));

        max_cta = std::max<size_t>(max_cta, b.ncta);
        max_segs = std::max<size_t>(max_segs, b.nseg);
        max_slots = std::max<size_t>(max_slots, sq);
        batches[chunk].push_back(b);
    }

    int upload() {
        if (d_tables) cudaFree(d_tables);
        CU(cudaMalloc(&d_tables, std::max<size_t>(host_tables.size(), 16)));
        CU(cudaMemcpy(d_tables, host_tables.data(), host_tables.size(), cudaMemcpyHostToDevice));
        for (auto& row : batches)
            for (auto& b : row) b.bind(d_tables);
        if (has_all) all.bind(d_tables);
        return EMESH_OK;
    }
    void release() {
        if (d_tables) cudaFree(d_tables);
        d_tables = nullptr;
    }
};

constexpr uint64_t kDefaultWindow = (uint64_t)16 << 20;  // elements per pipelining window

int persistent_grid(const void* fn, uint32_t ntasks);
// Lag between a segment's last STATS tile and its first BIN tile in the task
// order: one persistent grid (the stats root publishes within about one
// tile time; longer lags push scratch x out of L2).
// measured best (round 1, config 2): BIN interleaved 1:1 with STATS, a segment's BIN tiles
// in reverse tile order (the most recently written scratch first), 1.5 persistent grids of lag
bool quant_mix() { return true; }
bool bin_reverse() { return true; }
uint32_t quant_lag_tiles() {
    const int g = persistent_grid((const void*)k_quant<kSrcAminusB | kHasIn>, 1u << 30);
    return (uint32_t)std::max(1.0, 1.5 * (g > 0 ? g : 512));
}


// Ring plan: k chunks, min(S, len) subs each, windows of G segments.
Plan make_ring_plan(uint64_t n, uint32_t k, uint32_t S, uint64_t window_elems) {
    Plan p;
    p.n = n;
    p.k = k;
    p.S = S;
    p.batches.resize(k);
    std::vector<uint32_t> first(k + 1);
    uint64_t max_seg = 1;
    for (uint32_t c = 0; c < k; ++c) {
        uint64_t clo, clen;
        split_piece(n, k, c, &clo, &clen);
        const uint64_t ns = clen == 0 ? 1 : std::min<uint64_t>(S, clen);
        first[c] = (uint32_t)p.segs.size();
        for (uint64_t j = 0; j < ns; ++j) {
            uint64_t slo, slen;
            split_piece(clen, ns, j, &slo, &slen);
            p.segs.push_back({clo + slo, slen});
            max_seg = std::max(max_seg, slen);
        }
    }
    first[k] = (uint32_t)p.segs.size();
    uint64_t G = std::max<uint64_t>(1, window_elems / max_seg);
    // chunks shorter than S have fewer sub-slices; keep one window per chunk
    // then so every rank agrees on the window count (NCCL send/recv pairing).
    if (n < (uint64_t)k * S) G = S;
    G = std::min<uint64_t>(G, S);  // a chunk never has more than S segments
    for (uint32_t c = 0; c < k; ++c) {
        uint32_t w = 0;
        for (uint64_t s = first[c]; s < first[c + 1]; s += G, ++w)
            p.add_batch(c, w, (uint32_t)s, (uint32_t)std::min<uint64_t>(first[c + 1], s + G));
    }
    if (k > 1) p.add_all();
    return p;
}

// Multi-tensor ring: one ReduceJob per tensor, i.e.
// every tensor is split into k chunks x min(S, len) segments on its own
// (allreduce.hpp:107-118, :326-336); ring chunk c is the union of the
// tensors' chunk c ("bucketing": one launch / one transfer group per hop).
// Slots are chunk-major, tensors in order within a chunk. Windows: `nwin`
// per chunk by cumulative elements (equal counts on every chunk, as the
// NCCL schedule pairs windows); nwin = 0 sizes them from window_elems.
Plan make_tensor_ring_plan(const uint64_t* sizes, uint32_t nt, uint32_t k, uint32_t S, uint64_t window_elems) {
    Plan p;
    p.k = k;
    p.S = S;
    p.batches.resize(k);
    std::vector<uint64_t> off(nt + 1, 0);
    for (uint32_t t = 0; t < nt; ++t) off[t + 1] = off[t] + sizes[t];
    p.n = off[nt];
    std::vector<uint32_t> first(k + 1);
    uint64_t max_chunk = 1;
    for (uint32_t c = 0; c < k; ++c) {
        first[c] = (uint32_t)p.segs.size();
        uint64_t tot = 0;
        for (uint32_t t = 0; t < nt; ++t) {
            uint64_t clo, clen;
            split_piece(sizes[t], k, c, &clo, &clen);
            const uint64_t ns = clen == 0 ? 1 : std::min<uint64_t>(S, clen);
            for (uint64_t j = 0; j < ns; ++j) {
                uint64_t slo, slen;
                split_piece(clen, ns, j, &slo, &slen);
                p.segs.push_back({off[t] + clo + slo, slen});
            }
            tot += clen;
        }
        max_chunk = std::max(max_chunk, tot);
    }
    first[k] = (uint32_t)p.segs.size();
    const uint64_t W = std::max<uint64_t>(1, std::min<uint64_t>((max_chunk + window_elems - 1) / std::max<uint64_t>(window_elems, 1), 64));
    for (uint32_t c = 0; c < k; ++c) {
        uint64_t tot = 0;
        for (uint32_t s = first[c]; s < first[c + 1]; ++s) tot += p.segs[s].len;
        uint32_t s = first[c];
        uint64_t cum = 0;
        for (uint64_t w = 0; w < W; ++w) {
            const uint64_t end = tot * (w + 1) / W;  // segments starting before `end` join window w
            const uint32_t s0 = s;
            while (s < first[c + 1] && (cum < end || w + 1 == W)) cum += p.segs[s++].len;
            p.add_batch(c, (uint32_t)w, s0, s);
        }
    }
    if (k > 1) p.add_all();
    return p;
}

// Plan over an explicit segment list (the standalone codec API): one batch.
Plan make_list_plan(const uint64_t* lo, const uint64_t* len, uint32_t nseg) {
    Plan p;
    p.k = 1;
    p.batches.resize(1);
    for (uint32_t i = 0; i < nseg; ++i) p.segs.push_back({lo[i], len[i]});
    p.add_batch(0, 0, 0, nseg);
    return p;
}

// Device scratch shared by every batch launched on one stream.
struct Workspace {
    float* scratch = nullptr;
    StatP* leaf_stat = nullptr;
    SegAcc* acc = nullptr;  // zero between launches (self-cleaning, see SegAcc)
    uint32_t* seg_flags = nullptr;
    uint32_t* sync = nullptr;
    uint32_t* err = nullptr;
    size_t cap_slots = 0, cap_cta = 0, cap_segs = 0;

    template <typename T>
    static int grow(T*& p, size_t& cap, size_t want, size_t elems_per, bool zero) {
        if (want <= cap && p) return EMESH_OK;
        if (p) CU(cudaFree(p));
        const size_t bytes = std::max<size_t>(want, 1) * elems_per * sizeof(T);
        CU(cudaMalloc(&p, bytes));
        if (zero) CU(cudaMemset(p, 0, bytes));
        return EMESH_OK;
    }

    int reserve(size_t slots, size_t ctas, size_t segs) {
        if (!err) {  // [0] sticky bits, [1] culprit rank + 1 (kernels.cuh ring_fail)
            CU(cudaMalloc(&err, 4 * sizeof(uint32_t)));
            CU(cudaMemset(err, 0, 4 * sizeof(uint32_t)));
        }
        if (slots > cap_slots || !scratch) {
            size_t c = 0;
            TRY(grow(scratch, c, slots, 4, false));
            cap_slots = std::max<size_t>(slots, 1);
        }
        if (ctas > cap_cta || !leaf_stat) {
            size_t c = 0;
            TRY(grow(leaf_stat, c, ctas, 1, false));
            cap_cta = std::max<size_t>(ctas, 1);
        }
        if (segs > cap_segs || !seg_flags) {
            size_t c = 0;
            TRY(grow(seg_flags, c, segs, 1, true));
            c = 0;
            TRY(grow(acc, c, segs, 1, true));
            c = 0;
            TRY(grow(sync, c, kSyncReady + 3 * segs, 1, true));
            cap_segs = std::max<size_t>(segs, 1);
        }
        return EMESH_OK;
    }
    void release() {
        cudaFree(scratch); cudaFree(leaf_stat); cudaFree(acc); cudaFree(seg_flags); cudaFree(sync); cudaFree(err);
        *this = Workspace();
    }
};


// ---------------------------------------------------------------------------
// Launchers

struct QuantIO {
    int src;                  // kSrc* | kHasIn | kDivK
    const float* a;
    const float* b;
    const uint8_t* in_codes;
    const float* in_cb;
    float divisor;
    uint8_t* out_codes;
    float* out_cb;
    SegStat* stats;
    // peer transport: extra output destinations (peer arenas), arrival flags
    // to raise per finished segment, and the input wait
    uint32_t nx = 0;
    bool local_out = true;  // out_codes/out_cb is a destination too
    uint8_t* x_codes[kMaxDest] = {};
    float* x_cb[kMaxDest] = {};
    uint32_t nflags = 0;
    uint32_t* flags[kMaxDest] = {};
    const uint32_t* in_flag = nullptr;
    uint32_t epoch = 0;
    // ChunkMsg headers (peer transport): one per destination (nullptr: none), the incoming ones
    ChunkHdr* hdr_out[kMaxDest] = {};  // parallel to the destinations: [0] = out (when local_out), then x_*
    const ChunkHdr* in_hdr = nullptr;
    HdrRef hdr{};
    uint32_t phase_out = kPhaseRS;
    uint32_t culprit_in = kNoCulprit;
    uint32_t* wait_self = nullptr;        // "waiting" words (peer transport, spin_until_ge_sys)
    const uint32_t* wait_pred = nullptr;
    uint32_t* done_dst[kMaxDest] = {};    // owner's final quantizer: the peers' done words for this rank
    uint32_t ndone = 0;
};

enum ProfKind : int {
    // 0, 1: reserved (the round-1 two-kernel quantizer's separate passes)
    kProfQuantPG = 2,    // k_quant, hop-0 payload Q(theta_g - theta_l)
    kProfQuantHop = 3,   // k_quant, reduce-scatter hop (dequant-add-requant)
    kProfQuantFinal = 4, // k_quant, owner mean (/k) + quantize
    kProfQuantPlain = 5, // k_quant, plain buffer
    kProfNesterov = 6,   // k_apply<1>: dequant + Nesterov (+ theta_l write)
    kProfDequant = 7,    // k_apply<0>
    kProfFusedK1 = 8,    // k_nesterov_f32 (k == 1: PG + Nesterov)
    kProfF32Hop = 9,     // k_f32_hop (ReduceMode::fp32 accumulate / mean)
    kProfF32Apply = 10,  // k_f32_apply (ReduceMode::fp32 decode + Nesterov)
};

// Launch accounting + optional per-kernel CUDA-event profiling on the
// launching stream (bench.py's roofline numbers come from here).
struct Tracker {
    uint64_t launches = 0;
    bool prof = false;
    // peer-transport waits of this engine's kernels: error word + budget
    uint32_t* err = nullptr;
    unsigned long long timeout_ns = 30ull * 1000000000ull;
    struct Rec {
        int kind;
        cudaEvent_t a, b;
        double bytes;
    };
    std::vector<Rec> recs;
    struct OpRec {
        int kind, phase, hop, window;
        cudaEvent_t a, b;
    };
    std::vector<OpRec> ops;  // NCCL-mode op timeline (emesh_engine_timeline)
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    cudaEvent_t ev(cudaStream_t st) {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        cudaEvent_t e = pool[used++];
        cudaEventRecord(e, st);
        return e;
    }
    void reset() {
        recs.clear();
        ops.clear();
        used = 0;
    }
    void release() {
        for (auto e : pool) cudaEventDestroy(e);
        pool.clear();
        recs.clear();
        used = 0;
    }
};
Tracker g_codec_tracker;

// Co-resident grid of the persistent quantizer (occupancy x SMs, capped at the task count).
int persistent_grid(const void* fn, uint32_t ntasks) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> g(mu);
        for (auto& kv : cache)
            if (kv.first == fn) per_sm = kv.second;
        if (!per_sm) {
            if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQuantSmemBytes) != cudaSuccess)
                return -1;
            // the smallest carveout that holds kQuantMinBlocks CTAs (+1 KB reserved each): the rest
            // of the 256 KB stays L1, which stages the in-flight global loads
            int smem_sm = 0;
            cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
            const size_t need = (size_t)kQuantMinBlocks * (kQuantSmemBytes + 1024);
            int pct = smem_sm > 0 ? (int)((100 * need + smem_sm - 1) / (size_t)smem_sm) : 100;
            cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, std::min(pct, 100));
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, kQuantSmemBytes) != cudaSuccess)
                return -1;
            cache.push_back({fn, per_sm});
        }
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long want = (long long)per_sm * sms;
    return (int)std::max<long long>(1, std::min<long long>(want, ntasks));
}

int launch_quant(const Batch& bt, Workspace& ws, const QuantIO& io, cudaStream_t st, Tracker* tr,
                 uint32_t reserve_ctas = 0) {
    if (bt.ncta == 0) return EMESH_OK;
    QuantArgs a{};
    a.segs = bt.d_segs;
    a.cta_seg = bt.d_cta_seg;
    a.ncta = bt.ncta;
    a.nseg = bt.nseg;
    a.a = io.a;
    a.b = io.b;
    a.in_codes = io.in_codes;
    a.in_cb = io.in_cb;
    a.divisor = io.divisor;
    {
        int ex = 0;
        const float m = std::frexp(io.divisor, &ex);
        a.inv_divisor = (m == 0.5f) ? std::ldexp(1.0f, 1 - ex) : 0.f;  // exact reciprocal of a power of two
    }
    a.scratch = ws.scratch;
    a.ndest = 0;
    if (io.local_out) {
        a.dcodes[0] = io.out_codes;
        a.dcb[0] = io.out_cb;
        a.ndest = 1;
    }
    if (io.nflags > (uint32_t)kMaxDest || a.ndest + io.nx > (uint32_t)kMaxDest)
        return fail(EMESH_ECONFIG, "too many quantizer destinations");
    for (uint32_t d = 0; d < io.nx; ++d) {
        a.dcodes[a.ndest] = io.x_codes[d];
        a.dcb[a.ndest] = io.x_cb[d];
        ++a.ndest;
    }
    for (uint32_t f = 0; f < io.nflags; ++f) a.sflag[f] = io.flags[f];
    a.nflag = io.nflags;
    if (a.ndest == 0) return fail(EMESH_ECONFIG, "quantizer without a destination");
    a.ndest_fail = io.local_out ? 1 : a.ndest;  // a failed owner keeps its final payload local
    a.in_flag = io.in_flag;
    a.epoch = io.epoch;
    a.timeout_ns = tr ? tr->timeout_ns : 30ull * 1000000000ull;
    a.stats = io.stats;
    a.leaf_stat = ws.leaf_stat;
    a.acc = ws.acc;
    a.seg_flags = ws.seg_flags;
    a.err = ws.err;
    a.runs = bt.d_runs;
    a.nruns = bt.nruns;
    a.ntasks = bt.ntasks;
    a.sync = ws.sync;
    for (uint32_t d = 0; d < a.ndest; ++d) a.dhdr[d] = io.hdr_out[d];
    a.in_hdr = io.in_hdr;
    a.hdr = io.hdr;
    a.phase_out = io.phase_out;
    a.culprit_in = io.culprit_in;
    a.wait_self = io.wait_self;
    a.wait_pred = io.wait_pred;
    if (io.ndone > (uint32_t)kMaxDest) return fail(EMESH_ECONFIG, "too many done destinations");
    a.ndone = io.ndone;
    for (uint32_t d = 0; d < io.ndone; ++d) a.done_dst[d] = io.done_dst[d];
    CU(cudaMemsetAsync(ws.sync, 0, (kSyncReady + 3 * (size_t)bt.nseg) * sizeof(uint32_t), st));
    const bool prof = tr && tr->prof;
    cudaEvent_t e0 = prof ? tr->ev(st) : nullptr;
    void* args[] = {&a};
    const void* fn = nullptr;
    switch (io.src) {
        case kSrcA: fn = (const void*)k_quant<kSrcA>; break;
        case kSrcAminusB: fn = (const void*)k_quant<kSrcAminusB>; break;
        case kSrcA | kHasIn: fn = (const void*)k_quant<kSrcA | kHasIn>; break;
        case kSrcAminusB | kHasIn: fn = (const void*)k_quant<kSrcAminusB | kHasIn>; break;
        case kSrcA | kHasIn | kDivK: fn = (const void*)k_quant<kSrcA | kHasIn | kDivK>; break;
        case kSrcAminusB | kHasIn | kDivK: fn = (const void*)k_quant<kSrcAminusB | kHasIn | kDivK>; break;
        default: return fail(EMESH_ECONFIG, "unsupported producer %d", io.src);
    }
    // A plain launch suffices: a task is claimed only by a running CTA and only
    // ever waits on tasks claimed before it, so progress never depends on
    // co-residency. `reserve` CTA slots stay free for NCCL's kernels so the
    // ring's transfers overlap this kernel.
    int grid = persistent_grid(fn, bt.ntasks);
    if (grid <= 0) return fail(EMESH_ECUDA, "k_quant: occupancy query failed");
    grid = std::max(1, grid - (int)reserve_ctas);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = kQuantSmemBytes;
    lc.stream = st;
    CU(cudaLaunchKernelExC(&lc, fn, args));
    if (tr) tr->launches += 1;
    if (prof) {
        cudaEvent_t e2 = tr->ev(st);
        const double elems = (double)bt.elems;
        const double rd = elems * (((io.src & kSrcAminusB) ? 8.0 : 4.0) + ((io.src & kHasIn) ? 1.0 : 0.0)) +
                          ((io.src & kHasIn) ? 1028.0 * bt.nseg : 0.0);
        const double wr = elems + 1028.0 * bt.nseg;
        const int fam = (io.src & kDivK) ? 2 : (io.src & kHasIn) ? 1 : (io.src & kSrcAminusB) ? 0 : 3;
        tr->recs.push_back({kProfQuantPG + fam, e0, e2, rd + wr});
    }
    CU(cudaGetLastError());
    return EMESH_OK;
}

// Decode (+ Nesterov) of one batch for nw local replicas (thetas / bufs / locals, nw <= kMaxDest).
int launch_apply_multi(const Batch& bt, int mode, const uint8_t* codes, const float* cb, float* const* thetas,
                       float* const* bufs, float* const* locals, uint32_t nw, float* out, float lr, float mom,
                       cudaStream_t st, Tracker* tr, const uint32_t* gate = nullptr, uint32_t epoch = 0);

int launch_apply(const Batch& bt, int mode, const uint8_t* codes, const float* cb, float* theta, float* buf,
                 float* theta_local, float* out, float lr, float mom, cudaStream_t st, Tracker* tr,
                 const uint32_t* gate = nullptr, uint32_t epoch = 0) {
    return launch_apply_multi(bt, mode, codes, cb, &theta, &buf, &theta_local, 1, out, lr, mom, st, tr, gate, epoch);
}

int launch_apply_multi(const Batch& bt, int mode, const uint8_t* codes, const float* cb, float* const* thetas,
                       float* const* bufs, float* const* locals, uint32_t nw, float* out, float lr, float mom,
                       cudaStream_t st, Tracker* tr, const uint32_t* gate, uint32_t epoch) {
    if (bt.ncta == 0) return EMESH_OK;
    if (nw == 0 || nw > (uint32_t)kMaxDest) return fail(EMESH_ECONFIG, "decode: bad replica count");
    ApplyArgs a{};
    a.nw = nw;
    for (uint32_t w = 0; w < nw; ++w) {
        a.thetas[w] = thetas[w];
        a.bufs[w] = bufs[w];
        a.locals[w] = locals ? locals[w] : nullptr;
    }
    float* const theta = thetas[0];
    float* const buf = bufs[0];
    float* const theta_local = locals ? locals[0] : nullptr;
    a.gate = gate;
    a.epoch = epoch;
    a.segs = bt.d_segs;
    a.cta_seg = bt.d_cta_seg;
    a.ncta = bt.ncta;
    a.codes = codes;
    a.cb = cb;
    a.theta = theta;
    a.buf = buf;
    a.theta_local = theta_local;
    a.out = out;
    a.lr = lr;
    a.mom = mom;
    a.upw = bt.upw;
    const dim3 g(bt.ncta * bt.upw), blk(kThreads);
    const bool prof = tr && tr->prof;
    cudaEvent_t e0 = prof ? tr->ev(st) : nullptr;
    if (mode == 0) k_apply<0><<<g, blk, 0, st>>>(a);
    else if (nw == 1) k_apply<1><<<g, blk, 0, st>>>(a);
    else k_apply<2><<<g, blk, 0, st>>>(a);
    if (tr) tr->launches += 1;
    if (prof) {
        const double elems = (double)bt.elems;
        const double by = mode == 0 ? elems * 5.0 : elems * (1.0 + nw * (theta_local ? 20.0 : 16.0));
        tr->recs.push_back({mode == 0 ? kProfDequant : kProfNesterov, e0, tr->ev(st), by + 1024.0 * bt.nseg});
    }
    CU(cudaGetLastError());
    return EMESH_OK;
}

int flat_grid(uint64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (n / 4 + kThreads - 1) / kThreads;
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * 8));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
// the quantizer moves 32-byte octets (256-bit loads) and 8-byte code words
bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

// Process-global workspace for the standalone codec entry points.
std::mutex g_codec_mu;
Workspace g_codec_ws;

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================

extern "C" {

const char* emesh_last_error(void) { return g_err.c_str(); }
int emesh_abi_version(void) { return 1; }

// ---------------- codec ----------------------------------------------------

int emesh_quantize_segments(const float* x, const uint64_t* seg_lo, const uint64_t* seg_len, uint32_t nseg,
                            uint8_t* codes, float* codebooks, double* stats, emesh_stream_t stream) {
    if (nseg == 0) return EMESH_OK;
    if (!aligned32(x) || (reinterpret_cast<uintptr_t>(codes) & 7u))
        return fail(EMESH_ESHAPE, "quantize: x must be 32-byte and codes 8-byte aligned");
    for (uint32_t i = 0; i < nseg; ++i)
        if (seg_len[i] == 0) return fail(EMESH_ESHAPE, "quantize: empty chunk");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> g(g_codec_mu);
    Plan p = make_list_plan(seg_lo, seg_len, nseg);
    TRY(g_codec_ws.reserve(p.max_slots, p.max_cta, p.max_segs));
    // stream-ordered tables + stats (freed in stream order)
    void* d_tables = nullptr;
    SegStat* d_stats = nullptr;
    CU(cudaMallocAsync(&d_tables, std::max<size_t>(p.host_tables.size(), 16), st));
    CU(cudaMallocAsync(reinterpret_cast<void**>(&d_stats), sizeof(SegStat) * nseg, st));
    CU(cudaMemcpyAsync(d_tables, p.host_tables.data(), p.host_tables.size(), cudaMemcpyHostToDevice, st));
    Batch& b = p.batches[0][0];
    b.bind(d_tables);
    QuantIO io{kSrcA, x, nullptr, nullptr, nullptr, 1.f, codes, codebooks, d_stats};
    TRY(launch_quant(b, g_codec_ws, io, st, &g_codec_tracker));
    if (stats)
        CU(cudaMemcpy2DAsync(stats, 4 * sizeof(double), d_stats, sizeof(SegStat), 4 * sizeof(double), nseg,
                             cudaMemcpyDeviceToDevice, st));
    // pageable host_tables: the H2D copy above completed synchronously
    CU(cudaFreeAsync(d_tables, st));
    CU(cudaFreeAsync(d_stats, st));
    return EMESH_OK;
}

int emesh_codec_check(emesh_stream_t stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CU(cudaStreamSynchronize(st));
    std::lock_guard<std::mutex> g(g_codec_mu);
    if (!g_codec_ws.err) return EMESH_OK;
    uint32_t e = 0;
    CU(cudaMemcpy(&e, g_codec_ws.err, sizeof e, cudaMemcpyDeviceToHost));
    if (e) {
        CU(cudaMemset(g_codec_ws.err, 0, sizeof(uint32_t)));
        return fail(EMESH_ENUMERIC, "quantize: non-finite input");
    }
    return EMESH_OK;
}

int emesh_quantize(const float* x, uint64_t n, uint8_t* codes, float* codebook, double* stats,
                   emesh_stream_t stream) {
    if (n == 0) return fail(EMESH_ESHAPE, "quantize: empty chunk");
    const uint64_t lo = 0;
    TRY(emesh_quantize_segments(x, &lo, &n, 1, codes, codebook, stats, stream));
    return emesh_codec_check(stream);
}

int emesh_dequantize_segments(const uint8_t* codes, const float* codebooks, const uint64_t* seg_lo,
                              const uint64_t* seg_len, uint32_t nseg, float* out, emesh_stream_t stream) {
    if (nseg == 0) return EMESH_OK;
    if (!aligned16(out) || (reinterpret_cast<uintptr_t>(codes) & 3u))
        return fail(EMESH_ESHAPE, "dequantize: out must be 16-byte and codes 4-byte aligned");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Plan p = make_list_plan(seg_lo, seg_len, nseg);
    void* d_tables = nullptr;
    CU(cudaMallocAsync(&d_tables, std::max<size_t>(p.host_tables.size(), 16), st));
    CU(cudaMemcpyAsync(d_tables, p.host_tables.data(), p.host_tables.size(), cudaMemcpyHostToDevice, st));
    Batch& b = p.batches[0][0];
    b.bind(d_tables);
    TRY(launch_apply(b, 0, codes, codebooks, nullptr, nullptr, nullptr, out, 0.f, 0.f, st, &g_codec_tracker));
    CU(cudaFreeAsync(d_tables, st));
    return EMESH_OK;
}

int emesh_dequantize(const uint8_t* codes, const float* codebook, uint64_t n, float* out, emesh_stream_t stream) {
    if (n == 0) return EMESH_OK;
    const uint64_t lo = 0;
    return emesh_dequantize_segments(codes, codebook, &lo, &n, 1, out, stream);
}

uint64_t emesh_encode_quant_chunk(const uint8_t* codes, const float* cb, uint32_t n, uint8_t* out) {
    uint8_t* p = out;
    for (int i = 0; i < 4; ++i) *p++ = (uint8_t)(n >> (8 * i));
    for (int b = 0; b < kBuckets; ++b) {
        uint32_t u;
        std::memcpy(&u, &cb[b], 4);
        for (int i = 0; i < 4; ++i) *p++ = (uint8_t)(u >> (8 * i));
    }
    if (n) std::memcpy(p, codes, n);
    return 4 + 4 * kBuckets + (uint64_t)n;
}

int emesh_decode_quant_chunk(const uint8_t* buf, uint64_t len, uint8_t* codes, float* cb, uint32_t* count) {
    if (len < 4) return fail(EMESH_EDECODE, "truncated buffer");
    const uint32_t c = (uint32_t)buf[0] | ((uint32_t)buf[1] << 8) | ((uint32_t)buf[2] << 16) | ((uint32_t)buf[3] << 24);
    if (len - 4 < 4u * kBuckets) return fail(EMESH_EDECODE, "truncated buffer");
    for (int b = 0; b < kBuckets; ++b) {
        const uint8_t* q = buf + 4 + 4 * b;
        const uint32_t u = (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16) | ((uint32_t)q[3] << 24);
        float v;
        std::memcpy(&v, &u, 4);
        if (!std::isfinite(v)) return fail(EMESH_EDECODE, "non-finite codebook entry");
        cb[b] = v;
    }
    if (len - 4 - 4u * kBuckets != c) return fail(EMESH_EDECODE, "quant chunk count does not match payload");
    if (c && codes) std::memcpy(codes, buf + 4 + 4 * kBuckets, c);
    *count = c;
    return EMESH_OK;
}

// ---------------- optimizer ----------------------------------------------

int emesh_pseudo_gradient(const float* prev, const float* local, float* delta, uint64_t n, emesh_stream_t stream) {
    if (n == 0) return EMESH_OK;
    if (!aligned16(prev) || !aligned16(local) || !aligned16(delta))
        return fail(EMESH_ESHAPE, "pseudo_gradient: arenas must be 16-byte aligned");
    k_pseudo_gradient<<<flat_grid(n), kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(prev, local, delta, n);
    ++g_codec_tracker.launches;
    CU(cudaGetLastError());
    return EMESH_OK;
}

int emesh_adamw_step(float* params, const float* grads, float* m, float* v, uint64_t n, uint64_t step,
                     float inner_lr, float lr_scale, float beta1, float beta2, float eps, float weight_decay,
                     uint32_t* err_flag, emesh_stream_t stream) {
    if (!(lr_scale >= 0.0f && lr_scale <= 1.0f)) return fail(EMESH_ECONFIG, "lr_scale must be in [0,1]");
    if (step == 0) return fail(EMESH_ECONFIG, "adamw: step counts from 1 (the state's step after the increment)");
    if (n == 0) return EMESH_OK;
    if (!aligned16(params) || !aligned16(grads) || !aligned16(m) || !aligned16(v))
        return fail(EMESH_ESHAPE, "adamw: arenas must be 16-byte aligned");
    AdamWArgs h;
    h.lr = inner_lr * lr_scale;  // optim.hpp:72
    h.lrwd = h.lr * weight_decay;
    h.b1 = beta1;
    h.omb1 = 1.0f - beta1;
    h.b2 = beta2;
    h.omb2 = 1.0f - beta2;
    h.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta1), static_cast<double>(step)));
    h.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta2), static_cast<double>(step)));
    h.eps = eps;
    k_adamw<<<flat_grid(n), kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(params, grads, m, v, n, h,
                                                                                 err_flag);
    ++g_codec_tracker.launches;
    CU(cudaGetLastError());
    return EMESH_OK;
}

int emesh_nesterov_outer_step(float* theta, const float* avg, float* buf, uint64_t n, float lr, float mom,
                              emesh_stream_t stream) {
    if (n == 0) return EMESH_OK;
    if (!aligned16(theta) || !aligned16(avg) || !aligned16(buf))
        return fail(EMESH_ESHAPE, "nesterov: arenas must be 16-byte aligned");
    k_nesterov_f32<<<flat_grid(n), kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(theta, avg, nullptr, buf,
                                                                                       nullptr, n, lr, mom);
    ++g_codec_tracker.launches;
    CU(cudaGetLastError());
    return EMESH_OK;
}

}  // extern "C"

// ===========================================================================
// Ring engine
// ===========================================================================

struct emesh_engine {
    emesh_engine_config cfg{};
    int device = 0;
    uint32_t k = 1, rank = 0, workers = 1;
    bool virt = false;
    Plan plan;
    Workspace ws;
    ncclComm_t comm = nullptr;
    cudaStream_t s_comp = nullptr, s_comm = nullptr;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // outer_sync_host's copy engines (created on first use)
    cudaEvent_t ev_entry = nullptr, ev_done = nullptr, ev_comm_done = nullptr;
    std::vector<cudaEvent_t> ev_send, ev_recv;  // per window
    std::vector<emesh_ring_op> schedule;        // NCCL mode program (build_schedule)
    // quantizer CTAs left out of the persistent grid for NCCL's send/recv kernels (NCCL transport;
    // leaving one CTA slot per SM measured the same at 4 GPUs)
    uint32_t reserve_sms = 8;
    struct Arena {
        uint8_t* codes = nullptr;
        float* cbs = nullptr;
        SegStat* stats = nullptr;
    };
    std::vector<Arena> arenas;  // per local worker
    // peer transport (EMESH_TRANSPORT_P2P): ring over peer memory mapped with
    // CUDA IPC; codes / codebooks double-buffered by round parity; arrival
    // flags hold the round (epoch) number, so they never need resetting
    int transport = EMESH_TRANSPORT_NCCL;
    // engine setup (communicator init, its first collectives' lazy connects)
    // may take seconds at 3+ ranks: waits then get at least this budget
    unsigned long long setup_floor_ns = 0;
    bool failed = false;             // a round failed (ring timeout / NCCL): abort, never wait for peers
    bool fp32 = false;               // ReduceMode::fp32 engine (raw fp32 payloads)
    std::vector<uint64_t> sizes;     // multi-tensor engine: one ReduceJob per tensor (config 5)
    std::vector<float*> pay;         // fp32 payload arenas, per local worker (parity 0 under P2P)
    float* pay_alt = nullptr;        // fp32 payload arena, parity 1 (P2P)
    uint32_t epoch = 0;
    uint8_t* codes_alt = nullptr;  // parity-1 codes arena (parity 0: arenas[0].codes)
    float* cbs_alt = nullptr;
    uint32_t* rs_flag = nullptr;  // [slot] reduce-scatter payload arrived (epoch)
    uint32_t* ag_flag = nullptr;  // [slot] owner's final payload arrived (epoch)
    struct Peer {
        uint8_t* codes[2] = {nullptr, nullptr};
        float* cbs[2] = {nullptr, nullptr};
        float* pay[2] = {nullptr, nullptr};
        uint32_t* rs_flag = nullptr;
        uint32_t* ag_flag = nullptr;
        ChunkHdr* hdr[2] = {nullptr, nullptr};  // ChunkMsg headers by slot, per round parity
        uint32_t* done = nullptr;              // [k] owners' done words
    };
    // round commit (peer transport): this rank's done source word, gate word, slot metadata
    ChunkHdr* hdr_alt = nullptr;  // parity-1 headers (parity 0: hdr0)
    ChunkHdr* hdr0 = nullptr;
    uint32_t* done = nullptr;     // [k] owners' done words (written by their final quantizers / copy engines); [63] waiting word
    uint32_t* done_src = nullptr; // this rank's done value (k_done_value)
    uint32_t* gate = nullptr;     // the gate word the decode kernels check (k_round_gate)
    uint2* meta = nullptr;        // by slot: {ring chunk, elements}
    // NCCL transport's gate: page-locked host word mapped into the device; the host sets it to
    // the round number when it enqueues a round and to 0 when it aborts the communicator
    volatile uint32_t* h_gate = nullptr;  // NCCL transport: kGateSlots page-locked gate words (one per round in flight)
    uint32_t* gate_dev = nullptr;         // ... and the device word the decodes read (copied once per round)
    uint32_t plan_epoch = 0;      // RingPlan epoch (ChunkMsg epoch)
    unsigned long long job = 0;   // ReduceJob id of the next round (ChunkMsg job)
    bool job_set = false;
    int32_t culprit = -1;         // failed rank reported by the last failed round (-1: unknown)
    std::vector<Peer> peers;  // [rank]; own rank: local pointers
    // device mirrors for the host-buffer entry point
    std::vector<float*> h_theta, h_local, h_buf;
    Tracker tr;
    uint32_t windows = 1;
};

namespace {

void teardown_p2p(emesh_engine* e);
const uint8_t* payload_codes(const emesh_engine* e, uint32_t w);
const float* payload_cbs(const emesh_engine* e, uint32_t w);

int engine_alloc(emesh_engine* e) {
    const uint64_t n = e->plan.n;
    const size_t nslots = e->plan.segs.size();
    e->arenas.resize(e->workers);
    for (auto& a : e->arenas) {
        CU(cudaMalloc(&a.codes, ((n + 15) & ~uint64_t(15)) + 16));
        CU(cudaMalloc(&a.cbs, nslots * kBuckets * sizeof(float)));
        CU(cudaMalloc(&a.stats, nslots * sizeof(SegStat)));
        CU(cudaMemset(a.stats, 0, nslots * sizeof(SegStat)));
    }
    if (e->fp32) {
        e->pay.assign(e->workers, nullptr);
        for (auto& p : e->pay) CU(cudaMalloc(&p, n * sizeof(float) + 16));
    }
    TRY(e->ws.reserve(e->plan.max_slots, e->plan.max_cta, e->plan.max_segs));
    return EMESH_OK;
}

// ---- ReduceMode::fp32 launchers (allreduce.hpp:120-164)
struct F32IO {
    const float* a;
    const float* b;       // PG: theta_l, else nullptr
    const float* in;      // incoming partial sums or nullptr
    bool div = false;     // owner mean
    float k = 1.f;
    uint32_t ndest = 0;
    float* dst[kMaxDest] = {};
    uint32_t nflags = 0;
    uint32_t* flags[kMaxDest] = {};
    const uint32_t* in_flag = nullptr;
    uint32_t epoch = 0;
    ChunkHdr* hdr_out[kMaxDest] = {};  // parallel to dst
    const ChunkHdr* in_hdr = nullptr;
    HdrRef hdr{};
    uint32_t phase_out = kPhaseRS;
    uint32_t culprit_in = kNoCulprit;
    uint32_t ndest_fail = 0;  // destinations still written after a failure (0: all; see QuantArgs::ndest_fail)
    uint32_t* wait_self = nullptr;
    const uint32_t* wait_pred = nullptr;
};

int launch_f32_hop(const Batch& bt, Workspace& ws, const F32IO& io, cudaStream_t st, Tracker* tr) {
    if (bt.ncta == 0) return EMESH_OK;
    F32HopArgs a{};
    a.segs = bt.d_segs;
    a.cta_seg = bt.d_cta_seg;
    a.a = io.a;
    a.b = io.b;
    a.in = io.in;
    a.divisor = io.k;
    int ex = 0;
    a.inv_divisor = std::frexp(io.k, &ex) == 0.5f ? std::ldexp(1.0f, 1 - ex) : 0.f;
    a.ndest = io.ndest;
    a.ndest_fail = io.ndest_fail ? std::min(io.ndest_fail, io.ndest) : io.ndest;
    for (uint32_t d = 0; d < io.ndest; ++d) a.dst[d] = io.dst[d];
    a.nflag = io.nflags;
    for (uint32_t f = 0; f < io.nflags; ++f) a.sflag[f] = io.flags[f];
    a.seg_done = ws.sync + kSyncReady;
    a.err = ws.err;
    a.in_flag = io.in_flag;
    a.epoch = io.epoch;
    a.timeout_ns = tr ? tr->timeout_ns : 30ull * 1000000000ull;
    a.nseg = bt.nseg;
    for (uint32_t d = 0; d < io.ndest; ++d) a.dhdr[d] = io.hdr_out[d];
    a.in_hdr = io.in_hdr;
    a.hdr = io.hdr;
    a.phase_out = (uint8_t)io.phase_out;
    a.culprit_in = io.culprit_in;
    a.wait_self = io.wait_self;
    a.wait_pred = io.wait_pred;
    if (io.nflags) CU(cudaMemsetAsync(ws.sync + kSyncReady, 0, (size_t)bt.nseg * sizeof(uint32_t), st));
    const bool prof = tr && tr->prof;
    cudaEvent_t e0 = prof ? tr->ev(st) : nullptr;
    a.upw = bt.upw;
    const dim3 g(bt.ncta * bt.upw), blk(kThreads);
    const bool pg = io.b != nullptr, hin = io.in != nullptr;
    if (!hin) {
        if (pg) k_f32_hop<true, false, false><<<g, blk, 0, st>>>(a);
        else k_f32_hop<false, false, false><<<g, blk, 0, st>>>(a);
    } else if (!io.div) {
        if (pg) k_f32_hop<true, true, false><<<g, blk, 0, st>>>(a);
        else k_f32_hop<false, true, false><<<g, blk, 0, st>>>(a);
    } else {
        if (pg) k_f32_hop<true, true, true><<<g, blk, 0, st>>>(a);
        else k_f32_hop<false, true, true><<<g, blk, 0, st>>>(a);
    }
    if (tr) tr->launches += 1;
    if (prof) {
        const double elems = (double)bt.elems;
        const double by = elems * (4.0 * (1 + (pg ? 1 : 0) + (hin ? 1 : 0)) + 4.0 * io.ndest);
        tr->recs.push_back({kProfF32Hop, e0, tr->ev(st), by});
    }
    CU(cudaGetLastError());
    return EMESH_OK;
}

int launch_f32_apply(const Batch& bt, int mode, const float* pay, float* theta, float* buf, float* theta_local,
                     float* out, float lr, float mom, cudaStream_t st, Tracker* tr, const uint32_t* gate = nullptr,
                     uint32_t epoch = 0) {
    if (bt.ncta == 0) return EMESH_OK;
    ApplyArgs a{};
    a.segs = bt.d_segs;
    a.cta_seg = bt.d_cta_seg;
    a.ncta = bt.ncta;
    a.theta = theta;
    a.buf = buf;
    a.theta_local = theta_local;
    a.out = out;
    a.lr = lr;
    a.mom = mom;
    a.gate = gate;
    a.epoch = epoch;
    a.upw = bt.upw;
    const dim3 g(bt.ncta * bt.upw), blk(kThreads);
    const bool prof = tr && tr->prof;
    cudaEvent_t e0 = prof ? tr->ev(st) : nullptr;
    if (mode == 0) k_f32_apply<0><<<g, blk, 0, st>>>(a, pay);
    else k_f32_apply<1><<<g, blk, 0, st>>>(a, pay);
    if (tr) tr->launches += 1;
    if (prof) {
        const double elems = (double)bt.elems;
        const double by = mode == 0 ? elems * 8.0 : elems * (theta_local ? 24.0 : 20.0);
        tr->recs.push_back({kProfF32Apply, e0, tr->ev(st), by});
    }
    CU(cudaGetLastError());
    return EMESH_OK;
}

// virtual ring, fp32 payloads (allreduce.hpp:411-464 with ReduceMode::fp32)
int run_virtual_f32(emesh_engine* e, const float* const* A, const float* const* B, float* const* theta,
                    float* const* buf, float* const* local_out, float* const* out, float lr, float mom) {
    const uint32_t k = e->k;
    cudaStream_t st = e->s_comp;
    const bool pg = B != nullptr;
    for (uint32_t w = 0; w < k; ++w)
        for (const Batch& bt : e->plan.batches[w]) {
            F32IO io{A[w], pg ? B[w] : nullptr, nullptr};
            io.ndest = 1;
            io.dst[0] = e->pay[w];
            TRY(launch_f32_hop(bt, e->ws, io, st, &e->tr));
        }
    for (uint32_t s = 0; s + 1 < k; ++s)
        for (uint32_t w = 0; w < k; ++w) {
            const uint32_t pred = (w + k - 1) % k, recv_c = (w + k - s - 1) % k;
            for (const Batch& bt : e->plan.batches[recv_c]) {
                F32IO io{A[w], pg ? B[w] : nullptr, e->pay[pred], s + 2 == k, (float)k};
                io.ndest = 1;
                io.dst[0] = e->pay[w];
                TRY(launch_f32_hop(bt, e->ws, io, st, &e->tr));
            }
        }
    for (uint32_t w = 0; w < k; ++w)
        for (uint32_t c = 0; c < k; ++c) {
            const uint32_t owner = (c + k - 1) % k;
            for (const Batch& bt : e->plan.batches[c])
                TRY(launch_f32_apply(bt, out ? 0 : 1, e->pay[owner], out ? nullptr : theta[w], out ? nullptr : buf[w],
                                     (!out && local_out) ? local_out[w] : nullptr, out ? out[w] : nullptr, lr, mom,
                                     st, &e->tr));
        }
    return EMESH_OK;
}

// Producer flags for reduce-scatter hop s of a k-ring (s == k-2 finalizes).
int hop_src(bool from_theta, uint32_t s, uint32_t k) {
    int src = (from_theta ? kSrcAminusB : kSrcA) | kHasIn;
    if (s + 2 == k) src |= kDivK;
    return src;
}

// ---- virtual ring: all k workers on this GPU, one stream, zero-copy hand-off
// (worker w reads its predecessor's payload arena in place of a recv).
// One chunk of the virtual ring: its RS chain (hop 0 on the worker that
// owns the chunk's first payload, then one requantizing hop per successor,
// allreduce.hpp:411-446); run_virtual_apply then has every worker decode the
// owner's final bytes (the all-gather is zero-copy here). Each chunk's chain only
// reads its own previous hop, so running the ring chunk-major is the same
// arithmetic as hop-major; it lets host copies of chunk c+1 overlap chunk c.
int run_virtual_chain(emesh_engine* e, uint32_t c, const float* const* A, const float* const* B) {
    const uint32_t k = e->k;
    cudaStream_t st = e->s_comp;
    const bool pg = B != nullptr;
    for (const Batch& bt : e->plan.batches[c]) {  // hop 0: Q(own chunk) on worker c (s = 0)
        QuantIO io{pg ? kSrcAminusB : kSrcA, A[c], pg ? B[c] : nullptr, nullptr, nullptr, 1.f,
                   e->arenas[c].codes, e->arenas[c].cbs, e->arenas[c].stats};
        TRY(launch_quant(bt, e->ws, io, st, &e->tr));
    }
    for (uint32_t s = 0; s + 1 < k; ++s) {  // hop s + 1: worker w receives chunk c from pred
        const uint32_t w = (c + s + 1) % k, pred = (w + k - 1) % k;
        for (const Batch& bt : e->plan.batches[c]) {
            QuantIO io{hop_src(pg, s, k), A[w], pg ? B[w] : nullptr, e->arenas[pred].codes, e->arenas[pred].cbs,
                       (float)k, e->arenas[w].codes, e->arenas[w].cbs, e->arenas[w].stats};
            TRY(launch_quant(bt, e->ws, io, st, &e->tr));
        }
    }
    return EMESH_OK;
}

// Worker w decodes the owner's final bytes of chunk c (+ Nesterov).
int run_virtual_apply(emesh_engine* e, uint32_t c, uint32_t w, float* const* theta, float* const* buf,
                      float* const* local_out, float* const* out, float lr, float mom, cudaStream_t st = nullptr) {
    const uint32_t owner = (c + e->k - 1) % e->k;
    if (!st) st = e->s_comp;
    for (const Batch& bt : e->plan.batches[c]) {
        if (out) {
            TRY(launch_apply(bt, 0, e->arenas[owner].codes, e->arenas[owner].cbs, nullptr, nullptr, nullptr, out[w],
                             0.f, 0.f, st, &e->tr));
        } else {
            TRY(launch_apply(bt, 1, e->arenas[owner].codes, e->arenas[owner].cbs, theta[w], buf[w],
                             local_out ? local_out[w] : nullptr, nullptr, lr, mom, st, &e->tr));
        }
    }
    return EMESH_OK;
}

int run_virtual(emesh_engine* e, const float* const* A, const float* const* B, float* const* theta, float* const* buf,
                float* const* local_out, float* const* out, float lr, float mom) {
    if (e->fp32) return run_virtual_f32(e, A, B, theta, buf, local_out, out, lr, mom);
    for (uint32_t c = 0; c < e->k; ++c) {
        TRY(run_virtual_chain(e, c, A, B));
        if (!out && e->k <= (uint32_t)kMaxDest) {  // one decode of the owner's payload for every local replica
            const uint32_t owner = (c + e->k - 1) % e->k;
            for (const Batch& bt : e->plan.batches[c])
                TRY(launch_apply_multi(bt, 1, e->arenas[owner].codes, e->arenas[owner].cbs, theta, buf, local_out,
                                       e->k, nullptr, lr, mom, e->s_comp, &e->tr));
            continue;
        }
        for (uint32_t w = 0; w < e->k; ++w) TRY(run_virtual_apply(e, c, w, theta, buf, local_out, out, lr, mom));
    }
    return EMESH_OK;
}

// ---- NCCL ring: this process is ring position `rank`; payload windows move
// with ncclSend/ncclRecv on s_comm while s_comp runs the fused hop kernels on
// the previous window.
//
// The communicator is non-blocking (ncclConfig_t::blocking = 0) so that no
// NCCL call can park the host forever on a peer that stopped (connection
// setup inside ncclGroupEnd does exactly that in blocking mode). Every call
// that may answer ncclInProgress is settled here against step_timeout; on
// expiry the communicator is aborted and the round fails with EMESH_ERING
// (allreduce.hpp:466-470), which allreduce_with_retry turns into a re-plan.
double wait_budget_ns(const emesh_engine* e) {
    return std::max((double)e->tr.timeout_ns, (double)e->setup_floor_ns);
}

// The NCCL transport's commit gates: page-locked host words the decode
// kernels read, one per round in flight (the host may enqueue later rounds
// before the GPU reaches this round's decodes). A failure closes all of them.
constexpr uint32_t kGateSlots = 256;
// The rank a timed-out NCCL wait can name: every receive of the ring is from
// the predecessor, but past k = 2 a blocked predecessor may itself be waiting
// on a dead rank further up (NCCL carries no abort frames, allreduce.hpp:341-359),
// so the culprit is known only with a single peer; -1 = unknown (the
// membership service's own failure detection evicts the dead rank).
int32_t nccl_suspect(const emesh_engine* e) {
    return e->k == 2 ? (int32_t)((e->rank + 1) % 2) : -1;
}
void close_nccl_gates(emesh_engine* e) {
    if (e->h_gate)
        for (uint32_t i = 0; i < kGateSlots; ++i) e->h_gate[i] = 0u;
}

int nccl_settle(emesh_engine* e, ncclResult_t r, const char* what) {
    const auto t0 = std::chrono::steady_clock::now();
    int spins = 0;
    while (r == ncclInProgress) {
        if (ncclCommGetAsyncError(e->comm, &r) != ncclSuccess) break;
        if (r != ncclInProgress) break;
        const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (waited * 1e9 > wait_budget_ns(e)) {
            e->failed = true;
            close_nccl_gates(e);  // nothing of this round may commit
            e->culprit = nccl_suspect(e);
            ncclCommAbort(e->comm);
            e->comm = nullptr;
            return fail(EMESH_ERING, "NCCL %s did not complete within step_timeout (%.1f s)", what,
                        wait_budget_ns(e) * 1e-9);
        }
        if (++spins > 1000) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    if (r != ncclSuccess) {
        e->failed = true;
        close_nccl_gates(e);
        e->culprit = nccl_suspect(e);
        ncclCommAbort(e->comm);
        e->comm = nullptr;
        return fail(EMESH_ENCCL, "NCCL %s: %s", what, ncclGetErrorString(r));
    }
    return EMESH_OK;
}
#define NCS(call) TRY(nccl_settle(e, (call), #call))

// Release the communicator: finalize (settled against step_timeout, so a
// vanished peer cannot park the host) then destroy; abort after a failure.
void nccl_close(emesh_engine* e) {
    if (!e->comm) return;
    if (!e->failed && nccl_settle(e, ncclCommFinalize(e->comm), "ncclCommFinalize") != EMESH_OK) return;
    if (e->failed) ncclCommAbort(e->comm);
    else ncclCommDestroy(e->comm);
    e->comm = nullptr;
}

// Wait for `streams` to drain while NCCL kernels may be parked on a peer:
// polled against step_timeout and the communicator's async error; on expiry
// or error the communicator is aborted (its kernels exit) -> EMESH_ERING.
int nccl_drain(emesh_engine* e, std::initializer_list<cudaStream_t> streams, const char* what) {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        bool done = true;
        for (cudaStream_t st : streams) {
            const cudaError_t q = cudaStreamQuery(st);
            if (q == cudaErrorNotReady) { done = false; continue; }
            if (q != cudaSuccess) return fail(EMESH_ECUDA, "%s: stream error: %s", what, cudaGetErrorString(q));
        }
        if (done) return EMESH_OK;
        ncclResult_t ae = ncclSuccess;
        if (e->comm) ncclCommGetAsyncError(e->comm, &ae);
        const bool err = ae != ncclSuccess && ae != ncclInProgress;
        const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (err || waited * 1e9 > wait_budget_ns(e)) {
            e->failed = true;
            close_nccl_gates(e);  // the decodes still queued behind the aborted transfers skip
            e->culprit = nccl_suspect(e);
            if (e->comm) ncclCommAbort(e->comm);
            e->comm = nullptr;
            for (cudaStream_t st : streams) cudaStreamSynchronize(st);
            cudaGetLastError();
            if (err) return fail(EMESH_ERING, "%s: NCCL ring failed: %s", what, ncclGetErrorString(ae));
            return fail(EMESH_ERING, "%s: NCCL ring step timed out (step_timeout %.1f s)", what,
                        wait_budget_ns(e) * 1e-9);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
}

int xfer_window(emesh_engine* e, const Batch& snd, const Batch& rcv) {
    const uint32_t k = e->k, r = e->rank;
    const int succ = (int)((r + 1) % k), pred = (int)((r + k - 1) % k);
    auto& ar = e->arenas[0];
    if (e->fp32) {  // raw fp32 partial sums / means (allreduce.hpp:120-151)
        NCS(ncclGroupStart());
        for (const auto& r : snd.eruns)
            NCS(ncclSend(e->pay[0] + r.first, r.second, ncclFloat32, succ, e->comm, e->s_comm));
        for (const auto& r : rcv.eruns)
            NCS(ncclRecv(e->pay[0] + r.first, r.second, ncclFloat32, pred, e->comm, e->s_comm));
        NCS(ncclGroupEnd());
        return EMESH_OK;
    }
    NCS(ncclGroupStart());
    for (const auto& r : snd.eruns) NCS(ncclSend(ar.codes + r.first, r.second, ncclUint8, succ, e->comm, e->s_comm));
    NCS(ncclSend(ar.cbs + (size_t)snd.slot0 * kBuckets, (size_t)snd.nseg * kBuckets, ncclFloat32, succ, e->comm,
                e->s_comm));
    for (const auto& r : rcv.eruns) NCS(ncclRecv(ar.codes + r.first, r.second, ncclUint8, pred, e->comm, e->s_comm));
    NCS(ncclRecv(ar.cbs + (size_t)rcv.slot0 * kBuckets, (size_t)rcv.nseg * kBuckets, ncclFloat32, pred, e->comm,
                e->s_comm));
    NCS(ncclGroupEnd());
    return EMESH_OK;

}

// All-gather of window j on the NCCL transport: every owner broadcasts its
// final window (k grouped in-place broadcasts; the bytes are the ones the
// reference's all-gather forwards hop by hop, allreduce.hpp:446-464). NCCL's
// collective kernels spread a broadcast over all channels, where a send/recv
// pair gets a couple per peer: the ring forwarding moved ~150 GB/s per
// window at 4 GPUs.
int bcast_window(emesh_engine* e, uint32_t j) {
    const uint32_t k = e->k;
    auto& ar = e->arenas[0];
    NCS(ncclGroupStart());
    for (uint32_t c = 0; c < k; ++c) {
        const Batch& b = e->plan.batches[c][j];
        const int root = (int)((c + k - 1) % k);  // owner of chunk c
        if (e->fp32) {
            for (const auto& ru : b.eruns)
                NCS(ncclBroadcast(e->pay[0] + ru.first, e->pay[0] + ru.first, ru.second, ncclFloat32, root, e->comm,
                                  e->s_comm));
        } else {
            for (const auto& ru : b.eruns)
                NCS(ncclBroadcast(ar.codes + ru.first, ar.codes + ru.first, ru.second, ncclUint8, root, e->comm,
                                  e->s_comm));
            float* cb = ar.cbs + (size_t)b.slot0 * kBuckets;
            NCS(ncclBroadcast(cb, cb, (size_t)b.nseg * kBuckets, ncclFloat32, root, e->comm, e->s_comm));
        }
    }
    NCS(ncclGroupEnd());
    return EMESH_OK;
}

// The NCCL ring's program for ring position r, in issue order (pure host
// logic, exported as emesh_ring_schedule so CPU tests can execute it):
//   OWN   : quantize the hop-0 payload Q(delta[chunk r]) window by window
//   XFER  : send window j of send_chunk to r+1, receive window j of recv_chunk from r-1
//   QUANT : fused hop on the received window (dequant + add + requant; /k on the last hop)
//   APPLY : decode a final window (dequant + Nesterov, or plain dequantize)
// Reduce-scatter: allreduce.hpp:411-426; owner finalize :428-445; all-gather :446-464.
std::vector<emesh_ring_op> build_schedule(const Plan& P, uint32_t r) {
    const uint32_t k = P.k;
    std::vector<emesh_ring_op> ops;
    auto win = [&](uint32_t c, uint32_t j) -> const Batch& { return P.batches[c][j]; };
    const uint32_t W = (uint32_t)P.batches[0].size();
    auto op = [&](int32_t kind, int32_t phase, int32_t hop, uint32_t j, int32_t sc, int32_t rc) {
        emesh_ring_op o{};
        o.kind = kind;
        o.phase = phase;
        o.hop = hop;
        o.window = (int32_t)j;
        o.send_chunk = sc;
        o.recv_chunk = rc;
        if (sc >= 0) { o.send_seg0 = win(sc, j).slot0; o.send_nseg = win(sc, j).nseg; }
        if (rc >= 0) { o.recv_seg0 = win(rc, j).slot0; o.recv_nseg = win(rc, j).nseg; }
        o.final_hop = (kind == EMESH_OP_QUANT && hop + 2 == (int32_t)k) ? 1 : 0;
        ops.push_back(o);
    };
    if (k < 2) return ops;
    for (uint32_t j = 0; j < W; ++j) op(EMESH_OP_OWN, 0, 0, j, -1, (int32_t)r);
    for (uint32_t s = 0; s + 1 < k; ++s) {
        const int32_t send_c = (int32_t)((r + k - s) % k), recv_c = (int32_t)((r + k - s - 1) % k);
        for (uint32_t j = 0; j < W; ++j) {
            op(EMESH_OP_XFER, 0, (int32_t)s, j, send_c, recv_c);
            op(EMESH_OP_QUANT, 0, (int32_t)s, j, -1, recv_c);
        }
    }
    // all-gather: forward the final bytes k-1 hops, THEN decode: a round commits (Nesterov writes
    // theta / momentum) only once every final payload arrived, so a failed round leaves the state
    // untouched for allreduce_with_retry (trainer.hpp:375-381 applies Nesterov after the all-reduce)
    const int32_t own = (int32_t)((r + 1) % k);
    for (uint32_t s = 0; s + 1 < k; ++s) {
        const int32_t send_c = (int32_t)((r + 1 + k - s) % k), recv_c = (int32_t)((r + k - s) % k);
        for (uint32_t j = 0; j < W; ++j) op(EMESH_OP_XFER, 1, (int32_t)s, j, send_c, recv_c);
    }
    for (uint32_t j = 0; j < W; ++j) op(EMESH_OP_APPLY, 1, -1, j, -1, own);
    for (uint32_t s = 0; s + 1 < k; ++s) {
        const int32_t recv_c = (int32_t)((r + k - s) % k);
        for (uint32_t j = 0; j < W; ++j) op(EMESH_OP_APPLY, 1, (int32_t)s, j, -1, recv_c);
    }
    return ops;
}

int run_nccl(emesh_engine* e, const float* A, const float* B, float* theta, float* buf, float* local_out, float* out,
             float lr, float mom) {
    const uint32_t k = e->k;
    const bool pg = B != nullptr;
    auto& ar = e->arenas[0];
    cudaStream_t sc = e->s_comp, sm = e->s_comm;
    if (!e->comm) return fail(EMESH_ERING, "NCCL communicator was aborted by an earlier ring failure");
    const uint32_t ep = ++e->epoch;
    // the decodes commit unless the host aborts the communicator (nccl_drain / nccl_settle):
    // this round's host gate word is copied to the device word the decodes read once every
    // all-gather transfer finished (or was aborted), one DMA per round
    volatile uint32_t* const h_gate = e->h_gate + ep % kGateSlots;
    *h_gate = ep;
    bool gate_loaded = false;
    const auto& P = e->plan.batches;
    const uint32_t W = (uint32_t)P[0].size();
    for (uint32_t c = 1; c < k; ++c)
        if (P[c].size() != W) return fail(EMESH_ECONFIG, "ring chunks have unequal window counts");
    for (const emesh_ring_op& o : e->schedule) {
        const uint32_t j = (uint32_t)o.window;
        // timeline (profiling only): events on the op's stream, after its waits
        cudaStream_t ost = o.kind == EMESH_OP_XFER ? sm : sc;
        if (e->tr.prof) {
            if (o.kind == EMESH_OP_XFER && (o.phase == 0 || o.hop == 0)) CU(cudaStreamWaitEvent(sm, e->ev_send[j], 0));
            if (o.kind == EMESH_OP_QUANT || (o.kind == EMESH_OP_APPLY && o.hop >= 0))
                CU(cudaStreamWaitEvent(sc, e->ev_recv[j], 0));
            e->tr.ops.push_back({o.kind, o.phase, o.hop, o.window, e->tr.ev(ost), nullptr});
        }
        switch (o.kind) {
            case EMESH_OP_OWN: {
                if (e->fp32) {
                    F32IO io{A, B, nullptr};
                    io.ndest = 1;
                    io.dst[0] = e->pay[0];
                    TRY(launch_f32_hop(P[o.recv_chunk][j], e->ws, io, sc, &e->tr));
                } else {
                    QuantIO io{pg ? kSrcAminusB : kSrcA, A, B, nullptr, nullptr, 1.f, ar.codes, ar.cbs, ar.stats};
                    TRY(launch_quant(P[o.recv_chunk][j], e->ws, io, sc, &e->tr, e->reserve_sms));
                }
                CU(cudaEventRecord(e->ev_send[j], sc));
                break;
            }
            case EMESH_OP_XFER:
                // RS: the payload was produced by compute (ev_send); AG hop 0
                // forwards the owner's final bytes, later AG hops bytes this
                // stream itself received
                if (o.phase == 0 || o.hop == 0) CU(cudaStreamWaitEvent(sm, e->ev_send[j], 0));
                if (o.phase == 1) {  // the schedule's k-1 forwarding hops as one broadcast group
                    if (o.hop == 0) TRY(bcast_window(e, j));
                    CU(cudaEventRecord(e->ev_recv[j], sm));
                    break;
                }
                TRY(xfer_window(e, P[o.send_chunk][j], P[o.recv_chunk][j]));
                CU(cudaEventRecord(e->ev_recv[j], sm));
                break;
            case EMESH_OP_QUANT: {
                CU(cudaStreamWaitEvent(sc, e->ev_recv[j], 0));
                if (e->fp32) {
                    F32IO io{A, B, e->pay[0], o.hop + 2 == (int32_t)k, (float)k};
                    io.ndest = 1;
                    io.dst[0] = e->pay[0];
                    TRY(launch_f32_hop(P[o.recv_chunk][j], e->ws, io, sc, &e->tr));
                } else {
                    QuantIO io{hop_src(pg, (uint32_t)o.hop, k), A, B, ar.codes, ar.cbs, (float)k, ar.codes, ar.cbs,
                               ar.stats};
                    TRY(launch_quant(P[o.recv_chunk][j], e->ws, io, sc, &e->tr, e->reserve_sms));
                }
                CU(cudaEventRecord(e->ev_send[j], sc));
                break;
            }
            case EMESH_OP_APPLY:
                // every decode (the own chunk's too) waits for the LAST all-gather
                // transfer: the comm stream is in order, so then every final payload
                // arrived, or the host aborted the communicator after closing the gate.
                // An apply that only followed the compute stream could commit the own
                // chunk while a peer's payload never comes (a late peer's buffered
                // reduce-scatter sends complete; its all-gather then times out).
                CU(cudaStreamWaitEvent(sc, e->ev_recv[W - 1], 0));
                if (!gate_loaded) {
                    CU(cudaMemcpyAsync(e->gate_dev, const_cast<const uint32_t*>(h_gate), sizeof(uint32_t),
                                       cudaMemcpyHostToDevice, sc));
                    gate_loaded = true;
                }
                if (e->fp32)
                    TRY(launch_f32_apply(P[o.recv_chunk][j], out ? 0 : 1, e->pay[0], theta, buf, local_out, out, lr, mom,
                                         sc, &e->tr, e->gate_dev, ep));
                else if (out)
                    TRY(launch_apply(P[o.recv_chunk][j], 0, ar.codes, ar.cbs, nullptr, nullptr, nullptr, out, 0.f, 0.f,
                                     sc, &e->tr, e->gate_dev, ep));
                else
                    TRY(launch_apply(P[o.recv_chunk][j], 1, ar.codes, ar.cbs, theta, buf, local_out, nullptr, lr, mom,
                                     sc, &e->tr, e->gate_dev, ep));
                break;
            default:
                return fail(EMESH_ECONFIG, "bad schedule op");
        }
        if (e->tr.prof) e->tr.ops.back().b = e->tr.ev(ost);
    }
    return EMESH_OK;
}

// Peer transport round (EMESH_TRANSPORT_P2P). Same ring as run_nccl
// (allreduce.hpp:411-464) with the transfers folded into the kernels: each
// quantizer launch stores its payload into the successor's arena (parity
// buffer of this round) and flags every finished segment there; the next
// hop's quantizer waits segment by segment. The owner's final payload goes
// to every rank at once, which replaces the all-gather's k-1 forwarding hops
// (the bytes are identical: AG forwards them verbatim, allreduce.hpp:446-464).
// The round's commit (peer transport), after this rank's last quantizer:
// this rank's done value (the round, or poison naming the culprit) reaches
// every peer — stored by the last CTA of the final quantizer (int8), or by
// k_done_value + copy-engine writes (fp32 mode, an empty final chunk);
// k_round_gate waits for every other owner's done word and final-payload
// flags, validates the final payloads' headers and publishes the gate word
// that every decode kernel of the round checks. A round that failed anywhere
// therefore commits nowhere (theta / momentum untouched) and every rank
// reports it.
int p2p_commit(emesh_engine* e, int par, uint32_t ep, bool done_sent) {
    const uint32_t k = e->k, r = e->rank, succ = (r + 1) % k;
    cudaStream_t sc = e->s_comp, cm = e->s_comm;
    if (!done_sent) {  // fp32 mode: a one-thread kernel + copy-engine writes of the done word
        k_done_value<<<1, 32, 0, sc>>>(e->ws.err, ep, e->done_src);
        e->tr.launches += 1;
        CU(cudaGetLastError());
        CU(cudaEventRecord(e->ev_send[0], sc));
        CU(cudaStreamWaitEvent(cm, e->ev_send[0], 0));
        for (uint32_t d = 1; d < k; ++d) {  // after the payload (stream order)
            const uint32_t q = (r + d) % k;
            CU(cudaMemcpyAsync(e->peers[q].done + r, e->done_src, sizeof(uint32_t), cudaMemcpyDeviceToDevice, cm));
        }
    }
    GateArgs g{};
    g.done = e->done;
    g.gate = e->gate;
    g.err = e->ws.err;
    g.hdr = e->peers[r].hdr[par];
    g.meta = e->meta;
    g.want = HdrRef{e->job, e->plan_epoch, (uint8_t)(e->fp32 ? 0 : 1)};
    g.k = k;
    g.rank = r;
    g.own_chunk = succ;
    g.nslots = (uint32_t)e->plan.segs.size();
    g.epoch = ep;
    g.timeout_ns = (unsigned long long)wait_budget_ns(e);
    g.ag_flag = e->ag_flag;
    k_round_gate<<<1, kThreads, 0, sc>>>(g);
    e->tr.launches += 1;
    CU(cudaGetLastError());
    return EMESH_OK;
}

HdrRef round_hdr(const emesh_engine* e) { return HdrRef{e->job, e->plan_epoch, (uint8_t)(e->fp32 ? 0 : 1)}; }

// ReduceMode::fp32 over the peer transport: the same ring with raw fp32
// partial sums stored into the successor's payload arena.
int run_p2p_f32(emesh_engine* e, const float* A, const float* B, float* theta, float* buf, float* local_out,
                float* out, float lr, float mom) {
    const uint32_t k = e->k, r = e->rank, succ = (r + 1) % k, pred = (r + k - 1) % k;
    const uint32_t ep = e->epoch;
    const int par = (int)(ep & 1u);
    cudaStream_t sc = e->s_comp;
    const auto& P = e->plan.batches;
    const HdrRef H = round_hdr(e);
    {
        F32IO io{A, B, nullptr};
        io.ndest = 1;
        io.dst[0] = e->peers[succ].pay[par];
        io.hdr_out[0] = e->peers[succ].hdr[par];
        io.nflags = 1;
        io.flags[0] = e->peers[succ].rs_flag;
        io.epoch = ep;
        io.hdr = H;
        TRY(launch_f32_hop(P[r][0], e->ws, io, sc, &e->tr));
    }
    for (uint32_t s = 0; s + 1 < k; ++s) {
        const uint32_t rc = (r + k - s - 1) % k;
        const bool fin = s + 2 == k;
        F32IO io{A, B, e->peers[r].pay[par], fin, (float)k};
        io.in_flag = e->rs_flag;
        io.in_hdr = e->peers[r].hdr[par];
        io.culprit_in = pred;
        io.wait_self = e->done + kWaitSlot;
        io.wait_pred = e->peers[pred].done + kWaitSlot;
        io.epoch = ep;
        io.hdr = H;
        io.ndest = 1;
        if (fin) {
            io.dst[0] = e->peers[r].pay[par];
            io.hdr_out[0] = e->peers[r].hdr[par];
            io.phase_out = kPhaseAG;
            io.ndest_fail = 1;  // a failed owner keeps its (garbage) final local
            for (uint32_t q = 0; q < k; ++q)
                if (q != r) {
                    io.hdr_out[io.ndest] = e->peers[q].hdr[par];
                    io.dst[io.ndest++] = e->peers[q].pay[par];
                    io.flags[io.nflags++] = e->peers[q].ag_flag;
                }
        } else {
            io.dst[0] = e->peers[succ].pay[par];
            io.hdr_out[0] = e->peers[succ].hdr[par];
            io.nflags = 1;
            io.flags[0] = e->peers[succ].rs_flag;
        }
        TRY(launch_f32_hop(P[rc][0], e->ws, io, sc, &e->tr));
    }
    TRY(p2p_commit(e, par, ep, false));
    if (e->plan.has_all)  // one decode launch over all segments
        return launch_f32_apply(e->plan.all, out ? 0 : 1, e->peers[r].pay[par], theta, buf, local_out, out, lr, mom,
                                sc, &e->tr, e->gate, ep);
    for (uint32_t d = 0; d < k; ++d) {
        const uint32_t c = (succ + k - d) % k;
        TRY(launch_f32_apply(P[c][0], out ? 0 : 1, e->peers[r].pay[par], theta, buf, local_out, out, lr, mom, sc,
                             &e->tr, e->gate, ep));
    }
    return EMESH_OK;
}

// Host-buffer pipelining hooks (outer_sync_host): called on the compute
// stream before chunk c's inputs are first read (RS), before its decode, and
// after its decode.
struct HostPipe {
    std::function<int(uint32_t)> before_rs, before_apply, after_apply;
};

int run_p2p(emesh_engine* e, const float* A, const float* B, float* theta, float* buf, float* local_out, float* out,
            float lr, float mom, const HostPipe* hp = nullptr) {
    if (e->failed) return fail(EMESH_ERING, "engine unusable after a failed round (rebuild it over the survivors)");
    const uint32_t ep = ++e->epoch;
    if (!e->job_set) e->job = ep;  // ReduceJob id of this round (ChunkMsg job): the round number by default
    e->job_set = false;
    if (e->fp32) return run_p2p_f32(e, A, B, theta, buf, local_out, out, lr, mom);
    const uint32_t k = e->k, r = e->rank, succ = (r + 1) % k, pred = (r + k - 1) % k;
    const bool pg = B != nullptr;
    const int par = (int)(ep & 1u);
    auto& ar = e->arenas[0];
    cudaStream_t sc = e->s_comp;
    const auto& P = e->plan.batches;
    const HdrRef H = round_hdr(e);
    for (uint32_t c = 0; c < k; ++c)
        if (P[c].size() != 1) return fail(EMESH_ECONFIG, "peer transport expects one batch per chunk");
    auto mark = [&](int kind, int hop, bool begin) {
        if (!e->tr.prof) return;
        if (begin) e->tr.ops.push_back({kind, kind == EMESH_OP_APPLY ? 1 : 0, hop, 0, e->tr.ev(sc), nullptr});
        else e->tr.ops.back().b = e->tr.ev(sc);
    };
    auto to_succ = [&](QuantIO& io) {
        io.local_out = false;
        io.nx = 1;
        io.x_codes[0] = e->peers[succ].codes[par];
        io.x_cb[0] = e->peers[succ].cbs[par];
        io.hdr_out[0] = e->peers[succ].hdr[par];
        io.nflags = 1;
        io.flags[0] = e->peers[succ].rs_flag;
    };
    {   // hop-0 payload Q(delta[chunk r]) -> successor
        QuantIO io{pg ? kSrcAminusB : kSrcA, A, B, nullptr, nullptr, 1.f, nullptr, nullptr, ar.stats};
        to_succ(io);
        io.epoch = ep;
        io.hdr = H;
        if (hp) TRY(hp->before_rs(r));
        mark(EMESH_OP_OWN, 0, true);
        TRY(launch_quant(P[r][0], e->ws, io, sc, &e->tr));
        mark(EMESH_OP_OWN, 0, false);
    }
    for (uint32_t s = 0; s + 1 < k; ++s) {
        const uint32_t rc = (r + k - s - 1) % k;
        QuantIO io{hop_src(pg, s, k), A, B, e->peers[r].codes[par], e->peers[r].cbs[par], (float)k,
                   e->peers[r].codes[par], e->peers[r].cbs[par], ar.stats};
        io.in_flag = e->rs_flag;
        io.in_hdr = e->peers[r].hdr[par];
        io.culprit_in = pred;
        io.wait_self = e->done + kWaitSlot;
        io.wait_pred = e->peers[pred].done + kWaitSlot;
        io.epoch = ep;
        io.hdr = H;
        if (s + 2 < k) {
            to_succ(io);
        } else {  // owner: the quantizer stores the final payload locally and into every other rank
            io.local_out = true;
            io.hdr_out[0] = e->peers[r].hdr[par];
            io.phase_out = kPhaseAG;
            for (uint32_t q = 0; q < k; ++q)
                if (q != r) {
                    io.x_codes[io.nx] = e->peers[q].codes[par];
                    io.x_cb[io.nx] = e->peers[q].cbs[par];
                    ++io.nx;
                    io.hdr_out[io.nx] = e->peers[q].hdr[par];
                    io.flags[io.nflags++] = e->peers[q].ag_flag;
                    if (P[rc][0].ncta)  // the commit's done word, from the kernel (an empty chunk runs none)
                        io.done_dst[io.ndone++] = e->peers[q].done + r;
                }
        }
        if (hp) TRY(hp->before_rs(rc));
        mark(EMESH_OP_QUANT, (int)s, true);
        TRY(launch_quant(P[rc][0], e->ws, io, sc, &e->tr));
        mark(EMESH_OP_QUANT, (int)s, false);
    }
    // all-gather (the owner's final bytes to every rank, allreduce.hpp:446-464 forwards the same
    // bytes hop by hop) + the commit gate
    mark(EMESH_OP_XFER, 0, true);  // the commit: the gate (timeline only)
    TRY(p2p_commit(e, par, ep, P[succ][0].ncta > 0));
    mark(EMESH_OP_XFER, 0, false);
    // decode every chunk, committing only through the gate: one launch over all segments (the
    // per-chunk launches cost ~10-25 us each at small sizes), per chunk when the host pipeline
    // copies chunks back as they finish (outer_sync_host)
    if (!hp && e->plan.has_all) {
        mark(EMESH_OP_APPLY, -1, true);
        if (out)
            TRY(launch_apply(e->plan.all, 0, e->peers[r].codes[par], e->peers[r].cbs[par], nullptr, nullptr, nullptr,
                             out, 0.f, 0.f, sc, &e->tr, e->gate, ep));
        else
            TRY(launch_apply(e->plan.all, 1, e->peers[r].codes[par], e->peers[r].cbs[par], theta, buf, local_out,
                             nullptr, lr, mom, sc, &e->tr, e->gate, ep));
        mark(EMESH_OP_APPLY, -1, false);
        return EMESH_OK;
    }
    for (uint32_t d = 0; d < k; ++d) {
        const uint32_t c = (succ + k - d) % k;  // succ = own chunk; then chunks owned by r-1, r-2, ...
        if (hp) TRY(hp->before_apply(c));
        mark(EMESH_OP_APPLY, (int)d - 1, true);
        if (out)
            TRY(launch_apply(P[c][0], 0, e->peers[r].codes[par], e->peers[r].cbs[par], nullptr, nullptr, nullptr, out,
                             0.f, 0.f, sc, &e->tr, e->gate, ep));
        else
            TRY(launch_apply(P[c][0], 1, e->peers[r].codes[par], e->peers[r].cbs[par], theta, buf, local_out, nullptr,
                             lr, mom, sc, &e->tr, e->gate, ep));
        mark(EMESH_OP_APPLY, (int)d - 1, false);
        if (hp) TRY(hp->after_apply(c));
    }
    return EMESH_OK;
}

// Map every rank's parity arenas, headers and flags (CUDA IPC handles
// all-gathered over the NCCL communicator, with each rank's plan epoch).
// Returns false (and leaves the engine on NCCL) unless every rank mapped
// every peer; sets *stale when a peer runs a newer plan epoch
// (StalePlanError, allreduce.hpp:272) or an older one (its ring attempt is
// stale: RingFailureError on this side).
bool setup_p2p(emesh_engine* e, int* stale) {
    const uint32_t k = e->k, r = e->rank;
    *stale = 0;
    if (k > (uint32_t)kMaxDest) return false;
    const uint64_t n = e->plan.n;
    const size_t nslots = e->plan.segs.size();
    bool ok = (!e->fp32 || cudaMalloc(&e->pay_alt, n * sizeof(float) + 16) == cudaSuccess) &&
              cudaMalloc(&e->codes_alt, ((n + 15) & ~uint64_t(15)) + 16) == cudaSuccess &&
              cudaMalloc(&e->cbs_alt, nslots * kBuckets * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&e->rs_flag, nslots * sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&e->ag_flag, nslots * sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&e->hdr0, nslots * sizeof(ChunkHdr)) == cudaSuccess &&
              cudaMalloc(&e->hdr_alt, nslots * sizeof(ChunkHdr)) == cudaSuccess &&
              cudaMalloc(&e->done, 64 * sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&e->done_src, 16 * sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&e->gate, 16 * sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&e->meta, nslots * sizeof(uint2)) == cudaSuccess &&
              cudaMemset(e->rs_flag, 0, nslots * sizeof(uint32_t)) == cudaSuccess &&
              cudaMemset(e->ag_flag, 0, nslots * sizeof(uint32_t)) == cudaSuccess &&
              cudaMemset(e->hdr0, 0, nslots * sizeof(ChunkHdr)) == cudaSuccess &&
              cudaMemset(e->hdr_alt, 0, nslots * sizeof(ChunkHdr)) == cudaSuccess &&
              cudaMemset(e->done, 0, 64 * sizeof(uint32_t)) == cudaSuccess &&
              cudaMemset(e->gate, 0, 16 * sizeof(uint32_t)) == cudaSuccess;
    if (ok) {  // by slot: {ring chunk, elements} (the gate's header checks)
        std::vector<uint2> meta(nslots);
        for (uint32_t c = 0; c < k; ++c)
            for (const Batch& bt : e->plan.batches[c])
                for (uint32_t s = bt.slot0; s < bt.slot0 + bt.nseg; ++s) meta[s] = make_uint2(c, (uint32_t)e->plan.segs[s].len);
        ok = cudaMemcpy(e->meta, meta.data(), nslots * sizeof(uint2), cudaMemcpyHostToDevice) == cudaSuccess;
    }
    constexpr int kH = 11;
    constexpr size_t kRec = kH * sizeof(cudaIpcMemHandle_t) + 64;  // + plan epoch
    std::vector<uint8_t> mine(kRec, 0), all(kRec * k, 0);
    void* bufs[kH] = {e->arenas[0].codes, e->codes_alt, e->arenas[0].cbs, e->cbs_alt, e->rs_flag, e->ag_flag,
                      e->hdr0, e->hdr_alt, e->done, e->fp32 ? e->pay[0] : nullptr, e->pay_alt};
    const int nh = e->fp32 ? 11 : 9;  // every rank runs the same mode
    for (int h = 0; ok && h < nh; ++h)
        ok = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(mine.data()) + h, bufs[h]) == cudaSuccess;
    std::memcpy(mine.data() + kH * sizeof(cudaIpcMemHandle_t), &e->plan_epoch, sizeof(uint32_t));
    // all-gather the handle records (and everyone's ok) over NCCL
    uint8_t* d = nullptr;
    int* d_ok = nullptr;
    bool comm_ok = cudaMalloc(&d, kRec * (k + 1)) == cudaSuccess && cudaMalloc(&d_ok, sizeof(int)) == cudaSuccess;
    if (comm_ok) {
        comm_ok = cudaMemcpy(d, mine.data(), kRec, cudaMemcpyHostToDevice) == cudaSuccess &&
                  nccl_settle(e, ncclAllGather(d, d + kRec, kRec, ncclUint8, e->comm, e->s_comm), "ncclAllGather") ==
                      EMESH_OK &&
                  cudaMemcpyAsync(all.data(), d + kRec, kRec * k, cudaMemcpyDeviceToHost, e->s_comm) == cudaSuccess &&
                  nccl_drain(e, {e->s_comm}, "p2p handle exchange") == EMESH_OK;
    }
    if (comm_ok)
        for (uint32_t q = 0; q < k; ++q) {
            uint32_t pe = 0;
            std::memcpy(&pe, all.data() + q * kRec + kH * sizeof(cudaIpcMemHandle_t), sizeof pe);
            if (pe > e->plan_epoch) *stale = 1;                     // this rank's plan is behind
            else if (pe < e->plan_epoch && *stale == 0) *stale = -1;  // a peer's plan is behind
        }
    e->peers.assign(k, emesh_engine::Peer{});
    {
        auto& me = e->peers[r];
        me.codes[0] = e->arenas[0].codes; me.codes[1] = e->codes_alt;
        me.cbs[0] = e->arenas[0].cbs; me.cbs[1] = e->cbs_alt;
        me.pay[0] = e->fp32 ? e->pay[0] : nullptr; me.pay[1] = e->pay_alt;
        me.rs_flag = e->rs_flag; me.ag_flag = e->ag_flag;
        me.hdr[0] = e->hdr0; me.hdr[1] = e->hdr_alt;
        me.done = e->done;
    }
    for (uint32_t q = 0; ok && comm_ok && q < k; ++q) {
        if (q == r) continue;
        void* ptr[kH] = {};
        for (int h = 0; h < nh && ok; ++h) {
            cudaIpcMemHandle_t hd;
            std::memcpy(&hd, all.data() + q * kRec + h * sizeof(cudaIpcMemHandle_t), sizeof hd);
            ok = cudaIpcOpenMemHandle(&ptr[h], hd, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
        }
        auto& pq = e->peers[q];
        pq.codes[0] = (uint8_t*)ptr[0]; pq.codes[1] = (uint8_t*)ptr[1];
        pq.cbs[0] = (float*)ptr[2]; pq.cbs[1] = (float*)ptr[3];
        pq.rs_flag = (uint32_t*)ptr[4]; pq.ag_flag = (uint32_t*)ptr[5];
        pq.hdr[0] = (ChunkHdr*)ptr[6]; pq.hdr[1] = (ChunkHdr*)ptr[7];
        pq.done = (uint32_t*)ptr[8];
        pq.pay[0] = (float*)ptr[9]; pq.pay[1] = (float*)ptr[10];
    }
    cudaGetLastError();  // clear a failed open, if any
    // agree: every rank must have mapped every peer
    int v = (ok && comm_ok) ? 1 : 0;
    bool agreed = false;
    if (d_ok && cudaMemcpy(d_ok, &v, sizeof v, cudaMemcpyHostToDevice) == cudaSuccess &&
        nccl_settle(e, ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, e->comm, e->s_comm), "ncclAllReduce") ==
            EMESH_OK &&
        cudaMemcpyAsync(&v, d_ok, sizeof v, cudaMemcpyDeviceToHost, e->s_comm) == cudaSuccess &&
        nccl_drain(e, {e->s_comm}, "p2p mapping agreement") == EMESH_OK)
        agreed = v == 1;
    cudaFree(d);
    cudaFree(d_ok);
    if (!agreed) teardown_p2p(e);
    return agreed;
}

void teardown_p2p(emesh_engine* e) {
    for (uint32_t q = 0; q < e->peers.size(); ++q) {
        if (q == e->rank) continue;
        auto& pq = e->peers[q];
        void* ptrs[] = {pq.codes[0], pq.codes[1], pq.cbs[0], pq.cbs[1], pq.rs_flag, pq.ag_flag,
                        pq.hdr[0], pq.hdr[1], pq.done, pq.pay[0], pq.pay[1]};
        for (void* p : ptrs)
            if (p) cudaIpcCloseMemHandle(p);
    }
    e->peers.clear();
    void* own[] = {e->codes_alt, e->cbs_alt, e->pay_alt, e->rs_flag, e->ag_flag, e->hdr0, e->hdr_alt,
                   e->done, e->done_src, e->gate, e->meta};
    for (void* p : own)
        if (p) cudaFree(p);
    e->codes_alt = nullptr;
    e->cbs_alt = nullptr;
    e->pay_alt = nullptr;
    e->rs_flag = e->ag_flag = nullptr;
    e->hdr0 = e->hdr_alt = nullptr;
    e->done = e->done_src = e->gate = nullptr;
    e->meta = nullptr;
    cudaGetLastError();
}

const uint8_t* payload_codes(const emesh_engine* e, uint32_t w) {
    return (e->transport == EMESH_TRANSPORT_P2P && (e->epoch & 1u)) ? e->codes_alt : e->arenas[w].codes;
}
const float* payload_cbs(const emesh_engine* e, uint32_t w) {
    return (e->transport == EMESH_TRANSPORT_P2P && (e->epoch & 1u)) ? e->cbs_alt : e->arenas[w].cbs;
}

int engine_enter(emesh_engine* e, cudaStream_t user) {
    CU(cudaSetDevice(e->device));
    CU(cudaEventRecord(e->ev_entry, user));
    CU(cudaStreamWaitEvent(e->s_comp, e->ev_entry, 0));
    CU(cudaStreamWaitEvent(e->s_comm, e->ev_entry, 0));
    return EMESH_OK;
}

int engine_exit(emesh_engine* e, cudaStream_t user) {
    CU(cudaEventRecord(e->ev_comm_done, e->s_comm));
    CU(cudaStreamWaitEvent(e->s_comp, e->ev_comm_done, 0));
    CU(cudaEventRecord(e->ev_done, e->s_comp));
    CU(cudaStreamWaitEvent(user, e->ev_done, 0));
    return EMESH_OK;
}

}  // namespace

extern "C" {

uint64_t emesh_plan_segments(uint64_t n, uint32_t k, uint32_t S, uint64_t* seg_lo, uint64_t* seg_len) {
    if (k == 0) return 0;
    Plan p = make_ring_plan(n, k, S ? S : 4, (uint64_t)1 << 62);
    for (size_t i = 0; i < p.segs.size(); ++i) {
        if (seg_lo) seg_lo[i] = p.segs[i].lo;
        if (seg_len) seg_len[i] = p.segs[i].len;
    }
    return p.segs.size();
}

uint64_t emesh_plan_tensor_segments(const uint64_t* sizes, uint32_t nt, uint32_t k, uint32_t S, uint64_t* seg_lo,
                                    uint64_t* seg_len) {
    if (k == 0 || (nt && !sizes)) return 0;
    Plan p = make_tensor_ring_plan(sizes, nt, k, S ? S : 4, (uint64_t)1 << 62);
    for (size_t i = 0; i < p.segs.size(); ++i) {
        if (seg_lo) seg_lo[i] = p.segs[i].lo;
        if (seg_len) seg_len[i] = p.segs[i].len;
    }
    return p.segs.size();
}

uint64_t emesh_ring_schedule(uint64_t n, uint32_t k, uint32_t S, uint64_t window_elems, uint32_t rank,
                             emesh_ring_op* ops, uint64_t max_ops) {
    if (k == 0 || rank >= k) return 0;
    Plan p = make_ring_plan(n, k, S ? S : 4, window_elems ? window_elems : kDefaultWindow);
    std::vector<emesh_ring_op> v = build_schedule(p, rank);
    if (ops)
        for (size_t i = 0; i < v.size() && i < max_ops; ++i) ops[i] = v[i];
    return v.size();
}

int emesh_nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return EMESH_OK;
}

int emesh_engine_create(const emesh_engine_config* cfg, emesh_engine** out) {
    if (!cfg || !out) return fail(EMESH_ECONFIG, "null argument");
    if (cfg->k == 0) return fail(EMESH_ESHAPE, "empty ring");
    const uint32_t S = cfg->pipeline_subchunks ? cfg->pipeline_subchunks : 4;
    const bool virt = cfg->virtual_workers > 1 || cfg->k == 1;
    if (cfg->virtual_workers > 1 && cfg->virtual_workers != cfg->k)
        return fail(EMESH_ECONFIG, "virtual_workers must be 0/1 or equal k");
    if (!virt && cfg->rank >= cfg->k) return fail(EMESH_ECONFIG, "rank out of range");
    if (!virt && !cfg->nccl_id) return fail(EMESH_ECONFIG, "NCCL mode needs nccl_id");
    auto* e = new emesh_engine();
    e->cfg = *cfg;
    e->k = cfg->k;
    e->rank = virt ? 0 : cfg->rank;
    e->virt = virt;
    e->workers = virt ? cfg->k : 1;
    if (cfg->device >= 0) e->device = cfg->device;
    else cudaGetDevice(&e->device);
    auto bail = [&](int rc) { emesh_engine_destroy(e); return rc; };
    if (cudaSetDevice(e->device) != cudaSuccess) return bail(fail(EMESH_ECUDA, "cudaSetDevice"));
    // default window: a whole chunk for the virtual ring (nothing to overlap
    // with, and the persistent quantizer pipelines stats and bins across the
    // segments of a batch); a quarter chunk (>= 16M) under NCCL so transfers
    // of window j+1 overlap the kernels of window j
    if (cfg->transport > EMESH_TRANSPORT_P2P) return bail(fail(EMESH_ECONFIG, "unknown transport %u", cfg->transport));
    if (cfg->reduce_fp32 > 1) return bail(fail(EMESH_ECONFIG, "reduce_fp32 must be 0 or 1"));
    e->fp32 = cfg->reduce_fp32 == 1;
    const uint64_t chunk = (cfg->n + cfg->k - 1) / cfg->k;
    // the peer transport synchronizes per segment: one batch per chunk
    const bool try_p2p = !virt && cfg->k > 1 && cfg->transport != EMESH_TRANSPORT_NCCL;
    const uint64_t nccl_window = cfg->window_elems ? cfg->window_elems : std::max<uint64_t>(chunk / 4, kDefaultWindow);
    uint64_t window = (virt || try_p2p) ? ~uint64_t(0) >> 2 : nccl_window;  // whole chunks
    if (cfg->ntensors) {
        if (!cfg->tensor_numel) return bail(fail(EMESH_ECONFIG, "tensor_numel is NULL"));
        uint64_t tot = 0;
        for (uint32_t t = 0; t < cfg->ntensors; ++t) tot += cfg->tensor_numel[t];
        if (tot != cfg->n) return bail(fail(EMESH_ESHAPE, "tensor sizes sum to %llu, n = %llu",
                                            (unsigned long long)tot, (unsigned long long)cfg->n));
        e->sizes.assign(cfg->tensor_numel, cfg->tensor_numel + cfg->ntensors);
    }
    auto mkplan = [&](uint64_t win) {
        return e->sizes.empty() ? make_ring_plan(cfg->n, cfg->k, S, win)
                                : make_tensor_ring_plan(e->sizes.data(), (uint32_t)e->sizes.size(), cfg->k, S, win);
    };
    e->plan = mkplan(window);
    e->windows = (uint32_t)e->plan.batches[0].size();
    int rc = e->plan.upload();
    if (rc) return bail(rc);
    if (e->k > 1 && (rc = engine_alloc(e))) return bail(rc);
    e->tr.err = e->ws.err;
    if (cfg->step_timeout_s > 0) e->tr.timeout_ns = (unsigned long long)(cfg->step_timeout_s * 1e9);
    e->plan_epoch = cfg->plan_epoch;
    // setup waits (communicator init, the first round's lazy NCCL connects) get at least 30 s;
    // the floor is dropped once a round has drained successfully (emesh_engine_check)
    e->setup_floor_ns = 30ull * 1000000000ull;
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if (cudaStreamCreateWithPriority(&e->s_comp, cudaStreamNonBlocking, lo_prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&e->s_comm, cudaStreamNonBlocking, hi_prio) != cudaSuccess)
        return bail(fail(EMESH_ECUDA, "stream create"));
    cudaEventCreateWithFlags(&e->ev_entry, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e->ev_done, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e->ev_comm_done, cudaEventDisableTiming);
    e->ev_send.resize(e->windows);
    e->ev_recv.resize(e->windows);
    for (uint32_t j = 0; j < e->windows; ++j) {
        cudaEventCreateWithFlags(&e->ev_send[j], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e->ev_recv[j], cudaEventDisableTiming);
    }
    if (!virt && e->k > 1) {
        {   // the NCCL transport's commit gates: page-locked host words (see run_nccl)
            void* h = nullptr;
            if (cudaHostAlloc(&h, kGateSlots * sizeof(uint32_t), cudaHostAllocDefault) != cudaSuccess ||
                cudaMalloc(&e->gate_dev, sizeof(uint32_t)) != cudaSuccess)
                return bail(fail(EMESH_ECUDA, "gate word allocation"));
            e->h_gate = static_cast<volatile uint32_t*>(h);
            close_nccl_gates(e);
        }
        e->schedule = build_schedule(e->plan, e->rank);
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_id, sizeof id);
        ncclConfig_t ncfg = NCCL_CONFIG_INITIALIZER;
        ncfg.blocking = 0;  // every wait is bounded by step_timeout (nccl_settle)
        ncclResult_t r = ncclCommInitRankConfig(&e->comm, (int)e->k, id, (int)e->rank, &ncfg);
        if (r != ncclSuccess && r != ncclInProgress)
            return bail(fail(EMESH_ENCCL, "ncclCommInitRankConfig: %s", ncclGetErrorString(r)));
        if ((rc = nccl_settle(e, r, "ncclCommInitRankConfig"))) return bail(rc);
        e->transport = EMESH_TRANSPORT_NCCL;
        int stale = 0;
        const bool mapped = try_p2p && setup_p2p(e, &stale);
        if (stale) {  // the ranks disagree on the plan epoch (allreduce.hpp:272)
            if (mapped) teardown_p2p(e);
            e->failed = true;
            if (stale > 0) return bail(fail(EMESH_ESTALE, "a ring peer runs a newer plan epoch"));
            return bail(fail(EMESH_ERING, "a ring peer runs an older plan epoch (stale attempt)"));
        }
        if (mapped) {
            e->transport = EMESH_TRANSPORT_P2P;
            // NCCL only bootstrapped the mappings: release it now, while every
            // rank is here, so teardown never depends on a peer being alive
            nccl_close(e);
        } else if (!e->comm) {  // a peer vanished during setup (nccl_settle / nccl_drain aborted)
            const std::string why = emesh_last_error();
            return bail(fail(EMESH_ERING, "ring setup failed: %s", why.c_str()));
        } else if (cfg->transport == EMESH_TRANSPORT_P2P) {
            return bail(fail(EMESH_ECONFIG, "peer transport unavailable (CUDA IPC mapping failed on some rank)"));
        } else if (try_p2p) {  // AUTO fell back: NCCL windows
            e->plan.release();
            e->plan = mkplan(nccl_window);
            e->windows = (uint32_t)e->plan.batches[0].size();
            if ((rc = e->plan.upload()) || (rc = e->ws.reserve(e->plan.max_slots, e->plan.max_cta, e->plan.max_segs)))
                return bail(rc);
            e->schedule = build_schedule(e->plan, e->rank);
            for (auto ev : e->ev_send) cudaEventDestroy(ev);
            for (auto ev : e->ev_recv) cudaEventDestroy(ev);
            e->ev_send.assign(e->windows, nullptr);
            e->ev_recv.assign(e->windows, nullptr);
            for (uint32_t j = 0; j < e->windows; ++j) {
                cudaEventCreateWithFlags(&e->ev_send[j], cudaEventDisableTiming);
                cudaEventCreateWithFlags(&e->ev_recv[j], cudaEventDisableTiming);
            }
        }
    }
    *out = e;
    return EMESH_OK;
}

int emesh_engine_destroy(emesh_engine* e) {
    if (!e) return EMESH_OK;
    cudaSetDevice(e->device);
    if (e->comm && e->s_comp && e->s_comm && nccl_drain(e, {e->s_comp, e->s_comm}, "destroy") != EMESH_OK)
        cudaGetLastError();  // NCCL kernels parked on a vanished peer: aborted by nccl_drain
    if (e->s_comp) cudaStreamSynchronize(e->s_comp);
    if (e->s_comm) cudaStreamSynchronize(e->s_comm);
    teardown_p2p(e);
    nccl_close(e);  // aborts when a round failed: peers may be gone
    for (auto& a : e->arenas) { cudaFree(a.codes); cudaFree(a.cbs); cudaFree(a.stats); }
    if (e->h_gate) cudaFreeHost(const_cast<uint32_t*>(e->h_gate));
    if (e->gate_dev) cudaFree(e->gate_dev);
    for (auto* p : e->pay) cudaFree(p);
    for (auto* p : e->h_theta) cudaFree(p);
    for (auto* p : e->h_local) cudaFree(p);
    for (auto* p : e->h_buf) cudaFree(p);
    e->ws.release();
    e->plan.release();
    e->tr.release();
    for (auto ev : e->ev_send) cudaEventDestroy(ev);
    for (auto ev : e->ev_recv) cudaEventDestroy(ev);
    if (e->ev_entry) cudaEventDestroy(e->ev_entry);
    if (e->ev_done) cudaEventDestroy(e->ev_done);
    if (e->ev_comm_done) cudaEventDestroy(e->ev_comm_done);
    if (e->s_h2d) { cudaStreamSynchronize(e->s_h2d); cudaStreamDestroy(e->s_h2d); }
    if (e->s_d2h) { cudaStreamSynchronize(e->s_d2h); cudaStreamDestroy(e->s_d2h); }
    if (e->s_comp) cudaStreamDestroy(e->s_comp);
    if (e->s_comm) cudaStreamDestroy(e->s_comm);
    delete e;
    return EMESH_OK;
}

uint64_t emesh_engine_segments(const emesh_engine* e, uint64_t* lo, uint64_t* len) {
    const auto& s = e->plan.segs;
    for (size_t i = 0; i < s.size(); ++i) {
        if (lo) lo[i] = s[i].lo;
        if (len) len[i] = s[i].len;
    }
    return s.size();
}

uint64_t emesh_engine_launches(const emesh_engine* e) { return e->tr.launches; }

int emesh_engine_transport(const emesh_engine* e) { return (e && !e->virt && e->k > 1) ? e->transport : 0; }

int emesh_engine_profile(emesh_engine* e, int enable) {
    CU(cudaSetDevice(e->device));
    CU(cudaStreamSynchronize(e->s_comp));
    e->tr.reset();
    e->tr.prof = enable != 0;
    return EMESH_OK;
}

uint64_t emesh_engine_timeline(emesh_engine* e, double* rows, uint64_t max_rows) {
    if (!e) return 0;
    if (cudaSetDevice(e->device) != cudaSuccess || cudaStreamSynchronize(e->s_comp) != cudaSuccess ||
        cudaStreamSynchronize(e->s_comm) != cudaSuccess)
        return 0;
    const auto& v = e->tr.ops;
    for (size_t i = 0; i < v.size() && i < max_rows; ++i) {
        float t0 = 0.f, t1 = 0.f;
        cudaEventElapsedTime(&t0, v[0].a, v[i].a);
        cudaEventElapsedTime(&t1, v[0].a, v[i].b);
        double* r = rows + 6 * i;
        r[0] = v[i].kind; r[1] = v[i].phase; r[2] = v[i].hop; r[3] = v[i].window; r[4] = t0; r[5] = t1;
    }
    return v.size();
}

int emesh_engine_profile_read(emesh_engine* e, uint32_t kind, uint64_t* count, double* ms, double* bytes) {
    CU(cudaSetDevice(e->device));
    CU(cudaStreamSynchronize(e->s_comp));
    CU(cudaStreamSynchronize(e->s_comm));
    uint64_t c = 0;
    double t = 0, b = 0;
    for (const auto& r : e->tr.recs) {
        if ((uint32_t)r.kind != kind) continue;
        float x = 0.f;
        CU(cudaEventElapsedTime(&x, r.a, r.b));
        ++c;
        t += x;
        b += r.bytes;
    }
    if (count) *count = c;
    if (ms) *ms = t;
    if (bytes) *bytes = b;
    return EMESH_OK;
}

int emesh_engine_ring_allreduce(emesh_engine* e, const float* const* input, float* const* output,
                                emesh_stream_t stream) {
    cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
    for (uint32_t w = 0; w < e->workers; ++w)
        if (!aligned32(input[w]) || !aligned16(output[w])) return fail(EMESH_ESHAPE, "arenas must be 32-byte aligned");
    TRY(engine_enter(e, user));
    if (e->k == 1) {
        // allreduce.hpp:319: identity, zero communication
        CU(cudaMemcpyAsync(output[0], input[0], e->plan.n * sizeof(float), cudaMemcpyDeviceToDevice, e->s_comp));
    } else if (e->virt) {
        TRY(run_virtual(e, input, nullptr, nullptr, nullptr, nullptr, output, 0.f, 0.f));
    } else if (e->transport == EMESH_TRANSPORT_P2P) {
        TRY(run_p2p(e, input[0], nullptr, nullptr, nullptr, nullptr, output[0], 0.f, 0.f));
    } else {
        TRY(run_nccl(e, input[0], nullptr, nullptr, nullptr, nullptr, output[0], 0.f, 0.f));
    }
    return engine_exit(e, user);
}

int emesh_engine_outer_sync(emesh_engine* e, float* const* theta_g, float* const* theta_l, float* const* buf,
                            float lr, float mom, int write_local, emesh_stream_t stream) {
    cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
    for (uint32_t w = 0; w < e->workers; ++w)
        if (!aligned32(theta_g[w]) || !aligned32(theta_l[w]) || !aligned16(buf[w]))
            return fail(EMESH_ESHAPE, "arenas must be 32-byte aligned");
    TRY(engine_enter(e, user));
    if (e->k == 1) {
        // k == 1: avg = delta exactly (allreduce.hpp:319); PG + Nesterov fused, 20 B/param
        const uint64_t n = e->plan.n;
        cudaEvent_t e0 = e->tr.prof ? e->tr.ev(e->s_comp) : nullptr;
        k_nesterov_f32<<<flat_grid(n), kThreads, 0, e->s_comp>>>(theta_g[0], nullptr, theta_l[0], buf[0],
                                                                 write_local ? theta_l[0] : nullptr, n, lr, mom);
        if (e->tr.prof)
            e->tr.recs.push_back({kProfFusedK1, e0, e->tr.ev(e->s_comp), (double)n * (write_local ? 24.0 : 20.0)});
        e->tr.launches += 1;
        CU(cudaGetLastError());
    } else if (e->virt) {
        TRY(run_virtual(e, (const float* const*)theta_g, (const float* const*)theta_l, theta_g, buf,
                        write_local ? theta_l : nullptr, nullptr, lr, mom));
    } else if (e->transport == EMESH_TRANSPORT_P2P) {
        TRY(run_p2p(e, theta_g[0], theta_l[0], theta_g[0], buf[0], write_local ? theta_l[0] : nullptr, nullptr, lr,
                    mom));
    } else {
        TRY(run_nccl(e, theta_g[0], theta_l[0], theta_g[0], buf[0], write_local ? theta_l[0] : nullptr, nullptr, lr,
                     mom));
    }
    return engine_exit(e, user);
}

// Host-buffer outer sync on k virtual workers, pipelined by chunk: the
// inputs of chunk c (every worker's theta_g, theta_l, momentum over the
// chunk's element runs) go up on one copy stream, the ring of chunk c runs
// as soon as they landed, and its outputs come back on a second copy stream
// while later chunks are still uploading — PCIe is full duplex, so the
// round costs about max(upload, download) instead of their sum.
static int outer_sync_host_pipelined(emesh_engine* e, float* const* theta_g, float* const* theta_l, float* const* buf,
                              float lr, float mom, int write_local) {
    const uint32_t k = e->k;
    if (!e->s_h2d) CU(cudaStreamCreateWithFlags(&e->s_h2d, cudaStreamNonBlocking));
    if (!e->s_d2h) CU(cudaStreamCreateWithFlags(&e->s_d2h, cudaStreamNonBlocking));
    // ev[c]: chunk c's theta_g / theta_l of every worker landed; ev[k + c*k + w]:
    // worker w's momentum of chunk c landed; ev[k + k*k + c*k + w]: its outputs are final
    std::vector<cudaEvent_t> ev(k + 2 * k * k, nullptr);
    for (auto& x : ev) CU(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    auto ev_theta = [&](uint32_t c) { return ev[c]; };
    auto ev_buf = [&](uint32_t c, uint32_t w) { return ev[k + c * k + w]; };
    auto ev_out = [&](uint32_t c, uint32_t w) { return ev[k + k * k + c * k + w]; };
    int rc = EMESH_OK;
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> runs(k);
    for (uint32_t c = 0; c < k; ++c)  // the chunk's contiguous element runs, adjacent ones merged
        for (const Batch& bt : e->plan.batches[c])
            for (const auto& x : bt.eruns) {
                auto& r = runs[c];
                if (!r.empty() && r.back().first + r.back().second == x.first) r.back().second += x.second;
                else if (x.second) r.push_back(x);
            }
    auto copy = [&](float* dst, const float* src, uint32_t c, cudaMemcpyKind kind, cudaStream_t st) {
        for (const auto& x : runs[c])
            if (cudaMemcpyAsync(dst + x.first, src + x.first, x.second * sizeof(float), kind, st) != cudaSuccess)
                return fail(EMESH_ECUDA, "outer_sync_host: %s", cudaGetErrorString(cudaGetLastError()));
        return (int)EMESH_OK;
    };
    auto record = [&](cudaEvent_t x, cudaStream_t st) {
        return cudaEventRecord(x, st) == cudaSuccess ? (int)EMESH_OK : fail(EMESH_ECUDA, "event record");
    };
    auto wait = [&](cudaStream_t st, cudaEvent_t x) {
        return cudaStreamWaitEvent(st, x, 0) == cudaSuccess ? (int)EMESH_OK : fail(EMESH_ECUDA, "stream wait");
    };
    // uploads in need order: the chunk's theta_g / theta_l (its RS chain), then its momentum worker by
    // worker (each worker's decode + Nesterov), so the last bytes up gate only one worker's last decode
    for (uint32_t c = 0; c < k && !rc; ++c) {
        for (uint32_t w = 0; w < k && !rc; ++w) {
            rc = copy(e->h_theta[w], theta_g[w], c, cudaMemcpyHostToDevice, e->s_h2d);
            if (!rc) rc = copy(e->h_local[w], theta_l[w], c, cudaMemcpyHostToDevice, e->s_h2d);
        }
        if (!rc) rc = record(ev_theta(c), e->s_h2d);
        for (uint32_t w = 0; w < k && !rc; ++w) {
            rc = copy(e->h_buf[w], buf[w], c, cudaMemcpyHostToDevice, e->s_h2d);
            if (!rc) rc = record(ev_buf(c, w), e->s_h2d);
        }
    }
    for (uint32_t c = 0; c < k && !rc; ++c) {
        if ((rc = wait(e->s_comp, ev_theta(c)))) break;
        if ((rc = run_virtual_chain(e, c, e->h_theta.data(), e->h_local.data()))) break;
        for (uint32_t w = 0; w < k && !rc; ++w) {
            if ((rc = wait(e->s_comp, ev_buf(c, w)))) break;
            if ((rc = run_virtual_apply(e, c, w, e->h_theta.data(), e->h_buf.data(),
                                        write_local ? e->h_local.data() : nullptr, nullptr, lr, mom)))
                break;
            if ((rc = record(ev_out(c, w), e->s_comp)) || (rc = wait(e->s_d2h, ev_out(c, w)))) break;
            rc = copy(theta_g[w], e->h_theta[w], c, cudaMemcpyDeviceToHost, e->s_d2h);
            if (!rc) rc = copy(buf[w], e->h_buf[w], c, cudaMemcpyDeviceToHost, e->s_d2h);
            if (!rc && write_local) rc = copy(theta_l[w], e->h_local[w], c, cudaMemcpyDeviceToHost, e->s_d2h);
        }
    }
    cudaStreamSynchronize(e->s_h2d);
    cudaStreamSynchronize(e->s_comp);
    cudaStreamSynchronize(e->s_d2h);
    for (auto x : ev) cudaEventDestroy(x);
    if (rc) return rc;
    return emesh_engine_check(e);
}

// Host-buffer outer sync, one worker per GPU (peer transport): theta_g /
// theta_l go up chunk by chunk in the order the ring reads them (own chunk,
// then r-1, r-2, ...), the momentum in decode order, and each chunk's
// results come back on a second copy stream as soon as its decode ran.
static int outer_sync_host_p2p(emesh_engine* e, float* theta_g, float* theta_l, float* buf, float lr, float mom,
                               int write_local) {
    const uint32_t k = e->k, r = e->rank;
    if (!e->s_h2d) CU(cudaStreamCreateWithFlags(&e->s_h2d, cudaStreamNonBlocking));
    if (!e->s_d2h) CU(cudaStreamCreateWithFlags(&e->s_d2h, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> ev(3 * k, nullptr);  // [c] theta landed, [k + c] momentum landed, [2k + c] decoded
    for (auto& x : ev) CU(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> runs(k);
    for (uint32_t c = 0; c < k; ++c)
        for (const Batch& bt : e->plan.batches[c])
            for (const auto& x : bt.eruns) {
                auto& v = runs[c];
                if (!v.empty() && v.back().first + v.back().second == x.first) v.back().second += x.second;
                else if (x.second) v.push_back(x);
            }
    auto copy = [&](float* dst, const float* src, uint32_t c, cudaMemcpyKind kind, cudaStream_t st) {
        for (const auto& x : runs[c])
            if (cudaMemcpyAsync(dst + x.first, src + x.first, x.second * sizeof(float), kind, st) != cudaSuccess)
                return fail(EMESH_ECUDA, "outer_sync_host: %s", cudaGetErrorString(cudaGetLastError()));
        return (int)EMESH_OK;
    };
    float* dg = e->h_theta[0];
    float* dl = e->h_local[0];
    float* db = e->h_buf[0];
    int rc = EMESH_OK;
    for (uint32_t i = 0; i < k && !rc; ++i) {  // RS read order: r, r-1, ..., r+1
        const uint32_t c = (r + k - i) % k;
        rc = copy(dg, theta_g, c, cudaMemcpyHostToDevice, e->s_h2d);
        if (!rc) rc = copy(dl, theta_l, c, cudaMemcpyHostToDevice, e->s_h2d);
        if (!rc && cudaEventRecord(ev[c], e->s_h2d) != cudaSuccess) rc = fail(EMESH_ECUDA, "event record");
    }
    for (uint32_t d = 0; d < k && !rc; ++d) {  // decode order: r+1, r, r-1, ...
        const uint32_t c = (r + 1 + k - d) % k;
        rc = copy(db, buf, c, cudaMemcpyHostToDevice, e->s_h2d);
        if (!rc && cudaEventRecord(ev[k + c], e->s_h2d) != cudaSuccess) rc = fail(EMESH_ECUDA, "event record");
    }
    HostPipe hp;
    hp.before_rs = [&](uint32_t c) {
        return cudaStreamWaitEvent(e->s_comp, ev[c], 0) == cudaSuccess ? (int)EMESH_OK : fail(EMESH_ECUDA, "wait");
    };
    hp.before_apply = [&](uint32_t c) {
        return cudaStreamWaitEvent(e->s_comp, ev[k + c], 0) == cudaSuccess ? (int)EMESH_OK
                                                                              : fail(EMESH_ECUDA, "wait");
    };
    hp.after_apply = [&](uint32_t c) {
        if (cudaEventRecord(ev[2 * k + c], e->s_comp) != cudaSuccess ||
            cudaStreamWaitEvent(e->s_d2h, ev[2 * k + c], 0) != cudaSuccess)
            return fail(EMESH_ECUDA, "event record");
        int q = copy(theta_g, dg, c, cudaMemcpyDeviceToHost, e->s_d2h);
        if (!q) q = copy(buf, db, c, cudaMemcpyDeviceToHost, e->s_d2h);
        if (!q && write_local) q = copy(theta_l, dl, c, cudaMemcpyDeviceToHost, e->s_d2h);
        return q;
    };
    // (no engine_enter: the compute stream must not wait for the whole upload, only per chunk)
    if (!rc) rc = run_p2p(e, dg, dl, dg, db, write_local ? dl : nullptr, nullptr, lr, mom, &hp);
    cudaStreamSynchronize(e->s_h2d);
    const int crc = emesh_engine_check(e);  // bounded: a vanished peer surfaces as EMESH_ERING
    cudaStreamSynchronize(e->s_d2h);
    for (auto x : ev) cudaEventDestroy(x);
    return rc ? rc : crc;
}

int emesh_engine_outer_sync_host(emesh_engine* e, float* const* theta_g, float* const* theta_l, float* const* buf,
                                 float lr, float mom, int write_local) {
    CU(cudaSetDevice(e->device));
    const uint64_t n = e->plan.n;
    const size_t bytes = n * sizeof(float);
    if (e->h_theta.empty()) {
        e->h_theta.assign(e->workers, nullptr);
        e->h_local.assign(e->workers, nullptr);
        e->h_buf.assign(e->workers, nullptr);
        for (uint32_t w = 0; w < e->workers; ++w) {
            CU(cudaMalloc(&e->h_theta[w], bytes + 16));
            CU(cudaMalloc(&e->h_local[w], bytes + 16));
            CU(cudaMalloc(&e->h_buf[w], bytes + 16));
        }
    }
    if (e->virt && !e->fp32 && e->k > 1)
        return outer_sync_host_pipelined(e, theta_g, theta_l, buf, lr, mom, write_local);
    if (!e->virt && !e->fp32 && e->k > 1 && e->transport == EMESH_TRANSPORT_P2P)
        return outer_sync_host_p2p(e, theta_g[0], theta_l[0], buf[0], lr, mom, write_local);
    cudaStream_t st = e->s_comp;
    for (uint32_t w = 0; w < e->workers; ++w) {
        CU(cudaMemcpyAsync(e->h_theta[w], theta_g[w], bytes, cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(e->h_local[w], theta_l[w], bytes, cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(e->h_buf[w], buf[w], bytes, cudaMemcpyHostToDevice, st));
    }
    TRY(emesh_engine_outer_sync(e, e->h_theta.data(), e->h_local.data(), e->h_buf.data(), lr, mom, write_local,
                                reinterpret_cast<emesh_stream_t>(st)));
    for (uint32_t w = 0; w < e->workers; ++w) {
        CU(cudaMemcpyAsync(theta_g[w], e->h_theta[w], bytes, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(buf[w], e->h_buf[w], bytes, cudaMemcpyDeviceToHost, st));
        if (write_local) CU(cudaMemcpyAsync(theta_l[w], e->h_local[w], bytes, cudaMemcpyDeviceToHost, st));
    }
    CU(cudaStreamSynchronize(st));
    return emesh_engine_check(e);
}

int emesh_engine_check(emesh_engine* e) {
    CU(cudaSetDevice(e->device));
    if (e->transport == EMESH_TRANSPORT_NCCL && e->comm && !e->virt) {
        // NCCL waits have no device-side budget: bound them here. A peer that
        // stops leaves our send/recv pending; after step_timeout the
        // communicator is aborted and the round reports RingFailureError
        // (allreduce.hpp:466-470).
        TRY(nccl_drain(e, {e->s_comp, e->s_comm}, "ring round"));
    }
    CU(cudaStreamSynchronize(e->s_comp));
    CU(cudaStreamSynchronize(e->s_comm));
    if (!e->ws.err) return EMESH_OK;
    uint32_t v[2] = {0, 0};
    e->setup_floor_ns = 0;  // a round drained: later waits get step_timeout alone
    CU(cudaMemcpy(v, e->ws.err, sizeof v, cudaMemcpyDeviceToHost));
    if (v[0]) {
        CU(cudaMemset(e->ws.err, 0, 2 * sizeof(uint32_t)));
        if (v[0] & kErrRing) {  // the round failed on some rank: nothing was committed (k_round_gate)
            e->failed = true;
            e->culprit = (v[1] && (v[1] - 1) != kNoCulprit) ? (int32_t)(v[1] - 1) : -1;
            char who[48] = "unknown";
            if (e->culprit >= 0) snprintf(who, sizeof who, "rank %d", e->culprit);
            if (v[0] & kErrStale)  // allreduce.hpp:272
                return fail(EMESH_ESTALE, "newer plan epoch on the ring (culprit %s)", who);
            if (v[0] & kErrProto)  // allreduce.hpp:280-281
                return fail(EMESH_EPROTO, "ring protocol violation: unexpected chunk header (from %s)", who);
            // allreduce.hpp:466-470: a peer stopped or aborted mid-collective
            return fail(EMESH_ERING, "ring step failed: a peer stalled past step_timeout (%.1f s) or aborted; culprit %s",
                        (double)e->tr.timeout_ns * 1e-9, who);
        }
        return fail(EMESH_ENUMERIC, "quantize: non-finite input");
    }
    return EMESH_OK;
}

int emesh_engine_failed_rank(const emesh_engine* e) { return e ? e->culprit : -1; }

int emesh_engine_set_job(emesh_engine* e, uint64_t job_id) {
    if (!e) return fail(EMESH_ECONFIG, "null engine");
    e->job = job_id;
    e->job_set = true;
    return EMESH_OK;
}

int emesh_engine_payload(emesh_engine* e, uint32_t worker, const uint8_t** codes, const float** cbs,
                         const double** stats, uint64_t* stride) {
    if (worker >= e->arenas.size()) return fail(EMESH_ECONFIG, "no such local worker");
    if (codes) *codes = payload_codes(e, worker);
    if (cbs) *cbs = payload_cbs(e, worker);
    if (stats) *stats = reinterpret_cast<const double*>(e->arenas[worker].stats);
    if (stride) *stride = sizeof(SegStat);
    return EMESH_OK;
}

int emesh_engine_payload_host(emesh_engine* e, uint32_t worker, uint8_t* codes, float* cbs, double* stats) {
    if (worker >= e->arenas.size()) return fail(EMESH_ECONFIG, "no such local worker");
    TRY(emesh_engine_check(e));
    const auto& a = e->arenas[worker];
    const size_t nseg = e->plan.segs.size();
    if (codes && e->plan.n) CU(cudaMemcpy(codes, payload_codes(e, worker), e->plan.n, cudaMemcpyDeviceToHost));
    if (cbs) CU(cudaMemcpy(cbs, payload_cbs(e, worker), nseg * kBuckets * sizeof(float), cudaMemcpyDeviceToHost));
    if (stats)
        CU(cudaMemcpy2D(stats, 4 * sizeof(double), a.stats, sizeof(SegStat), 4 * sizeof(double), nseg,
                        cudaMemcpyDeviceToHost));
    return EMESH_OK;
}

}  // extern "C"
