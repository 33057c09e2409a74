// Checkpoint serialization straight from / into device arenas
// (tensor.hpp:111-161 write/read_tensor + write/read_params,
// checkpoint.hpp:19-68 Checkpoint + encode/decode_checkpoint,
// checkpoint.hpp:190-224 the file framing).
//
// The five parameter sets of a Checkpoint (params, retained, AdamW m / v,
// Nesterov buffer) stay where the engine keeps them: one flat fp32 arena each
// in HBM, canonical tensor order. Serialization is therefore a layout walk:
// the host emits the small headers (name, rank, extents, counts, scalars)
// and the tensor data moves as contiguous device<->host copies landing at
// their byte offsets (fp32 LE == the arena bytes on this little-endian host).
// Pageable buffers are staged through a small ring of pinned blocks so the
// DMA of block j+1 overlaps the host copy / digest of block j; page-locked
// buffers are copied into directly. Decoding validates the whole byte
// structure on the host first (every DecodeError / ShapeError the reference
// raises, at the byte offset where it raises it), uploads, and then scans
// the uploaded arenas for non-finite values on the device (read_tensor's
// isfinite check, tensor.hpp:134-137).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "emesh_b200.h"
#include "sha256.h"

namespace emesh_b200 {
int set_error(int code, const std::string& msg);  // emesh_b200.cu (thread-local last error)
}

using emesh_b200::set_error;
using emesh_b200::Sha256;

namespace {

constexpr int kSets = 5;  // params, retained, adam m, adam v, nesterov buffer (encode order)

std::string fmt(const char* f, ...) __attribute__((format(printf, 1, 2)));
std::string fmt(const char* f, ...) {
    char b[512];
    va_list ap;
    va_start(ap, f);
    vsnprintf(b, sizeof b, f, ap);
    va_end(ap);
    return b;
}

#define CKU(call)                                                                                   \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return set_error(EMESH_ECUDA, fmt("%s: %s", #call, cudaGetErrorString(e_)));            \
    } while (0)

// ------------------------------------------------------------------ device

// First (lowest) element index of a non-finite value in x[0, n), atomicMin
// into *first (initialised to ~0). HBM-bound single pass, 16 B loads.
__global__ void k_first_nonfinite(const float* __restrict__ x, uint64_t n, unsigned long long* first) {
    const uint64_t n4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    unsigned long long best = ~0ull;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
        const float4 v = __ldcs(x4 + q);
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (!isfinite(e[j]) && q * 4 + j < best) best = q * 4 + j;
        if (best != ~0ull) break;  // later q of this thread are larger
    }
    for (uint64_t i = n4 * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        if (!isfinite(x[i]) && i < best) best = i;
    for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(first, best);
}

// ------------------------------------------------------------------ layout

struct TensorRec {
    std::string name;
    std::vector<uint32_t> shape;
    uint64_t numel = 1;
    uint64_t elem_off = 0;  // within the set's arena
    uint64_t data_off = 0;  // byte offset of the data in the payload
};

struct Layout {
    std::vector<TensorRec> t;  // one set's tensors (all five sets share them)
    uint64_t numel = 0;
    uint64_t set_bytes = 0;    // encoded bytes of one write_params
};

int layout_from_view(const emesh_checkpoint* ck, Layout& L) {
    if (!ck) return set_error(EMESH_ECONFIG, "null checkpoint");
    if (ck->ntensors && (!ck->names || !ck->ranks || !ck->extents))
        return set_error(EMESH_ECONFIG, "checkpoint view: names / ranks / extents required");
    L.t.resize(ck->ntensors);
    uint64_t e = 0;
    L.numel = 0;
    L.set_bytes = 4;
    for (uint32_t i = 0; i < ck->ntensors; ++i) {
        auto& r = L.t[i];
        r.name = ck->names[i] ? ck->names[i] : "";
        r.shape.assign(ck->extents + e, ck->extents + e + ck->ranks[i]);
        e += ck->ranks[i];
        r.numel = 1;
        for (uint32_t x : r.shape) {
            if (x == 0) return set_error(EMESH_ESHAPE, "zero extent in tensor shape");  // tensor.hpp:31-33
            r.numel *= x;
        }
        r.elem_off = L.numel;
        L.numel += r.numel;
        L.set_bytes += 4 + r.name.size() + 4 + 4ull * r.shape.size() + 4 * r.numel;
    }
    return EMESH_OK;
}

uint64_t encoded_size(const Layout& L) {
    return 8 + kSets * L.set_bytes + 8 + 8 + 8 + 4 + 32;  // checkpoint.hpp:32-47
}

// One piece of the payload, in stream order: host bytes or a device range.
struct Piece {
    const uint8_t* host;
    const float* dev;
    uint64_t bytes;
};

struct Emit {
    std::vector<uint8_t> hdr;  // all header bytes; header pieces hold offsets until finish() fixes the pointers
    std::vector<Piece> pieces;
    void u32(uint32_t v) { for (int i = 0; i < 4; ++i) hdr.push_back((uint8_t)(v >> (8 * i))); }
    void u64(uint64_t v) { for (int i = 0; i < 8; ++i) hdr.push_back((uint8_t)(v >> (8 * i))); }
    void raw(const void* p, size_t n) { hdr.insert(hdr.end(), (const uint8_t*)p, (const uint8_t*)p + n); }
    uint64_t open = 0;
    void cut_dev(const float* p, uint64_t bytes) {  // close the current header run, then a device piece
        if (hdr.size() > open) pieces.push_back({reinterpret_cast<const uint8_t*>(open), nullptr, hdr.size() - open});
        open = hdr.size();
        if (bytes) pieces.push_back({nullptr, p, bytes});
    }
    void finish() {
        cut_dev(nullptr, 0);
        for (auto& p : pieces)
            if (!p.dev) p.host = hdr.data() + reinterpret_cast<uintptr_t>(p.host);
    }
};

// checkpoint.hpp:32-47 / tensor.hpp:115-120,144-147, in stream order
void build_pieces(const emesh_checkpoint* ck, const Layout& L, Emit& E) {
    const float* sets[kSets] = {ck->params, ck->retained, ck->adam_m, ck->adam_v, ck->nesterov_buf};
    auto params = [&](const float* arena) {
        E.u32((uint32_t)L.t.size());
        for (const auto& r : L.t) {
            E.u32((uint32_t)r.name.size());
            E.raw(r.name.data(), r.name.size());
            E.u32((uint32_t)r.shape.size());
            for (uint32_t x : r.shape) E.u32(x);
            E.cut_dev(arena + r.elem_off, 4 * r.numel);
        }
    };
    E.u64(ck->outer_step);
    params(sets[0]);
    params(sets[1]);
    E.u64(ck->adam_step);
    params(sets[2]);
    params(sets[3]);
    params(sets[4]);
    E.u64(ck->rng_seed);
    E.u64(ck->data_counter);
    E.u32(ck->shard);
    E.raw(ck->config_hash, 32);
    E.finish();
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Pinned staging ring shared by all calls of the process (allocated once).
struct Staging {
    static constexpr int kSlots = 4;
    static constexpr size_t kBlock = 16u << 20;
    uint8_t* buf[kSlots] = {};
    std::mutex mu;
    int ensure() {
        if (buf[0]) return EMESH_OK;
        for (auto& b : buf)
            if (cudaHostAlloc(reinterpret_cast<void**>(&b), kBlock, cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                return set_error(EMESH_ECUDA, "checkpoint staging: cudaHostAlloc failed");
            }
        return EMESH_OK;
    }
};
Staging g_stage;

// Stream the pieces device->host in order into sink(ptr, n).
template <typename Sink>
int stream_out(const std::vector<Piece>& pieces, cudaStream_t st, Sink&& sink) {
    std::lock_guard<std::mutex> g(g_stage.mu);
    int rc = g_stage.ensure();
    if (rc) return rc;
    cudaEvent_t ev[Staging::kSlots];
    for (auto& e : ev) CKU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct Pend { int slot; const uint8_t* host; uint64_t n; };
    std::deque<Pend> q;
    bool busy[Staging::kSlots] = {};
    int next = 0;
    auto pop = [&]() -> int {
        Pend p = q.front();
        q.pop_front();
        if (p.slot < 0) return sink(p.host, p.n);
        if (cudaEventSynchronize(ev[p.slot]) != cudaSuccess) return set_error(EMESH_ECUDA, "checkpoint D2H failed");
        busy[p.slot] = false;
        return sink(g_stage.buf[p.slot], p.n);
    };
    for (const auto& pc : pieces) {
        if (!pc.dev) { q.push_back({-1, pc.host, pc.bytes}); continue; }
        for (uint64_t off = 0; off < pc.bytes && rc == EMESH_OK; off += Staging::kBlock) {
            const uint64_t nb = std::min<uint64_t>(Staging::kBlock, pc.bytes - off);
            while (busy[next] && rc == EMESH_OK) rc = pop();
            if (rc) break;
            if (cudaMemcpyAsync(g_stage.buf[next], reinterpret_cast<const uint8_t*>(pc.dev) + off, nb,
                                cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaEventRecord(ev[next], st) != cudaSuccess) {
                rc = set_error(EMESH_ECUDA, fmt("checkpoint D2H: %s", cudaGetErrorString(cudaGetLastError())));
                break;
            }
            busy[next] = true;
            q.push_back({next, nullptr, nb});
            next = (next + 1) % Staging::kSlots;
        }
        if (rc) break;
    }
    while (!q.empty() && rc == EMESH_OK) rc = pop();
    cudaStreamSynchronize(st);
    for (auto& e : ev) cudaEventDestroy(e);
    return rc;
}

// ------------------------------------------------------------------ parse

struct ParseErr {
    uint64_t off = ~0ull;  // byte offset where the reference raises it
    int code = EMESH_OK;
    std::string msg;
};

struct Parsed {
    uint64_t outer_step = 0, adam_step = 0, rng_seed = 0, data_counter = 0;
    uint32_t shard = 0;
    uint8_t hash[32] = {};
    std::vector<TensorRec> set[kSets];
    ParseErr err;
};

// Sequential parse with ByteReader semantics (bytes.hpp:52-92), stopping at
// the first error the reference would throw; data bytes are skipped, not read.
struct Reader {
    const uint8_t* b;
    uint64_t len, pos = 0;
    ParseErr* err;
    bool take(uint64_t n) {
        if (n > len - pos) {
            err->off = pos;
            err->code = EMESH_EDECODE;
            err->msg = "truncated buffer";
            return false;
        }
        pos += n;
        return true;
    }
    bool u32(uint32_t& v) {
        if (!take(4)) return false;
        const uint8_t* p = b + pos - 4;
        v = (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
        return true;
    }
    bool u64(uint64_t& v) {
        uint32_t lo, hi;
        if (!u32(lo) || !u32(hi)) return false;
        v = (uint64_t)lo | (uint64_t)hi << 32;
        return true;
    }
    bool fail(int code, const char* m) {
        err->off = pos;
        err->code = code;
        err->msg = m;
        return false;
    }
};

// tensor.hpp:122-154 read_tensor / read_params
bool parse_params(Reader& r, std::vector<TensorRec>& out) {
    uint32_t count;
    if (!r.u32(count)) return false;
    uint64_t elem = 0;
    for (uint32_t i = 0; i < count; ++i) {
        TensorRec t;
        uint32_t nlen;
        if (!r.u32(nlen)) return false;
        const uint64_t name_at = r.pos;
        if (!r.take(nlen)) return false;
        t.name.assign(reinterpret_cast<const char*>(r.b + name_at), nlen);
        uint32_t rank;
        if (!r.u32(rank)) return false;
        if (rank > 8) return r.fail(EMESH_EDECODE, "implausible tensor rank");
        t.shape.resize(rank);
        size_t cnt = 1;
        for (uint32_t& e : t.shape) {
            if (!r.u32(e)) return false;
            if (e == 0) return r.fail(EMESH_EDECODE, "zero extent");
            if (cnt > (1u << 28) / std::max<uint32_t>(e, 1)) return r.fail(EMESH_EDECODE, "implausible tensor size");
            cnt *= e;
        }
        t.numel = cnt;
        t.data_off = r.pos;
        t.elem_off = elem;
        // the reference reads the floats one by one: a truncation lands on the
        // first incomplete float (data before it is still checked for finiteness)
        const uint64_t avail = (r.len - r.pos) / 4;
        if (avail < cnt) {
            out.push_back(t);  // partial data [data_off, data_off + 4 avail) precedes the error
            r.pos += 4 * avail;
            return r.fail(EMESH_EDECODE, "truncated buffer");
        }
        r.pos += 4 * cnt;
        elem += cnt;
        for (const auto& o : out)  // ModelParams::add, tensor.hpp:59-63 (after the tensor was read)
            if (o.name == t.name) {
                out.push_back(t);
                return r.fail(EMESH_ESHAPE, ("duplicate parameter name: " + t.name).c_str());
            }
        out.push_back(std::move(t));
    }
    return true;
}

bool same_shapes(const std::vector<TensorRec>& a, const std::vector<TensorRec>& b) {  // tensor.hpp:72-79
    if (a.size() != b.size()) return false;
    for (size_t i = 0; i < a.size(); ++i)
        if (a[i].name != b[i].name || a[i].shape != b[i].shape) return false;
    return true;
}

// checkpoint.hpp:49-66 decode_checkpoint
void parse_checkpoint(const uint8_t* b, uint64_t len, Parsed& P) {
    Reader r{b, len, 0, &P.err};
    if (!r.u64(P.outer_step)) return;
    if (!parse_params(r, P.set[0]) || !parse_params(r, P.set[1])) return;
    if (!r.u64(P.adam_step)) return;
    if (!parse_params(r, P.set[2]) || !parse_params(r, P.set[3]) || !parse_params(r, P.set[4])) return;
    if (!r.u64(P.rng_seed) || !r.u64(P.data_counter) || !r.u32(P.shard)) return;
    if (!r.take(32)) return;
    std::memcpy(P.hash, b + r.pos - 32, 32);
    if (r.pos != len) { r.fail(EMESH_EDECODE, "trailing bytes after decode"); return; }
    for (int s = 1; s < kSets; ++s)
        if (!same_shapes(P.set[0], P.set[s])) {
            r.fail(EMESH_EDECODE, "checkpoint tensor shapes inconsistent");
            return;
        }
}

// Host-side finiteness scan of the data bytes preceding a structural error
// (error path only: nothing is uploaded when the structure is invalid).
uint64_t first_nonfinite_host(const uint8_t* b, const Parsed& P, uint64_t limit) {
    for (const auto& set : P.set)
        for (const auto& t : set) {
            const uint64_t end = std::min<uint64_t>(t.data_off + 4 * t.numel, limit);
            for (uint64_t o = t.data_off; o + 4 <= end; o += 4) {
                float v;
                std::memcpy(&v, b + o, 4);
                if (!std::isfinite(v)) return o;
            }
        }
    return ~0ull;
}

// Any non-finite float in the tensor payloads, scanned on the host before a
// single byte reaches the caller's arenas (a malformed checkpoint must leave
// the destination untouched, like the reference's decode_checkpoint, which
// returns by value): exponent-field test on the raw words, split over threads.
bool any_nonfinite_host(const uint8_t* b, const Parsed& P) {
    std::vector<std::pair<uint64_t, uint64_t>> ranges;  // byte ranges of every tensor payload
    uint64_t total = 0;
    for (const auto& set : P.set)
        for (const auto& t : set)
            if (t.numel) {
                ranges.push_back({t.data_off, 4 * t.numel});
                total += 4 * t.numel;
            }
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const unsigned nt = total < (64ull << 20) ? 1u : hw;
    std::vector<int> bad(nt, 0);
    auto scan = [&](unsigned w) {
        const uint64_t lo = total * w / nt, hi = total * (w + 1) / nt;  // this thread's share of the bytes
        uint64_t pos = 0;
        for (const auto& r : ranges) {
            const uint64_t a = std::max(lo, pos), e = std::min(hi, pos + r.second);
            pos += r.second;
            if (a >= e) continue;
            const uint64_t a4 = (a - (pos - r.second)) & ~uint64_t(3), e4 = e - (pos - r.second);
            for (uint64_t o = a4; o + 4 <= e4; o += 4) {
                uint32_t u;
                std::memcpy(&u, b + r.first + o, 4);
                if ((u & 0x7f800000u) == 0x7f800000u) { bad[w] = 1; return; }
            }
        }
    };
    if (nt == 1) scan(0);
    else {
        std::vector<std::thread> th;
        for (unsigned w = 0; w < nt; ++w) th.emplace_back(scan, w);
        for (auto& t : th) t.join();
    }
    for (int v : bad)
        if (v) return true;
    return false;
}

int check_layout(const Layout& L, const std::vector<TensorRec>& got) {
    if (got.size() != L.t.size())
        return set_error(EMESH_EDECODE, fmt("checkpoint holds %zu tensors, the destination arenas %zu", got.size(),
                                            L.t.size()));
    for (size_t i = 0; i < got.size(); ++i)
        if (got[i].name != L.t[i].name || got[i].shape != L.t[i].shape)
            return set_error(EMESH_EDECODE, fmt("checkpoint tensor %zu (%s) differs from the destination layout", i,
                                                got[i].name.c_str()));
    return EMESH_OK;
}

// Upload the parsed tensor data into the five arenas, then the device scan.
int upload_and_scan(const uint8_t* b, const Parsed& P, const emesh_checkpoint* ck, const Layout& L,
                    cudaStream_t st) {
    float* sets[kSets] = {ck->params, ck->retained, ck->adam_m, ck->adam_v, ck->nesterov_buf};
    for (int s = 0; s < kSets; ++s)
        if (L.numel && !sets[s]) return set_error(EMESH_ECONFIG, "checkpoint view: null device arena");
    const bool pinned = is_pinned(b);
    {
        std::lock_guard<std::mutex> g(g_stage.mu);
        int rc = pinned ? EMESH_OK : g_stage.ensure();
        if (rc) return rc;
        cudaEvent_t ev[Staging::kSlots] = {};
        bool used[Staging::kSlots] = {};
        for (auto& e : ev) CKU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        int next = 0;
        for (int s = 0; s < kSets && rc == EMESH_OK; ++s)
            for (const auto& t : P.set[s]) {
                const uint8_t* src = b + t.data_off;
                uint8_t* dst = reinterpret_cast<uint8_t*>(sets[s] + t.elem_off);
                const uint64_t bytes = 4 * t.numel;
                if (pinned) {
                    if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) rc = EMESH_ECUDA;
                    continue;
                }
                for (uint64_t off = 0; off < bytes; off += Staging::kBlock) {
                    const uint64_t nb = std::min<uint64_t>(Staging::kBlock, bytes - off);
                    if (used[next] && cudaEventSynchronize(ev[next]) != cudaSuccess) { rc = EMESH_ECUDA; break; }
                    std::memcpy(g_stage.buf[next], src + off, nb);
                    if (cudaMemcpyAsync(dst + off, g_stage.buf[next], nb, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                        cudaEventRecord(ev[next], st) != cudaSuccess) {
                        rc = EMESH_ECUDA;
                        break;
                    }
                    used[next] = true;
                    next = (next + 1) % Staging::kSlots;
                }
                if (rc) break;
            }
        cudaStreamSynchronize(st);  // the staging blocks are reused by the next call
        for (auto& e : ev) cudaEventDestroy(e);
        if (rc) return set_error(EMESH_ECUDA, fmt("checkpoint H2D: %s", cudaGetErrorString(cudaGetLastError())));
    }
    if (!L.numel) return EMESH_OK;
    unsigned long long* d_first = nullptr;
    CKU(cudaMallocAsync(reinterpret_cast<void**>(&d_first), kSets * sizeof(unsigned long long), st));
    CKU(cudaMemsetAsync(d_first, 0xff, kSets * sizeof(unsigned long long), st));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (L.numel / 4 + 255) / 256;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * 8));
    for (int s = 0; s < kSets; ++s) k_first_nonfinite<<<grid, 256, 0, st>>>(sets[s], L.numel, d_first + s);
    unsigned long long first[kSets];
    CKU(cudaMemcpyAsync(first, d_first, sizeof first, cudaMemcpyDeviceToHost, st));
    CKU(cudaFreeAsync(d_first, st));
    CKU(cudaStreamSynchronize(st));
    // the earliest non-finite value in stream order wins (sets are serialized in order)
    for (int s = 0; s < kSets; ++s)
        if (first[s] != ~0ull) return set_error(EMESH_EDECODE, "non-finite value in tensor payload");
    return EMESH_OK;
}

int decode_into(const uint8_t* b, uint64_t len, emesh_checkpoint* ck, cudaStream_t st) {
    Layout L;
    int rc = layout_from_view(ck, L);
    if (rc) return rc;
    Parsed P;
    parse_checkpoint(b, len, P);
    if (P.err.code != EMESH_OK) {
        // a non-finite float read before the structural error is what the reference reports
        if (first_nonfinite_host(b, P, P.err.off) < P.err.off)
            return set_error(EMESH_EDECODE, "non-finite value in tensor payload");
        return set_error(P.err.code, P.err.msg);
    }
    if ((rc = check_layout(L, P.set[0]))) return rc;
    if (any_nonfinite_host(b, P)) return set_error(EMESH_EDECODE, "non-finite value in tensor payload");
    if ((rc = upload_and_scan(b, P, ck, L, st))) return rc;
    ck->outer_step = P.outer_step;
    ck->adam_step = P.adam_step;
    ck->rng_seed = P.rng_seed;
    ck->data_counter = P.data_counter;
    ck->shard = P.shard;
    std::memcpy(ck->config_hash, P.hash, 32);
    return EMESH_OK;
}

}  // namespace

extern "C" {

int emesh_sha256(const void* data, uint64_t n, uint8_t out[32]) {
    Sha256 h;
    h.update(data, n);
    h.finish(out);
    return EMESH_OK;
}

int emesh_checkpoint_encoded_size(const emesh_checkpoint* ck, uint64_t* bytes) {
    Layout L;
    int rc = layout_from_view(ck, L);
    if (rc) return rc;
    *bytes = encoded_size(L);
    return EMESH_OK;
}

int emesh_checkpoint_encode(const emesh_checkpoint* ck, uint8_t* out, uint64_t cap, uint64_t* written,
                            emesh_stream_t stream) {
    Layout L;
    int rc = layout_from_view(ck, L);
    if (rc) return rc;
    const uint64_t need = encoded_size(L);
    if (written) *written = need;
    if (cap < need) return set_error(EMESH_ESHAPE, fmt("checkpoint needs %llu bytes, buffer holds %llu",
                                                       (unsigned long long)need, (unsigned long long)cap));
    Emit E;
    build_pieces(ck, L, E);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (is_pinned(out)) {  // DMA straight into place
        uint64_t pos = 0;
        for (const auto& p : E.pieces) {
            if (p.dev) CKU(cudaMemcpyAsync(out + pos, p.dev, p.bytes, cudaMemcpyDeviceToHost, st));
            else std::memcpy(out + pos, p.host, p.bytes);
            pos += p.bytes;
        }
        CKU(cudaStreamSynchronize(st));
        return EMESH_OK;
    }
    uint64_t pos = 0;
    return stream_out(E.pieces, st, [&](const uint8_t* p, uint64_t n) -> int {
        std::memcpy(out + pos, p, n);
        pos += n;
        return EMESH_OK;
    });
}

int emesh_checkpoint_decode(const uint8_t* buf, uint64_t len, emesh_checkpoint* ck, emesh_stream_t stream) {
    return decode_into(buf, len, ck, reinterpret_cast<cudaStream_t>(stream));
}

int emesh_checkpoint_probe(const uint8_t* buf, uint64_t len, uint32_t* ntensors, uint64_t* numel,
                           uint64_t* name_bytes, uint32_t* rank_sum) {
    Parsed P;
    ParseErr err;
    Reader r{buf, len, 0, &err};
    uint64_t step;
    if (!r.u64(step) || !parse_params(r, P.set[0])) return set_error(err.code, err.msg);
    uint64_t n = 0, nb = 0;
    uint32_t rs = 0;
    for (const auto& t : P.set[0]) { n += t.numel; nb += t.name.size() + 1; rs += (uint32_t)t.shape.size(); }
    if (ntensors) *ntensors = (uint32_t)P.set[0].size();
    if (numel) *numel = n;
    if (name_bytes) *name_bytes = nb;
    if (rank_sum) *rank_sum = rs;
    return EMESH_OK;
}

int emesh_checkpoint_layout(const uint8_t* buf, uint64_t len, char* names, uint64_t names_cap, uint32_t* ranks,
                            uint32_t* extents, uint32_t extents_cap) {
    Parsed P;
    ParseErr err;
    Reader r{buf, len, 0, &err};
    uint64_t step;
    if (!r.u64(step) || !parse_params(r, P.set[0])) return set_error(err.code, err.msg);
    uint64_t at = 0;
    uint32_t e = 0;
    for (size_t i = 0; i < P.set[0].size(); ++i) {
        const auto& t = P.set[0][i];
        if (at + t.name.size() + 1 > names_cap || e + t.shape.size() > extents_cap)
            return set_error(EMESH_ESHAPE, "checkpoint layout: output arrays too small");
        std::memcpy(names + at, t.name.c_str(), t.name.size() + 1);
        at += t.name.size() + 1;
        ranks[i] = (uint32_t)t.shape.size();
        for (uint32_t x : t.shape) extents[e++] = x;
    }
    return EMESH_OK;
}

// checkpoint.hpp:190-203: u64 LE payload length, sha256(payload), payload.
// The payload streams device -> pinned -> file while it is hashed; the head
// is patched in place at the end (no full host copy of the payload).
int emesh_checkpoint_write_file(const char* path, const emesh_checkpoint* ck, emesh_stream_t stream) {
    Layout L;
    int rc = layout_from_view(ck, L);
    if (rc) return rc;
    FILE* f = std::fopen(path, "wb");
    if (!f) return set_error(EMESH_EIO, fmt("cannot write checkpoint file %s", path));
    std::setvbuf(f, nullptr, _IOFBF, 8u << 20);
    uint8_t head[40] = {};
    const uint64_t total = encoded_size(L);
    for (int i = 0; i < 8; ++i) head[i] = (uint8_t)(total >> (8 * i));
    bool ok = std::fwrite(head, 1, 40, f) == 40;
    Emit E;
    build_pieces(ck, L, E);
    Sha256 h;
    rc = stream_out(E.pieces, reinterpret_cast<cudaStream_t>(stream), [&](const uint8_t* p, uint64_t n) -> int {
        h.update(p, n);
        if (std::fwrite(p, 1, n, f) != n) return set_error(EMESH_EIO, fmt("short write to %s", path));
        return EMESH_OK;
    });
    h.finish(head + 8);
    ok = ok && rc == EMESH_OK && std::fseek(f, 8, SEEK_SET) == 0 && std::fwrite(head + 8, 1, 32, f) == 32;
    ok = (std::fclose(f) == 0) && ok;
    if (rc) return rc;
    if (!ok) return set_error(EMESH_EIO, fmt("cannot write checkpoint file %s", path));
    return EMESH_OK;
}

// checkpoint.hpp:205-224
int emesh_checkpoint_read_file(const char* path, emesh_checkpoint* ck, emesh_stream_t stream) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return set_error(EMESH_EIO, fmt("cannot read checkpoint file %s", path));
    uint8_t head[40];
    if (std::fread(head, 1, 40, f) != 40) {
        std::fclose(f);
        return set_error(EMESH_EDECODE, "truncated checkpoint file");
    }
    uint64_t total = 0;
    for (int i = 0; i < 8; ++i) total |= (uint64_t)head[i] << (8 * i);
    std::fseek(f, 0, SEEK_END);
    const long fsize = std::ftell(f);
    std::fseek(f, 40, SEEK_SET);
    if (fsize < 40 || total > (uint64_t)fsize - 40) {
        std::fclose(f);
        return set_error(EMESH_EDECODE, "truncated checkpoint file");
    }
    std::vector<uint8_t> payload(total);
    Sha256 h;
    for (uint64_t off = 0; off < total;) {
        const uint64_t nb = std::min<uint64_t>(total - off, 16u << 20);
        if (std::fread(payload.data() + off, 1, nb, f) != nb) {
            std::fclose(f);
            return set_error(EMESH_EDECODE, "truncated checkpoint file");
        }
        h.update(payload.data() + off, nb);
        off += nb;
    }
    std::fclose(f);
    uint8_t dg[32];
    h.finish(dg);
    if (std::memcmp(dg, head + 8, 32) != 0) return set_error(EMESH_EIO, "checkpoint file hash mismatch");
    return decode_into(payload.data(), total, ck, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
