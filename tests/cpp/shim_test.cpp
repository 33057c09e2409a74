// C++ drop-in check (include/emesh_b200.hpp): every emesh::b200 function
// against the reference's own emesh:: function on the same host data,
// bit for bit. The ring is checked against a transport-free restatement
// built from the reference's own pieces (ring_detail::split, encode_slice /
// decode_slice, the hop order of allreduce.hpp:411-464).
// Built by tests/cpp/Makefile against /root/reference/proj/include; run by
// tests/test_cpp_shim.py on a GPU. Exit 0 iff every check passes.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "emesh_b200.hpp"

using namespace emesh;

static int failures = 0;
#define EXPECT(cond, ...)                      \
    do {                                       \
        if (!(cond)) {                         \
            std::printf("FAIL: " __VA_ARGS__); \
            std::printf("\n");                 \
            ++failures;                        \
        }                                      \
    } while (0)

static bool same_bits(const std::vector<float>& a, const std::vector<float>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 4 * a.size()) == 0);
}

static std::vector<float> randv(size_t n, uint32_t seed, float scale, float shift = 0.f) {
    std::mt19937 g(seed);
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    std::vector<float> v(n);
    for (auto& x : v) x = u(g) * scale + shift;
    return v;
}

static ModelParams model(uint32_t seed, float scale) {
    ModelParams p;
    p.add("embed", Tensor({300, 7}, randv(2100, seed, scale)));
    p.add("norm", Tensor({13}, randv(13, seed + 1, scale)));
    p.add("proj", Tensor({50, 41}, randv(2050, seed + 2, scale)));
    return p;
}

static bool same_params(const ModelParams& a, const ModelParams& b) { return same_bits(a.flatten(), b.flatten()); }

// allreduce.hpp:314-464 without a transport: worker r's ring position, hop by hop.
static std::vector<std::vector<Bytes>> g_final_wire;  // [chunk][sub]: the bytes the all-gather forwards

static std::vector<std::vector<float>> ring_restated(const std::vector<std::vector<float>>& in, uint32_t S,
                                                     ReduceMode mode) {
    g_final_wire.assign(in.size(), {});
    using namespace ring_detail;
    const size_t k = in.size(), n = in[0].size();
    auto chunks = split(n, k);
    auto subs_of = [&](uint32_t c) {
        auto [lo, hi] = chunks[c];
        size_t len = hi - lo;
        auto subs = split(len, len == 0 ? 1 : std::min<size_t>(S, len));
        for (auto& s : subs) { s.first += lo; s.second += lo; }
        return subs;
    };
    std::vector<std::vector<float>> acc = in;
    for (size_t s = 0; s + 1 < k; ++s) {
        std::vector<std::vector<Bytes>> sent(k);  // what rank r ships at hop s
        for (size_t r = 0; r < k; ++r)
            for (auto [lo, hi] : subs_of((uint32_t)((r + k - s) % k)))
                sent[r].push_back(encode_slice(std::span<const float>(acc[r].data() + lo, hi - lo), mode));
        for (size_t r = 0; r < k; ++r) {
            const size_t pred = (r + k - 1) % k;
            auto subs = subs_of((uint32_t)((r + k - s - 1) % k));
            for (size_t j = 0; j < subs.size(); ++j) {
                std::vector<float> vals = decode_slice(sent[pred][j], mode);
                for (size_t i = 0; i < vals.size(); ++i) acc[r][subs[j].first + i] += vals[i];
            }
        }
    }
    std::vector<float> result(n);
    for (size_t r = 0; r < k; ++r) {  // owner of chunk (r+1)%k: mean, encode, every rank decodes
        for (auto [lo, hi] : subs_of((uint32_t)((r + 1) % k))) {
            std::vector<float> mean(hi - lo);
            for (size_t i = 0; i < mean.size(); ++i) mean[i] = acc[r][lo + i] / static_cast<float>(k);
            Bytes wire = encode_slice(mean, mode);
            g_final_wire[(r + 1) % k].push_back(wire);
            std::vector<float> v = decode_slice(wire, mode);
            std::copy(v.begin(), v.end(), result.begin() + lo);
        }
    }
    return std::vector<std::vector<float>>(k, result);
}

int main() {
    // quant.hpp: quantize / dequantize / wire codec
    for (auto [n, seed, scale, shift] : {std::tuple<size_t, uint32_t, float, float>{1, 1, 1.f, 0.f},
                                         {2, 2, 1.f, 0.f}, {4097, 3, 1e-3f, 0.f}, {100003, 4, 2.f, 7.f},
                                         {65536, 5, 1e-20f, 0.f}}) {
        auto x = randv(n, seed, scale, shift);
        if (n > 8) x[n / 3] = shift + 40 * scale;  // an outlier (clipping)
        QuantChunk a = quantize(x), b = b200::quantize(x);
        EXPECT(a.indices == b.indices, "quantize codes n=%zu", n);
        EXPECT(same_bits(a.codebook, b.codebook), "quantize codebook n=%zu", n);
        EXPECT(same_bits(dequantize(a), b200::dequantize(a)), "dequantize n=%zu", n);
        EXPECT(encode_quant_chunk(a) == b200::encode_quant_chunk(a), "encode n=%zu", n);
        QuantChunk d = b200::decode_quant_chunk(encode_quant_chunk(a));
        EXPECT(d.indices == a.indices && same_bits(d.codebook, a.codebook), "decode n=%zu", n);
    }
    {
        std::vector<float> c(1000, 2.5f);
        QuantChunk a = quantize(c), b = b200::quantize(c);
        EXPECT(a.indices == b.indices && same_bits(a.codebook, b.codebook), "constant chunk");
    }
    bool thrown = false;
    try { b200::quantize(std::vector<float>{}); } catch (const ShapeError&) { thrown = true; }
    EXPECT(thrown, "empty quantize must throw ShapeError");
    thrown = false;
    try { b200::quantize(std::vector<float>{1.f, NAN, 2.f}); } catch (const NumericError&) { thrown = true; }
    EXPECT(thrown, "non-finite quantize must throw NumericError");
    thrown = false;
    try { b200::decode_quant_chunk(Bytes{1, 2, 3}); } catch (const DecodeError&) { thrown = true; }
    EXPECT(thrown, "truncated decode must throw DecodeError");

    // optim.hpp: pseudo-gradient, Nesterov, AdamW
    ModelParams prev = model(10, 1.f), local = model(10, 1.f);
    {
        auto f = local.flatten();
        auto d = randv(f.size(), 11, 1e-3f);
        for (size_t i = 0; i < f.size(); ++i) f[i] -= d[i];
        local.unflatten(f);
    }
    ModelParams pa = compute_pseudo_gradient(prev, local), pb = b200::compute_pseudo_gradient(prev, local);
    EXPECT(same_params(pa, pb), "compute_pseudo_gradient");
    HyperParams hp;
    ModelParams ta = prev, tb = prev;
    NesterovState sa = NesterovState::zeros_like(prev), sb = NesterovState::zeros_like(prev);
    for (int it = 0; it < 2; ++it) {
        nesterov_outer_step(ta, pa, sa, hp);
        b200::nesterov_outer_step(tb, pa, sb, hp);
    }
    EXPECT(same_params(ta, tb) && same_params(sa.buffer, sb.buffer), "nesterov_outer_step");
    ModelParams wa = prev, wb = prev;
    AdamWState aa = AdamWState::zeros_like(prev), ab = AdamWState::zeros_like(prev);
    for (int it = 0; it < 3; ++it) {
        ModelParams g = model(20 + it, 1e-2f);
        adamw_step(wa, g, aa, hp, 0.3f * (it + 1));
        b200::adamw_step(wb, g, ab, hp, 0.3f * (it + 1));
    }
    EXPECT(same_params(wa, wb) && same_params(aa.m, ab.m) && same_params(aa.v, ab.v) && aa.step == ab.step,
           "adamw_step");

    // allreduce.hpp: k workers on this GPU, both modes, vs the restatement
    for (ReduceMode mode : {ReduceMode::int8, ReduceMode::fp32}) {
        for (uint32_t k : {2u, 3u, 4u}) {
            const size_t n = 100003;
            RingPlan plan;
            for (uint32_t i = 0; i < k; ++i) plan.order.push_back("w" + std::to_string(i));
            ReduceOptions opts;
            opts.pipeline_subchunks = 4;
            std::vector<ReduceJob> jobs;
            std::vector<std::vector<float>> ins;
            for (uint32_t i = 0; i < k; ++i) {
                ins.push_back(randv(n, 100 + i, 1e-2f));
                jobs.push_back(ReduceJob{1, ins.back(), mode});
            }
            b200::RingEngine eng(n, plan, opts, mode, nullptr, k);
            auto got = eng.ring_allreduce(jobs);
            auto want = ring_restated(ins, 4, mode);
            for (uint32_t w = 0; w < k; ++w)
                EXPECT(same_bits(got[w], want[w]), "ring mode=%d k=%u worker %u", (int)mode, k, w);
            if (mode == ReduceMode::int8)  // wire interop: the reference's all-gather bytes, segment by segment
                for (uint32_t c = 0; c < k; ++c) {
                    auto wire = eng.final_payloads(c, (c + k - 1) % k);  // the owner's arena
                    EXPECT(wire == g_final_wire[c], "final wire payloads k=%u chunk %u", k, c);
                }
        }
    }
    // trainer.hpp:355-382 outer sync, k = 4 local workers
    {
        const uint32_t k = 4;
        RingPlan plan;
        for (uint32_t i = 0; i < k; ++i) plan.order.push_back("w" + std::to_string(i));
        ReduceOptions opts;
        opts.pipeline_subchunks = 4;
        std::vector<ModelParams> ret(k, prev), loc, want_ret;
        std::vector<NesterovState> st(k, NesterovState::zeros_like(prev));
        std::vector<std::vector<float>> deltas;
        for (uint32_t w = 0; w < k; ++w) {
            ModelParams l = prev;
            auto f = l.flatten();
            auto d = randv(f.size(), 200 + w, 1e-3f);
            for (size_t i = 0; i < f.size(); ++i) f[i] -= d[i];
            l.unflatten(f);
            loc.push_back(l);
            deltas.push_back(compute_pseudo_gradient(prev, l).flatten());
        }
        auto mean = ring_restated(deltas, 4, ReduceMode::int8)[0];
        ModelParams avg = prev.zeros_like();
        avg.unflatten(mean);
        ModelParams expect_theta = prev;
        NesterovState expect_st = NesterovState::zeros_like(prev);
        nesterov_outer_step(expect_theta, avg, expect_st, HyperParams{});
        b200::RingEngine eng(prev.element_count(), plan, opts, ReduceMode::int8, nullptr, k);
        std::vector<ModelParams*> pr, pl;
        std::vector<NesterovState*> ps;
        for (uint32_t w = 0; w < k; ++w) { pr.push_back(&ret[w]); pl.push_back(&loc[w]); ps.push_back(&st[w]); }
        eng.outer_sync(pr, pl, ps, HyperParams{});
        for (uint32_t w = 0; w < k; ++w) {
            EXPECT(same_params(ret[w], expect_theta), "outer_sync theta worker %u", w);
            EXPECT(same_params(st[w].buffer, expect_st.buffer), "outer_sync momentum worker %u", w);
            EXPECT(same_params(loc[w], expect_theta), "outer_sync local = retained worker %u", w);
        }
    }
    std::printf(failures ? "cpp shim: %d FAILURES\n" : "cpp shim OK\n", failures);
    return failures ? 1 : 0;
}
