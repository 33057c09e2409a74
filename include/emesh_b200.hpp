// emesh_b200.hpp — C++ drop-in for the reference's outer-sync API
// (proj/include/emesh: quant.hpp, optim.hpp, allreduce.hpp, trainer.hpp:355-382)
// over the C ABI of libemesh_b200.so (include/emesh_b200.h).
//
// Every function has the signature of its reference counterpart and lives in
// namespace emesh::b200, taking and returning the reference's own types
// (QuantChunk, ModelParams, NesterovState, AdamWState, HyperParams, ReduceJob,
// ReduceOptions, RingPlan) and throwing the reference's exception classes
// (errors.hpp). A maintainer switches a call site from emesh::quantize to
// emesh::b200::quantize; the results are bit-identical (codes, codebooks,
// updated parameters). These host-data overloads copy to and from the GPU
// (parity and integration use); the throughput path keeps the arenas resident
// and calls emesh_engine_outer_sync on device pointers.
//
// Requires the reference headers on the include path (-I proj/include), the
// CUDA runtime and -lemesh_b200.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "emesh/allreduce.hpp"
#include "emesh/errors.hpp"
#include "emesh/optim.hpp"
#include "emesh/quant.hpp"
#include "emesh/tensor.hpp"
#include "emesh_b200.h"

namespace emesh::b200 {

// C ABI status -> the reference's exception (errors.hpp)
inline void check(int rc) {
    if (rc == EMESH_OK) return;
    const std::string what = emesh_last_error();
    switch (rc) {
        case EMESH_ESHAPE: throw ShapeError(what);
        case EMESH_ENUMERIC: throw NumericError(what);
        case EMESH_EDECODE: throw DecodeError(what);
        case EMESH_ECONFIG: throw ConfigError(what);
        case EMESH_ERING: throw RingFailureError("", what);
        case EMESH_ENCCL: throw RingFailureError("", what);
        case EMESH_ESTALE: throw StalePlanError(0, what);
        case EMESH_EPROTO: throw Error(what);
        default: throw FatalError(what);
    }
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw FatalError(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer (256-byte aligned by cudaMalloc; 32 bytes of slack for
// the 32-byte octet grid the quantizer reads)
template <typename T>
class DeviceBuffer {
public:
    explicit DeviceBuffer(size_t n) : n_(n) {
        cuda_check(cudaMalloc(&p_, (n ? n : 1) * sizeof(T) + 32), "cudaMalloc");
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    ~DeviceBuffer() { cudaFree(p_); }
    T* get() const { return p_; }
    void upload(const T* h, size_t n) { cuda_check(cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D"); }
    void download(T* h, size_t n) const {
        cuda_check(cudaMemcpy(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

// ---------------------------------------------------------------- quant.hpp

// quant.hpp:28
inline QuantChunk quantize(std::span<const float> values) {
    const size_t n = values.size();
    DeviceBuffer<float> x(n);
    DeviceBuffer<uint8_t> codes(n);
    DeviceBuffer<float> cb(QuantChunk::kBuckets);
    if (n) x.upload(values.data(), n);
    check(emesh_quantize(x.get(), n, codes.get(), cb.get(), nullptr, nullptr));
    QuantChunk q;
    q.codebook.resize(QuantChunk::kBuckets);
    q.indices.resize(n);
    cb.download(q.codebook.data(), QuantChunk::kBuckets);
    if (n) codes.download(q.indices.data(), n);
    return q;
}

// quant.hpp:89
inline void dequantize_into(const QuantChunk& chunk, std::span<float> out) {
    if (out.size() != chunk.count()) throw ShapeError("dequantize: output size mismatch");
    if (chunk.codebook.size() != QuantChunk::kBuckets) throw ShapeError("dequantize: malformed codebook");
    const size_t n = chunk.count();
    if (!n) return;
    DeviceBuffer<uint8_t> codes(n);
    DeviceBuffer<float> cb(QuantChunk::kBuckets), y(n);
    codes.upload(chunk.indices.data(), n);
    cb.upload(chunk.codebook.data(), QuantChunk::kBuckets);
    check(emesh_dequantize(codes.get(), cb.get(), n, y.get(), nullptr));
    cuda_check(cudaDeviceSynchronize(), "dequantize");
    y.download(out.data(), n);
}

// quant.hpp:96
inline std::vector<float> dequantize(const QuantChunk& chunk) {
    std::vector<float> out(chunk.count());
    b200::dequantize_into(chunk, out);  // qualified: ADL would also find emesh::dequantize_into
    return out;
}

// quant.hpp:111 (wire layout quant.hpp:102)
inline Bytes encode_quant_chunk(const QuantChunk& chunk) {
    if (chunk.codebook.size() != QuantChunk::kBuckets) throw ShapeError("encode_quant_chunk: malformed codebook");
    Bytes out(4 + 4 * QuantChunk::kBuckets + chunk.count());
    emesh_encode_quant_chunk(chunk.indices.data(), chunk.codebook.data(), static_cast<uint32_t>(chunk.count()),
                             out.data());
    return out;
}

// quant.hpp:117
inline QuantChunk decode_quant_chunk(const Bytes& buf) {
    QuantChunk q;
    q.codebook.resize(QuantChunk::kBuckets);
    q.indices.resize(buf.size());
    uint32_t count = 0;
    check(emesh_decode_quant_chunk(buf.data(), buf.size(), q.indices.data(), q.codebook.data(), &count));
    q.indices.resize(count);
    return q;
}

// ---------------------------------------------------------------- optim.hpp

// optim.hpp:99
inline ModelParams compute_pseudo_gradient(const ModelParams& theta_prev, const ModelParams& theta_local) {
    if (!theta_prev.same_shapes(theta_local)) throw ShapeError("compute_pseudo_gradient: shape mismatch");
    const std::vector<float> a = theta_prev.flatten(), b = theta_local.flatten();
    const size_t n = a.size();
    ModelParams delta = theta_prev.zeros_like();
    if (!n) return delta;
    DeviceBuffer<float> da(n), db(n), dd(n);
    da.upload(a.data(), n);
    db.upload(b.data(), n);
    check(emesh_pseudo_gradient(da.get(), db.get(), dd.get(), n, nullptr));
    std::vector<float> d(n);
    cuda_check(cudaDeviceSynchronize(), "pseudo_gradient");
    dd.download(d.data(), n);
    delta.unflatten(d);
    return delta;
}

// optim.hpp:116
inline void nesterov_outer_step(ModelParams& params, const ModelParams& avg_delta, NesterovState& state,
                                const HyperParams& hp) {
    if (!params.same_shapes(avg_delta)) throw ShapeError("nesterov_outer_step: shape mismatch");
    if (!params.same_shapes(state.buffer)) throw ShapeError("nesterov_outer_step: momentum buffer shape mismatch");
    std::vector<float> th = params.flatten(), b = state.buffer.flatten();
    const std::vector<float> d = avg_delta.flatten();
    const size_t n = th.size();
    if (!n) return;
    DeviceBuffer<float> dth(n), dd(n), db(n);
    dth.upload(th.data(), n);
    dd.upload(d.data(), n);
    db.upload(b.data(), n);
    check(emesh_nesterov_outer_step(dth.get(), dd.get(), db.get(), n, hp.outer_lr, hp.outer_momentum, nullptr));
    cuda_check(cudaDeviceSynchronize(), "nesterov_outer_step");
    dth.download(th.data(), n);
    db.download(b.data(), n);
    params.unflatten(th);
    state.buffer.unflatten(b);
}

// optim.hpp:63
inline void adamw_step(ModelParams& params, const ModelParams& grads, AdamWState& state, const HyperParams& hp,
                       float lr_scale) {
    if (!params.same_shapes(grads)) throw ShapeError("adamw_step: params/grads shape mismatch");
    if (!params.same_shapes(state.m) || !params.same_shapes(state.v))
        throw ShapeError("adamw_step: optimizer state shape mismatch");
    if (!(lr_scale >= 0.0f && lr_scale <= 1.0f)) throw RangeError("lr_scale must be in [0,1]");
    state.step += 1;
    std::vector<float> p = params.flatten(), m = state.m.flatten(), v = state.v.flatten();
    const std::vector<float> g = grads.flatten();
    const size_t n = p.size();
    if (!n) return;
    DeviceBuffer<float> dp(n), dg(n), dm(n), dv(n);
    DeviceBuffer<uint32_t> err(1);
    dp.upload(p.data(), n);
    dg.upload(g.data(), n);
    dm.upload(m.data(), n);
    dv.upload(v.data(), n);
    cuda_check(cudaMemset(err.get(), 0, sizeof(uint32_t)), "memset");
    check(emesh_adamw_step(dp.get(), dg.get(), dm.get(), dv.get(), n, state.step, hp.inner_lr, lr_scale, hp.beta1,
                           hp.beta2, hp.eps, hp.weight_decay, err.get(), nullptr));
    uint32_t bad = 0;
    cuda_check(cudaDeviceSynchronize(), "adamw_step");
    err.download(&bad, 1);
    if (bad) throw NumericError("non-finite gradient");
    dp.download(p.data(), n);
    dm.download(m.data(), n);
    dv.download(v.data(), n);
    params.unflatten(p);
    state.m.unflatten(m);
    state.v.unflatten(v);
}

// ---------------------------------------------------------------- allreduce.hpp / trainer.hpp

// One ring position (RingPlan.self_index of plan.order.size() processes, one
// GPU each), or all k workers on this GPU (`local_workers` = k). The ring is
// RingPlan::order; the segmentation is ReduceOptions::pipeline_subchunks; the
// mode is fixed per engine (ReduceJob.mode must match).
class RingEngine {
public:
    RingEngine(uint64_t n, const RingPlan& plan, const ReduceOptions& opts, ReduceMode mode,
               const uint8_t* nccl_id /* 128 B, rank 0's emesh_nccl_unique_id; nullptr when local */,
               uint32_t local_workers = 1, int device = -1)
        : n_(n), k_(static_cast<uint32_t>(plan.order.size())), mode_(mode),
          workers_(local_workers > 1 ? local_workers : 1), order_(plan.order), plan_epoch_(plan.epoch) {
        emesh_engine_config cfg{};
        cfg.n = n;
        cfg.k = k_;
        cfg.rank = plan.self_index;
        cfg.pipeline_subchunks = opts.pipeline_subchunks;
        cfg.virtual_workers = local_workers > 1 ? local_workers : 0;
        cfg.nccl_id = nccl_id;
        cfg.device = device;
        cfg.transport = EMESH_TRANSPORT_AUTO;
        cfg.reduce_fp32 = mode == ReduceMode::fp32 ? 1u : 0u;
        cfg.step_timeout_s = opts.step_timeout;
        cfg.plan_epoch = plan.epoch;
        S_ = opts.pipeline_subchunks ? opts.pipeline_subchunks : 4;
        check(emesh_engine_create(&cfg, &e_));
    }
    RingEngine(const RingEngine&) = delete;
    RingEngine& operator=(const RingEngine&) = delete;
    ~RingEngine() { emesh_engine_destroy(e_); }

    emesh_engine* handle() const { return e_; }

    // allreduce.hpp:314 on host vectors: the mean every rank decodes. jobs has
    // one entry per local worker; each input is left untouched (:47-48).
    std::vector<std::vector<float>> ring_allreduce(const std::vector<ReduceJob>& jobs) {
        if (jobs.size() != workers_) throw ShapeError("ring_allreduce: one job per local worker");
        std::vector<const float*> pin;
        std::vector<float*> pout;
        std::vector<std::vector<float>> res(workers_);
        for (const ReduceJob& j : jobs) {
            if (j.mode != mode_) throw ConfigError("ring_allreduce: job mode differs from the engine's");
            if (j.input.size() != n_) throw ShapeError("ring_allreduce: input size differs from the plan");
        }
        struct Bufs {
            std::vector<DeviceBuffer<float>*> v;
            ~Bufs() { for (auto* b : v) delete b; }
        } own;
        for (uint32_t w = 0; w < workers_; ++w) {
            auto* bi = new DeviceBuffer<float>(n_);
            auto* bo = new DeviceBuffer<float>(n_);
            own.v.push_back(bi);
            own.v.push_back(bo);
            if (n_) bi->upload(jobs[w].input.data(), n_);
            pin.push_back(bi->get());
            pout.push_back(bo->get());
        }
        round_check(emesh_engine_ring_allreduce(e_, pin.data(), pout.data(), nullptr));
        round_check(emesh_engine_check(e_));
        for (uint32_t w = 0; w < workers_; ++w) {
            res[w].resize(n_);
            if (n_) cuda_check(cudaMemcpy(res[w].data(), pout[w], n_ * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
        }
        return res;
    }

    // trainer.hpp:355-382 for each local worker: delta = retained - local ->
    // ring all-reduce -> Nesterov on retained with the mean; local = retained.
    void outer_sync(std::vector<ModelParams*> retained, std::vector<ModelParams*> local,
                    std::vector<NesterovState*> outer, const HyperParams& hp) {
        if (retained.size() != workers_ || local.size() != workers_ || outer.size() != workers_)
            throw ShapeError("outer_sync: one entry per local worker");
        std::vector<std::vector<float>> g(workers_), l(workers_), b(workers_);
        std::vector<float*> pg, pl, pb;
        for (uint32_t w = 0; w < workers_; ++w) {
            g[w] = retained[w]->flatten();
            l[w] = local[w]->flatten();
            b[w] = outer[w]->buffer.flatten();
            if (g[w].size() != n_ || l[w].size() != n_ || b[w].size() != n_)
                throw ShapeError("outer_sync: parameter count differs from the plan");
            pg.push_back(g[w].data());
            pl.push_back(l[w].data());
            pb.push_back(b[w].data());
        }
        round_check(emesh_engine_outer_sync_host(e_, pg.data(), pl.data(), pb.data(), hp.outer_lr, hp.outer_momentum, 1));
        for (uint32_t w = 0; w < workers_; ++w) {
            retained[w]->unflatten(g[w]);
            local[w]->unflatten(l[w]);
            outer[w]->buffer.unflatten(b[w]);
        }
    }

    // Wire interop: the reference's wire payload of every
    // segment of chunk c after the last round, i.e. encode_slice(mean, int8)
    // (allreduce.hpp:153-157, quant.hpp:102-131) — the bytes the reference's
    // all-gather forwards, ready for ring_detail::encode_chunk_msg over TCP.
    std::vector<Bytes> final_payloads(uint32_t chunk, uint32_t worker = 0) const {
        if (mode_ != ReduceMode::int8) throw ConfigError("final_payloads: int8 engines only");
        if (chunk >= k_) throw ShapeError("final_payloads: no such chunk");
        const uint64_t nseg = emesh_engine_segments(e_, nullptr, nullptr);
        std::vector<uint64_t> lo(nseg), len(nseg);
        emesh_engine_segments(e_, lo.data(), len.data());
        std::vector<uint8_t> codes(n_ + 16);
        std::vector<float> cbs(nseg * QuantChunk::kBuckets);
        check(emesh_engine_payload_host(e_, worker, codes.data(), cbs.data(), nullptr));
        // chunk-major segment table: chunk c holds split(n, k)[c] cut into min(S, len) subs
        uint64_t first = 0;
        for (uint32_t c = 0; c < chunk; ++c) first += subs_in_chunk(c);
        std::vector<Bytes> out;
        for (uint64_t s = first; s < first + subs_in_chunk(chunk); ++s) {
            if (len[s] == 0) { out.emplace_back(); continue; }  // empty slices travel empty (allreduce.hpp:153)
            QuantChunk q;
            q.codebook.assign(cbs.begin() + s * QuantChunk::kBuckets, cbs.begin() + (s + 1) * QuantChunk::kBuckets);
            q.indices.assign(codes.begin() + lo[s], codes.begin() + lo[s] + len[s]);
            out.push_back(b200::encode_quant_chunk(q));
        }
        return out;
    }

    // A round's status as the reference raises it (allreduce.hpp:466-472): RingFailureError naming
    // the culprit node of the plan (emesh_engine_failed_rank), StalePlanError, or check()'s mapping.
    // A failed round committed nothing (the engine's commit gate), so a retry restarts from the
    // same retained / local / momentum state.
    void round_check(int rc) const {
        if (rc == EMESH_ERING) {
            const int who = emesh_engine_failed_rank(e_);
            throw RingFailureError(who >= 0 && static_cast<size_t>(who) < order_.size() ? order_[who] : std::string(),
                                   emesh_last_error());
        }
        if (rc == EMESH_ESTALE) throw StalePlanError(plan_epoch_ + 1, emesh_last_error());
        check(rc);
    }

private:
    uint64_t subs_in_chunk(uint32_t c) const {
        const uint64_t clen = n_ / k_ + (c < n_ % k_ ? 1 : 0);
        return clen == 0 ? 1 : std::min<uint64_t>(S_, clen);
    }

    emesh_engine* e_ = nullptr;
    uint64_t S_ = 4;
    uint64_t n_;
    uint32_t k_;
    ReduceMode mode_;
    uint32_t workers_;
    std::vector<std::string> order_;
    uint32_t plan_epoch_ = 0;
};

// allreduce.hpp:485-518 `allreduce_with_retry` over GPU ring engines:
// builds one engine per membership epoch (make_engine(plan) -> an engine
// with ring_allreduce(std::vector<ReduceJob>) like b200::RingEngine; the
// caller exchanges the NCCL id among plan.order), reports the culprit of a
// RingFailureError, waits for the mesh to commit the eviction and restarts
// from the preserved input; a StalePlanError refetches the mesh. `mesh` is
// the reference's MeshClient (report_failure, wait_epoch_change, fetch_mesh)
// or anything with those members.
template <class MakeEngine, class Mesh>
RetryResult allreduce_with_retry(MakeEngine&& make_engine, Mesh& mesh, MeshState mesh_state, const std::string& self_id,
                                 const ReduceJob& job, const ReduceOptions& opts) {
    uint32_t failures = 0;
    for (;;) {
        if (mesh_state.find(self_id) == nullptr) throw FatalError("this node is no longer in the mesh");
        if (mesh_state.members.size() < 1) throw FatalError("no participants left");
        RingPlan plan = RingPlan::from_mesh(mesh_state, self_id, job.id);
        try {
            auto engine = make_engine(plan);
            RetryResult out;
            out.value = std::move(engine->ring_allreduce(std::vector<ReduceJob>{job})[0]);
            out.participants = static_cast<uint32_t>(plan.order.size());
            out.attempts = failures;
            out.epoch = mesh_state.epoch;
            return out;
        } catch (const RingFailureError& rf) {
            failures += 1;
            if (failures > opts.max_retries) throw FatalError("all-reduce retries exhausted: " + std::string(rf.what()));
            if (!rf.failed_node.empty() && rf.failed_node != self_id) mesh.report_failure(rf.failed_node);
            try {
                mesh_state = mesh.wait_epoch_change(mesh_state.epoch, opts.evict_wait);
            } catch (const TimeoutError&) {
                mesh_state = mesh.fetch_mesh();  // maybe it changed and we missed it
            }
        } catch (const StalePlanError&) {
            failures += 1;
            if (failures > opts.max_retries) throw FatalError("all-reduce retries exhausted");
            mesh_state = mesh.fetch_mesh();
        }
    }
}

}  // namespace emesh::b200
