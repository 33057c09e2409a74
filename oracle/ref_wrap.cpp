// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shims over the UNMODIFIED reference library (header-only C++20,
// /root/reference/proj/include/emesh). oracle/Makefile compiles this file
// against the reference headers where they lie, with the reference's own
// RelWithDebInfo flags (-O2 -g -DNDEBUG -std=gnu++20, no -march: no FMA,
// proj/CMakeLists.txt:3-9), into oracle/_ref/libemesh_ref.so. Python tests
// and bench.py's reference arm load it through oracle/pyoracle.py.
//
// Error convention: 0 ok, 1 ShapeError, 2 NumericError, 3 DecodeError,
// 9 any other emesh::Error / std::exception.
#include <arpa/inet.h>
#include <netinet/in.h>
#include <sys/socket.h>
#include <unistd.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "emesh/allreduce.hpp"
#include "emesh/checkpoint.hpp"
#include "emesh/optim.hpp"
#include "emesh/quant.hpp"
#include "emesh/sha256.hpp"
#include "emesh/sim.hpp"
#include "emesh/tcp.hpp"
#include "emesh/tensor.hpp"

using namespace emesh;

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError&) {
        return 1;
    } catch (const NumericError&) {
        return 2;
    } catch (const DecodeError&) {
        return 3;
    } catch (const std::exception&) {
        return 9;
    }
}

ModelParams single_tensor(const float* p, uint64_t n) {
    ModelParams m;
    m.add("w", Tensor({static_cast<uint32_t>(n)}, std::vector<float>(p, p + n)));
    return m;
}

// Reserve k distinct ephemeral ports for a TCP ring (the TcpEnv ctor takes
// its peer list up front, and a ring has no construction order without one).
std::vector<uint16_t> free_ports(size_t k) {
    std::vector<int> fds;
    std::vector<uint16_t> ports;
    for (size_t i = 0; i < k; ++i) {
        int fd = ::socket(AF_INET, SOCK_STREAM, 0);
        sockaddr_in sa{};
        sa.sin_family = AF_INET;
        sa.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
        sa.sin_port = 0;
        ::bind(fd, reinterpret_cast<sockaddr*>(&sa), sizeof sa);
        socklen_t len = sizeof sa;
        ::getsockname(fd, reinterpret_cast<sockaddr*>(&sa), &len);
        ports.push_back(ntohs(sa.sin_port));
        fds.push_back(fd);
    }
    for (int fd : fds) ::close(fd);
    return ports;
}

}  // namespace

extern "C" {

int ref_quantize(const float* x, uint64_t n, uint8_t* codes, float* cb) {
    return guarded([&] {
        QuantChunk q = quantize(std::span<const float>(x, n));
        std::memcpy(codes, q.indices.data(), n);
        std::memcpy(cb, q.codebook.data(), 256 * sizeof(float));
    });
}

int ref_dequantize(const uint8_t* codes, const float* cb, uint64_t n, float* out) {
    return guarded([&] {
        QuantChunk q;
        q.codebook.assign(cb, cb + 256);
        q.indices.assign(codes, codes + n);
        dequantize_into(q, std::span<float>(out, n));
    });
}

int ref_encode_quant_chunk(const uint8_t* codes, const float* cb, uint64_t n, uint8_t* out,
                           uint64_t* out_len) {
    return guarded([&] {
        QuantChunk q;
        q.codebook.assign(cb, cb + 256);
        q.indices.assign(codes, codes + n);
        Bytes b = encode_quant_chunk(q);
        std::memcpy(out, b.data(), b.size());
        *out_len = b.size();
    });
}

int ref_decode_quant_chunk(const uint8_t* buf, uint64_t len, uint8_t* codes, float* cb,
                           uint64_t* count) {
    return guarded([&] {
        QuantChunk q = decode_quant_chunk(Bytes(buf, buf + len));
        std::memcpy(codes, q.indices.data(), q.indices.size());
        std::memcpy(cb, q.codebook.data(), 256 * sizeof(float));
        *count = q.indices.size();
    });
}

int ref_pseudo_gradient(const float* prev, const float* local, uint64_t n, float* out) {
    return guarded([&] {
        ModelParams d = compute_pseudo_gradient(single_tensor(prev, n), single_tensor(local, n));
        std::memcpy(out, d.entries[0].second.data.data(), n * sizeof(float));
    });
}

int ref_nesterov(float* theta, const float* avg, float* buf, uint64_t n, float lr, float momentum) {
    return guarded([&] {
        HyperParams hp;
        hp.outer_lr = lr;
        hp.outer_momentum = momentum;
        ModelParams p = single_tensor(theta, n);
        NesterovState st;
        st.buffer = single_tensor(buf, n);
        nesterov_outer_step(p, single_tensor(avg, n), st, hp);
        std::memcpy(theta, p.entries[0].second.data.data(), n * sizeof(float));
        std::memcpy(buf, st.buffer.entries[0].second.data.data(), n * sizeof(float));
    });
}

int ref_adamw(float* p, const float* g, float* m, float* v, uint64_t n, uint64_t step_before, float inner_lr,
              float lr_scale, float beta1, float beta2, float eps, float weight_decay) {
    return guarded([&] {
        HyperParams hp;
        hp.inner_lr = inner_lr;
        hp.beta1 = beta1;
        hp.beta2 = beta2;
        hp.eps = eps;
        hp.weight_decay = weight_decay;
        ModelParams params = single_tensor(p, n);
        AdamWState st;
        st.step = step_before;
        st.m = single_tensor(m, n);
        st.v = single_tensor(v, n);
        adamw_step(params, single_tensor(g, n), st, hp, lr_scale);
        std::memcpy(p, params.entries[0].second.data.data(), n * sizeof(float));
        std::memcpy(m, st.m.entries[0].second.data.data(), n * sizeof(float));
        std::memcpy(v, st.v.entries[0].second.data.data(), n * sizeof(float));
    });
}

// ring_allreduce over the deterministic simulator (allreduce.hpp:314 via
// the same driver shape as the reference test harness). outs: k*n floats.
int ref_ring_allreduce_sim(const float* const* inputs, uint32_t k, uint64_t n, uint32_t S,
                           int mode, int pipelined, float* outs, uint64_t* bytes_sent) {
    return guarded([&] {
        SimWorld w;
        w.set_default_link({1e9, 1e-4, {}});
        MeshState mesh;
        mesh.epoch = 1;
        for (uint32_t i = 0; i < k; ++i) {
            std::string id = "n" + std::to_string(i);
            mesh.members.push_back({id, i, i});
            mesh.ring.push_back(id);
        }
        ReduceOptions opts;
        opts.pipeline_subchunks = S;
        opts.pipelined = pipelined != 0;
        std::mutex mu;
        for (uint32_t i = 0; i < k; ++i) {
            std::string id = "n" + std::to_string(i);
            std::vector<float> input(inputs[i], inputs[i] + n);
            w.spawn(id, "node-" + id, [&, i, id, input] {
                Env env = w.env(id);
                RingIO io(env);
                env.rt->sleep_for(0.01);
                RingPlan plan = RingPlan::from_mesh(mesh, id, 1);
                ReduceJob job{1, input, mode ? ReduceMode::int8 : ReduceMode::fp32};
                auto out = ring_allreduce(env, io, plan, job, opts);
                std::lock_guard<std::mutex> g(mu);
                std::memcpy(outs + static_cast<size_t>(i) * n, out.data(), n * sizeof(float));
                if (bytes_sent) bytes_sent[i] = env.net->bytes_sent();
            });
        }
        w.run();
    });
}

// One full outer-sync round of the reference over real TCP loopback with k
// node threads in this process: per node compute_pseudo_gradient ->
// flatten -> ring_allreduce -> unflatten -> nesterov_outer_step
// (trainer.hpp:355-382, minus barrier/hash/checkpoint bookkeeping).
// theta_g (n) and buf (n) are updated in place from node 0's result; every
// node's copy is checked bit-identical (returns 9 if not). seconds[0] =
// wall time of the round (max over nodes, barrier-aligned start).
int ref_outer_sync_tcp(float* theta_g, const float* const* theta_l, float* buf, uint32_t k,
                       uint64_t n, uint32_t S, int mode, float lr, float momentum,
                       double* seconds) {
    return guarded([&] {
        std::vector<uint16_t> ports = free_ports(k);
        std::vector<std::unique_ptr<TcpEnv>> envs;
        for (uint32_t i = 0; i < k; ++i) {
            uint32_t succ = (i + 1) % k;
            std::vector<PeerAddr> peers;
            if (k > 1) peers.push_back({"n" + std::to_string(succ), "127.0.0.1", ports[succ]});
            envs.emplace_back(std::make_unique<TcpEnv>("n" + std::to_string(i), ports[i], peers));
        }
        MeshState mesh;
        mesh.epoch = 1;
        for (uint32_t i = 0; i < k; ++i) {
            std::string id = "n" + std::to_string(i);
            mesh.members.push_back({id, i, i});
            mesh.ring.push_back(id);
        }
        ReduceOptions opts;
        opts.pipeline_subchunks = S;
        opts.step_timeout = 600.0;
        HyperParams hp;
        hp.outer_lr = lr;
        hp.outer_momentum = momentum;

        std::vector<ModelParams> results(k);
        std::vector<ModelParams> bufs(k);
        std::vector<std::string> errors(k);
        std::vector<double> elapsed(k, 0.0);
        std::vector<std::unique_ptr<RingIO>> ios(k);
        for (uint32_t i = 0; i < k; ++i) {
            Env env{envs[i].get(), envs[i].get()};
            ios[i] = std::make_unique<RingIO>(env);
        }
        std::vector<ModelParams> retained(k), local(k);
        for (uint32_t i = 0; i < k; ++i) {
            retained[i] = single_tensor(theta_g, n);
            local[i] = single_tensor(theta_l[i], n);
            bufs[i] = single_tensor(buf, n);
        }
        std::mutex mu;
        std::condition_variable cv;
        uint32_t ready = 0;
        std::vector<std::thread> threads;
        for (uint32_t i = 0; i < k; ++i) {
            threads.emplace_back([&, i] {
                try {
                    Env env{envs[i].get(), envs[i].get()};
                    RingPlan plan = RingPlan::from_mesh(mesh, "n" + std::to_string(i), 1);
                    {
                        std::unique_lock<std::mutex> l(mu);
                        ++ready;
                        cv.notify_all();
                        cv.wait(l, [&] { return ready == k; });
                    }
                    auto t0 = std::chrono::steady_clock::now();
                    ModelParams delta = compute_pseudo_gradient(retained[i], local[i]);
                    ReduceJob job{1, delta.flatten(), mode ? ReduceMode::int8 : ReduceMode::fp32};
                    std::vector<float> avgv = ring_allreduce(env, *ios[i], plan, job, opts);
                    ModelParams avg = delta;  // same shapes
                    avg.unflatten(avgv);
                    NesterovState st;
                    st.buffer = std::move(bufs[i]);
                    nesterov_outer_step(retained[i], avg, st, hp);
                    bufs[i] = std::move(st.buffer);
                    auto t1 = std::chrono::steady_clock::now();
                    elapsed[i] = std::chrono::duration<double>(t1 - t0).count();
                } catch (const std::exception& e) {
                    errors[i] = e.what();
                }
            });
        }
        for (auto& t : threads) t.join();
        for (auto& io : ios) io->shutdown();
        for (uint32_t i = 0; i < k; ++i)
            if (!errors[i].empty()) throw FatalError("node " + std::to_string(i) + ": " + errors[i]);
        for (uint32_t i = 1; i < k; ++i)
            if (std::memcmp(retained[i].entries[0].second.data.data(),
                            retained[0].entries[0].second.data.data(), n * sizeof(float)) != 0)
                throw FatalError("replicas diverged");
        std::memcpy(theta_g, retained[0].entries[0].second.data.data(), n * sizeof(float));
        std::memcpy(buf, bufs[0].entries[0].second.data.data(), n * sizeof(float));
        double mx = 0;
        for (double e : elapsed) mx = e > mx ? e : mx;
        if (seconds) seconds[0] = mx;
    });
}

}  // extern "C"

// ---- checkpoints (tensor.hpp:111-161, checkpoint.hpp:19-68,190-224) ----
// A Checkpoint assembled from flat arrays: names[nt], ranks[nt], extents
// (sum ranks), sets[5] = params, retained, inner.m, inner.v, outer.buffer
// (each the concatenated tensor data in order).
static Checkpoint ck_from_flat(uint64_t outer_step, uint32_t nt, const char* const* names, const uint32_t* ranks,
                               const uint32_t* extents, const float* const* sets, uint64_t adam_step,
                               uint64_t rng_seed, uint64_t data_counter, uint32_t shard, const uint8_t* hash) {
    Checkpoint ck;
    ModelParams* ps[5] = {&ck.params, &ck.retained, &ck.inner.m, &ck.inner.v, &ck.outer.buffer};
    for (int s = 0; s < 5; ++s) {
        uint64_t e = 0, off = 0;
        for (uint32_t i = 0; i < nt; ++i) {
            std::vector<uint32_t> shape(extents + e, extents + e + ranks[i]);
            e += ranks[i];
            size_t n = Tensor::element_count(shape);
            ps[s]->add(names[i], Tensor(shape, std::vector<float>(sets[s] + off, sets[s] + off + n)));
            off += n;
        }
    }
    ck.outer_step = outer_step;
    ck.inner.step = adam_step;
    ck.rng_seed = rng_seed;
    ck.data_counter = data_counter;
    ck.shard = shard;
    std::memcpy(ck.config_hash.data(), hash, 32);
    return ck;
}

// Flat view of a decoded Checkpoint: scalars[5] = outer_step, inner.step,
// rng_seed, data_counter, shard; sets[s] receive numel floats each (numel_cap).
static void ck_to_flat(const Checkpoint& ck, float* const* sets, uint64_t numel_cap, uint64_t* scalars,
                       uint8_t* hash) {
    const ModelParams* ps[5] = {&ck.params, &ck.retained, &ck.inner.m, &ck.inner.v, &ck.outer.buffer};
    for (int s = 0; s < 5; ++s) {
        uint64_t off = 0;
        for (const auto& [n, t] : ps[s]->entries) {
            if (off + t.size() > numel_cap) throw Error("numel_cap too small");
            if (sets && sets[s]) std::memcpy(sets[s] + off, t.data.data(), t.size() * sizeof(float));
            off += t.size();
        }
    }
    scalars[0] = ck.outer_step;
    scalars[1] = ck.inner.step;
    scalars[2] = ck.rng_seed;
    scalars[3] = ck.data_counter;
    scalars[4] = ck.shard;
    std::memcpy(hash, ck.config_hash.data(), 32);
}

template <typename F>
static int guarded_msg(char* msg, uint64_t cap, F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        std::snprintf(msg, cap, "%s", e.what());
        return 1;
    } catch (const NumericError& e) {
        std::snprintf(msg, cap, "%s", e.what());
        return 2;
    } catch (const DecodeError& e) {
        std::snprintf(msg, cap, "%s", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::snprintf(msg, cap, "%s", e.what());
        return 9;
    }
}

extern "C" {

int ref_encode_checkpoint(uint64_t outer_step, uint32_t nt, const char* const* names, const uint32_t* ranks,
                          const uint32_t* extents, const float* const* sets, uint64_t adam_step, uint64_t rng_seed,
                          uint64_t data_counter, uint32_t shard, const uint8_t* hash, uint8_t* out, uint64_t cap,
                          uint64_t* len) {
    return guarded([&] {
        Bytes b = encode_checkpoint(ck_from_flat(outer_step, nt, names, ranks, extents, sets, adam_step, rng_seed,
                                                 data_counter, shard, hash));
        *len = b.size();
        if (b.size() > cap) throw Error("cap");
        std::memcpy(out, b.data(), b.size());
    });
}

int ref_decode_checkpoint(const uint8_t* buf, uint64_t len, float* const* sets, uint64_t numel_cap,
                          uint64_t* scalars, uint8_t* hash, char* msg, uint64_t msg_cap) {
    return guarded_msg(msg, msg_cap, [&] {
        Bytes b(buf, buf + len);
        ck_to_flat(decode_checkpoint(b), sets, numel_cap, scalars, hash);
    });
}

int ref_write_checkpoint_file(const char* path, uint64_t outer_step, uint32_t nt, const char* const* names,
                              const uint32_t* ranks, const uint32_t* extents, const float* const* sets,
                              uint64_t adam_step, uint64_t rng_seed, uint64_t data_counter, uint32_t shard,
                              const uint8_t* hash) {
    return guarded([&] {
        write_checkpoint_file(path, ck_from_flat(outer_step, nt, names, ranks, extents, sets, adam_step, rng_seed,
                                                 data_counter, shard, hash));
    });
}

int ref_read_checkpoint_file(const char* path, float* const* sets, uint64_t numel_cap, uint64_t* scalars,
                             uint8_t* hash, char* msg, uint64_t msg_cap) {
    return guarded_msg(msg, msg_cap, [&] { ck_to_flat(read_checkpoint_file(path), sets, numel_cap, scalars, hash); });
}

int ref_sha256(const uint8_t* p, uint64_t n, uint8_t* out) {
    auto d = Sha256::hash(p, n);
    std::memcpy(out, d.data(), 32);
    return 0;
}

}  // extern "C"
