// emesh::b200::allreduce_with_retry (include/emesh_b200.hpp) against the
// reference's retry contract (allreduce.hpp:485-518; tests
// test_allreduce.cpp:416-481): scripted engines fail a membership epoch with
// RingFailureError(culprit) / StalePlanError, a scripted mesh evicts the
// reported culprit; survivors must return the survivor mean of the
// untouched inputs, with the right participant / attempt counts, and the
// retry cap must end in FatalError. Host-only (no GPU): the engine factory is
// the scripted one, exactly as the reference's ChurnHarness scripts SimWorld.
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "emesh/rng.hpp"
#include "emesh_b200.hpp"

using namespace emesh;

static int g_fail = 0;
#define EXPECT(c, ...)                                       \
    do {                                                     \
        if (!(c)) {                                          \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                        \
            std::printf("\n");                               \
            ++g_fail;                                        \
        }                                                    \
    } while (0)

// The scripted world: every node's input, and per plan epoch an optional failure.
struct World {
    std::map<std::string, std::vector<float>> inputs;
    struct Failure { bool stale = false; std::string culprit; };
    std::map<uint32_t, Failure> fail_at;  // plan epoch -> failure of that attempt
    int attempts = 0;
};

// One attempt's engine: the mean over the plan's members (what every rank decodes).
struct FakeEngine {
    World* w;
    RingPlan plan;
    std::vector<std::vector<float>> ring_allreduce(const std::vector<ReduceJob>& jobs) {
        ++w->attempts;
        auto f = w->fail_at.find(plan.epoch);
        if (f != w->fail_at.end()) {
            if (f->second.stale) throw StalePlanError(plan.epoch + 1, "newer plan epoch on the ring");
            throw RingFailureError(f->second.culprit, "ring peer lost");
        }
        const size_t n = jobs[0].input.size();
        std::vector<float> sum(n, 0.f);
        for (const auto& id : plan.order)
            for (size_t i = 0; i < n; ++i) sum[i] += w->inputs[id][i];
        for (auto& v : sum) v /= static_cast<float>(plan.order.size());
        return {sum};
    }
};

// The scripted membership service (the reference's MeshClient surface).
struct FakeMesh {
    MeshState state;
    std::vector<std::string> reported;
    bool stale_refetch = false;
    void report_failure(const std::string& node) {
        reported.push_back(node);
        MeshState next = state;
        next.epoch += 1;
        next.members.clear();
        next.ring.clear();
        for (const auto& m : state.members)
            if (m.id != node) next.members.push_back(m);
        for (const auto& id : state.ring)
            if (id != node) next.ring.push_back(id);
        state = next;
    }
    MeshState wait_epoch_change(uint64_t epoch, double) {
        if (state.epoch == epoch) throw TimeoutError("no epoch change");
        return state;
    }
    MeshState fetch_mesh() {
        stale_refetch = true;
        return state;
    }
};

static MeshState mesh_of(int k) {
    MeshState s;
    s.epoch = 1;
    for (int i = 0; i < k; ++i) {
        MeshMember m;
        m.id = "w" + std::to_string(i);
        m.rank = static_cast<uint32_t>(i);
        s.members.push_back(m);
        s.ring.push_back(m.id);
    }
    return s;
}

static std::vector<float> seeded(int seed, int node, size_t n) {
    std::vector<float> v(n);
    for (size_t i = 0; i < n; ++i) v[i] = rng_uniform(seed, node, 0, i);
    return v;
}

int main() {
    const size_t n = 4096;
    ReduceOptions opts;
    opts.pipeline_subchunks = 4;
    auto run = [&](World& w, FakeMesh& mesh, const std::string& self, uint32_t max_retries, RetryResult* out,
                   std::string* fatal) {
        ReduceJob job;
        job.id = 7;
        job.input = w.inputs[self];
        job.mode = ReduceMode::fp32;
        ReduceOptions o = opts;
        o.max_retries = max_retries;
        try {
            *out = b200::allreduce_with_retry(
                [&](const RingPlan& plan) { return std::make_unique<FakeEngine>(FakeEngine{&w, plan}); }, mesh,
                mesh.state, self, job, o);
        } catch (const FatalError& e) {
            *fatal = e.what();
        }
        return job;
    };
    {   // no failure: the plain result (test_allreduce.cpp:416-429)
        World w;
        for (int i = 0; i < 3; ++i) w.inputs["w" + std::to_string(i)] = seeded(55, i, n);
        FakeMesh mesh{mesh_of(3)};
        RetryResult r;
        std::string fatal;
        run(w, mesh, "w0", 5, &r, &fatal);
        EXPECT(fatal.empty(), "no-failure run died: %s", fatal.c_str());
        EXPECT(r.participants == 3 && r.attempts == 0 && r.epoch == 1, "plain result counts");
    }
    {   // mid-collective crash of w2: survivor mean, the culprit reported (:431-446)
        World w;
        for (int i = 0; i < 4; ++i) w.inputs["w" + std::to_string(i)] = seeded(66, i, n);
        w.fail_at[1] = {false, "w2"};
        FakeMesh mesh{mesh_of(4)};
        RetryResult r;
        std::string fatal;
        const ReduceJob job = run(w, mesh, "w0", 5, &r, &fatal);
        EXPECT(fatal.empty(), "crash run died: %s", fatal.c_str());
        EXPECT(r.participants == 3 && r.attempts == 1 && r.epoch == 2, "survivor counts %u %u %llu", r.participants,
               r.attempts, (unsigned long long)r.epoch);
        EXPECT(mesh.reported.size() == 1 && mesh.reported[0] == "w2", "culprit reported");
        std::vector<float> want(n, 0.f);
        for (const char* id : {"w0", "w1", "w3"})
            for (size_t i = 0; i < n; ++i) want[i] += w.inputs[id][i];
        for (auto& v : want) v /= 3.f;
        EXPECT(std::memcmp(r.value.data(), want.data(), 4 * n) == 0, "survivor mean");
        EXPECT(job.input == w.inputs["w0"], "input preserved across retries (:472-481)");
    }
    {   // two sequential crashes: 2-way mean after two retries (:448-462)
        World w;
        for (int i = 0; i < 4; ++i) w.inputs["w" + std::to_string(i)] = seeded(67, i, n);
        w.fail_at[1] = {false, "w1"};
        w.fail_at[2] = {false, "w2"};
        FakeMesh mesh{mesh_of(4)};
        RetryResult r;
        std::string fatal;
        run(w, mesh, "w3", 5, &r, &fatal);
        EXPECT(fatal.empty(), "two-crash run died: %s", fatal.c_str());
        EXPECT(r.participants == 2 && r.attempts == 2, "two-crash counts");
    }
    {   // retry cap exhaustion is fatal with diagnostics (:464-471)
        World w;
        for (int i = 0; i < 3; ++i) w.inputs["w" + std::to_string(i)] = seeded(68, i, n);
        w.fail_at[1] = {false, "w1"};
        w.fail_at[2] = {false, "w2"};
        FakeMesh mesh{mesh_of(3)};
        RetryResult r;
        std::string fatal;
        run(w, mesh, "w0", 1, &r, &fatal);
        EXPECT(fatal.find("retries") != std::string::npos, "cap exhaustion must be fatal: '%s'", fatal.c_str());
    }
    {   // StalePlanError: refetch the mesh and retry (allreduce.hpp:512-515)
        World w;
        for (int i = 0; i < 3; ++i) w.inputs["w" + std::to_string(i)] = seeded(70, i, n);
        w.fail_at[1] = {true, ""};
        FakeMesh mesh{mesh_of(3)};
        RetryResult r;
        std::string fatal;
        // a stale plan does not change the epoch here; the refetch hands back the same mesh, the
        // scripted failure stays -> the cap ends it
        run(w, mesh, "w0", 2, &r, &fatal);
        EXPECT(mesh.stale_refetch, "StalePlanError must refetch the mesh");
        EXPECT(mesh.reported.empty(), "StalePlanError reports no culprit");
        EXPECT(fatal.find("retries") != std::string::npos, "stale plans exhaust the cap: '%s'", fatal.c_str());
    }
    {   // an empty culprit (timeout without a named node) is not reported; self is never reported
        World w;
        for (int i = 0; i < 3; ++i) w.inputs["w" + std::to_string(i)] = seeded(71, i, n);
        w.fail_at[1] = {false, "w0"};
        FakeMesh mesh{mesh_of(3)};
        RetryResult r;
        std::string fatal;
        run(w, mesh, "w0", 1, &r, &fatal);
        EXPECT(mesh.reported.empty(), "a node never reports itself");
    }
    if (g_fail) {
        std::printf("%d failure(s)\n", g_fail);
        return 1;
    }
    std::printf("cpp retry OK\n");
    return 0;
}
