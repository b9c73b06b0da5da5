// plan.h -- host planning helpers shared by build_plan (api.cpp) and the host-only planning API (debug_plan.cpp):
// a small persistent spin pool for the regrid's plan phases, and the three per-leaf / per-root phases of a plan
// (leaf launch order, face-neighbour table, leaf descriptors) split into parts whose outputs are merged in part order,
// so the plan is the same (bitwise) for any number of threads.
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "comm.h"
#include "device.h"
#include "tree.h"

namespace amr {

// Worker threads that spin (hot, ~0.1 us dispatch) only while the pool is ARMED -- build_plan arms it for its
// duration on large trees -- and sleep on a condition variable otherwise.  run(parts, f) executes f(0) .. f(parts - 1) on the
// calling thread and the workers (parts fetched dynamically); unarmed, in a forked child, or with one thread it runs
// them in order on the caller; a second caller while a job runs (loopback virtual ranks plan concurrently) runs its
// parts serially too.  The OpenMP team of round 1 lost to its wake-up cost at this granularity (DESIGN s7).
// Threads: AMR_HOST_THREADS (total, including the caller), default min(8, hardware threads / LOCAL_WORLD_SIZE).
class HostPool {
  public:
    static HostPool& get();
    int threads() const { return nworkers_ + 1; }
    // whether run() would use the workers (armed, with workers): parts are only worth splitting then
    bool active() const { return nworkers_ > 0 && !serial_ && armed_.load(std::memory_order_relaxed) > 0; }
    void arm();
    void disarm();
    template <class F>
    void run(int parts, F&& f) {
        struct Thunk {
            static void call(void* p, int k) { (*static_cast<F*>(p))(k); }
        };
        run_erased(parts, &Thunk::call, static_cast<void*>(&f));
    }
    // (test hook) force the serial path for the calls that follow: 1 = serial, 0 = pool as configured
    void set_serial(bool s) { serial_ = s; }

  private:
    explicit HostPool(int workers);
    struct Job {
        void (*fn)(void*, int);
        void* ctx;
        int parts;
        uint64_t id;   // generation: a later job may reuse the same stack address
        std::atomic<int> next{0}, done{0};
    };
    void worker();
    void run_erased(int parts, void (*fn)(void*, int), void* ctx);
    int nworkers_ = 0;
    int pid_ = 0;
    bool serial_ = false;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::mutex job_m_;   // one job at a time (try_lock; the loser runs serially)
    std::condition_variable cv_;
    std::atomic<int> armed_{0};
    std::atomic<Job*> cur_{nullptr};
    std::atomic<uint64_t> gen_{0};   // id of the last published job (workers spin on it read-only)
    uint64_t seq_ = 0;               // (under job_m_)
    std::atomic<int> busy_{0};
};

// build_plan arms the pool for trees of at least this many leaves (configs[3]: 13.5 k; configs[2] stays serial)
constexpr int64_t kPoolMinLeaves = 8192;

// arms the pool for a scope (build_plan of a large tree)
struct PoolArm {
    PoolArm() { HostPool::get().arm(); }
    ~PoolArm() { HostPool::get().disarm(); }
    PoolArm(const PoolArm&) = delete;
    PoolArm& operator=(const PoolArm&) = delete;
};

// Leaves of the roots root_ok accepts, per level in Morton order (PatchTree::leaves_morton_roots), concatenated
// level by level into leaf_ids (the launch order).
template <class RootOk>
void plan_leaf_order(const PatchTree& t, RootOk root_ok, std::vector<int32_t>& leaf_ids);
// nb4 of the subtrees of `roots` (PatchTree::face_neighbours_roots)
void plan_face_neighbours(const PatchTree& t, const std::vector<int32_t>& roots, std::vector<int32_t>& nb4);
// nb4 after a regrid, in O(changes) (one rank, the previous table complete): the same-level neighbours of every
// deleted slot lose it (-1, missing), then every created patch -- in level order, so that its parent's entries are
// final -- gets its entries from its parent's and its neighbours point back to it.  Equal to plan_face_neighbours
// over all roots on every active patch (AMR_CHECK_INCR=1 compares them in build_plan).
void update_face_neighbours(const PatchTree& t, const std::vector<int32_t>& created, const std::vector<int32_t>& deleted,
                            std::vector<int32_t>& nb4);

// Leaf descriptors (LeafDesc), proxy-strip tasks (ProxyTask, numbered in leaf order) and reflux tasks of the leaves
// in leaf_ids order, from the face-neighbour table nb4.  halo_mode 2 with world > 1 marks remote face neighbours
// (LeafDesc.pad).  Returns false with err set (the first failing leaf in leaf order) on a mesh inconsistency.
struct DescOut {
    std::vector<LeafDesc> leaves;
    std::vector<ProxyTask> ptasks;
    std::vector<RefluxTask> rtasks;
};
bool plan_descriptors(const PatchTree& t, const std::vector<int32_t>& nb4, const std::vector<int32_t>& leaf_ids,
                      const Owners& owner, int world, int rank, int halo_mode, DescOut& out, std::string& err);

// ---------------------------------------------------------------- template definitions
template <class RootOk>
void plan_leaf_order(const PatchTree& t, RootOk root_ok, std::vector<int32_t>& leaf_ids) {
    HostPool& pool = HostPool::get();
    const std::vector<int32_t>& rm = t.root_morton();
    const int parts = pool.active() ? std::max(1, std::min<int>(16 * pool.threads(), (int)rm.size())) : 1;   // (refinement is clustered)
    // per-part, per-level scratch kept across plans (thread_local: loopback virtual ranks plan concurrently)
    static thread_local std::vector<std::vector<std::vector<int32_t>>> per;
    static thread_local std::vector<std::vector<int32_t>> stacks;
    // (the parts run on the workers: they use the caller's scratch through these references, not their own
    // thread_local instances)
    std::vector<std::vector<std::vector<int32_t>>>& P = per;
    std::vector<std::vector<int32_t>>& S = stacks;
    if ((int)P.size() < parts) P.resize(parts);
    if ((int)S.size() < parts) S.resize(parts);
    const size_t nr = rm.size();
    pool.run(parts, [&](int k) {
        const size_t r0 = nr * k / parts, r1 = nr * (k + 1) / parts;
        t.leaves_morton_span(r0, r1, P[k], [](int) { return true; }, root_ok, S[k]);
    });
    leaf_ids.clear();
    for (int l = 0; l < t.levels; ++l)
        for (int k = 0; k < parts; ++k) leaf_ids.insert(leaf_ids.end(), P[k][l].begin(), P[k][l].end());
}

}  // namespace amr
