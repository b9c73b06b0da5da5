// ctx.h -- the library context behind the opaque amr_ctx handle (include/amr.h).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/amr.h"
#include "comm.h"
#include "device.h"
#include "tree.h"

namespace amr {

template <class T>
struct DevArray {
    T* p = nullptr;
    size_t cap = 0, count = 0;
    bool owned = true;         // false: a view into a PlanArena (not freed here)
    DevArray() = default;
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept : p(o.p), cap(o.cap), count(o.count), owned(o.owned) {
        o.p = nullptr; o.cap = o.count = 0; o.owned = true;
    }
    DevArray& operator=(DevArray&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; cap = o.cap; count = o.count; owned = o.owned;
            o.p = nullptr; o.cap = o.count = 0; o.owned = true;
        }
        return *this;
    }
    ~DevArray() { release(); }   // every device / pinned buffer of a ctx is freed with it
    // point into memory owned elsewhere (the plan arena); drops an owned buffer first
    void view(T* ptr, size_t n) {
        release();
        p = ptr;
        count = n;
        owned = false;
    }
    cudaError_t upload(const std::vector<T>& v, cudaStream_t s) {
        if (!owned) { p = nullptr; cap = 0; owned = true; }
        count = v.size();
        if (v.size() > cap) {   // grow with 50 % slack: regrids that add a few patches do not reallocate
            if (p) cudaFree(p);
            p = nullptr;
            cap = std::max<size_t>(v.size() + v.size() / 2, 16);
            cudaError_t e = cudaMalloc(&p, cap * sizeof(T));
            if (e != cudaSuccess) { cap = 0; return e; }
        }
        if (v.empty()) return cudaSuccess;
        return cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    }
    // grows with 50 % slack (a proxy count growing by one must not re-allocate); slack = false for arrays sized
    // by the fixed slot capacity
    cudaError_t reserve(size_t n, bool slack = true) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = std::max<size_t>(slack ? n + n / 2 : n, 16);
        cudaError_t e = cudaMalloc(&p, cap * sizeof(T));
        if (e != cudaSuccess) cap = 0;
        return e;
    }
    void release() {
        if (p && owned) cudaFree(p);
        p = nullptr;
        cap = count = 0;
        owned = true;
    }
};

// bit interleave x0 y0 x1 y1 ... (Morton / Z order) by magic-number spreading

}  // namespace amr

using namespace amr;

// NVTX ranges (header-only NVTX v3; free when no tool is attached): host-side enqueue timeline of steps, stages,
// exchanges and regrid phases for nsys
#include <nvtx3/nvToolsExt.h>
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

struct amr_ctx {
    amr_config cfg{};
    PatchTree tree;
    int n = 0, g = 4;
    Geometry geo{};
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double* U[3] = {nullptr, nullptr, nullptr};
    void* own_pool = nullptr;
    int un = 0;
    size_t PS = 0;   // doubles per slot

    // plan (rebuilt after every mesh change)
    std::vector<int32_t> canon, canon_pos;      // canonical order; id -> tree index
    std::vector<int32_t> leaf_ids;               // launch order
    std::vector<int32_t> leaf_pos;               // id -> leaf index or -1
    std::vector<int32_t> sib;                    // sibling groups: parent id + its 4 leaf children's leaf indices
    std::vector<LeafDesc> leaves;
    std::vector<LeafDesc> gleaves, singles;        // Central4 n = 8, 16: 32 x 32 blocks of leaves / the rest
    DevArray<LeafDesc> d_gleaves, d_singles;
    std::vector<ProxyTask> ptasks;
    std::vector<RefluxTask> rtasks;
    std::vector<std::vector<RestrictTask>> rlev;  // rlev[l]: parents at level l-1 of level-l children
    DevArray<LeafDesc> d_leaves;
    DevArray<ProxyTask> d_ptasks;
    DevArray<RefluxTask> d_rtasks;
    std::vector<DevArray<RestrictTask>> d_rlev;
    // the per-plan descriptor arrays packed into ONE host buffer and ONE device buffer (one H2D copy per plan; the
    // DevArrays above are views into it)
    // host side of the plan arena: pinned (the packed upload is one DMA, no staging through pageable memory),
    // grown geometrically, never zero-filled; freed with the ctx
    char* arena_host = nullptr;
    size_t arena_host_cap = 0;
    cudaEvent_t arena_ev = nullptr;   // recorded after the arena's upload: the next fill waits for it
    DevArray<char> arena_dev;
    DevArray<ProlongTask> d_prolong;
    DevArray<double> proxy, freg, staging, d_maxeta, d_partial, unf_scratch;
    DevArray<int32_t> d_slots, d_amb, d_sib, d_flist, d_fcount;
    DevArray<int32_t> x_sidx, x_ridx;             // multi-rank exchange slot lists
    DevArray<double> x_send, x_recv;              // multi-rank exchange buffers
    int64_t leaf_cells = 0;

    // device scalars: dt, lambda bits, err[4]
    double* d_dt = nullptr;
    unsigned long long* d_lambda = nullptr;
    int32_t* d_err = nullptr;
    unsigned long long* d_tmp = nullptr;
    void* h_pinned = nullptr;   // {int32 err[4]; double dt}
    bool own_pool_nccl = false;  // own_pool from ncclMemAlloc (peer_map 1)
    void* freg_nccl = nullptr;   // flux registers from ncclMemAlloc (peer_map 1; c->freg is a view of it)
    bool lambda_valid = false;
    bool ghost_valid = false;      // proxies hold the ghost strips of U^n under the current plan (post-stage fill)
    double sim_time_fix = 0.0;     // host correction of the device time sum (rolled-back steps)
    std::vector<int32_t> nb4;      // face neighbours W, E, S, N of every slot (PatchTree::face_neighbours)
    bool nb4_full = false;         // nb4 holds every active patch's entries (one rank, since the last full build)
    bool nb4_incr = false;         // the next build_plan may update nb4 from the regrid's created / deleted slots
    std::vector<int32_t> nb4_created, nb4_deleted;
    // the leaf launch order kept per level as (Morton key of (i, j), slot), sorted -- the depth-first order from the
    // roots in Morton order (one rank) -- and updated at a regrid from the leaves it removed / added (O(leaves) merge
    // instead of a tree walk)
    std::vector<std::vector<std::pair<uint64_t, int32_t>>> lo_lvl;
    bool lo_full = false;
    std::vector<std::pair<int32_t, std::pair<uint64_t, int32_t>>> lo_rm, lo_add;   // (level, (key, slot))
    std::vector<uint8_t> lo_mark;
    bool canon_valid = false;      // canon / canon_pos match the tree (ensure_canon)
    double last_dt = 0.0;

    // flags of the last evaluation, per id
    std::vector<uint8_t> fl_ref, fl_crs, fl_amb;
    std::vector<double> fl_eta;
    std::vector<double> fl_eta_raw;    // per-leaf indicator gathered from the device (scratch)
    std::vector<uint8_t> fl_amb_raw;
    // regrid scratch kept across regrids (capacity-sized, reset entry by entry: no per-regrid allocation / fill)
    std::vector<uint8_t> rq_ref, rq_crs, rq_new;
    std::vector<int32_t> rq_set, rq_new_ids;
    std::vector<std::pair<uint64_t, int32_t>> rq_order;   // requested slots by canonical position (apply_regrid)

    // stats / timing
    amr_stats st{};
    bool timing = false;
    std::vector<cudaEvent_t> ev_free, ev_pending;   // pairs (start, stop)
    std::vector<int64_t> ev_cells;
    std::vector<double> ev_bytes;

    // CUDA graphs of one step (use_graphs, single rank): one per position of U^n in the buffer rotation,
    // re-captured when the plan changes
    uint64_t plan_version = 0;
    int64_t plan_steps = 0;     // steps taken with the current plan
    bool capturing = false;
    bool trace_on = getenv("AMR_TRACE") != nullptr;   // launch timeline (performance work only)
    std::vector<cudaEvent_t> trace_ev;
    std::vector<std::string> trace_name;
    cudaGraphExec_t gexec[3] = {nullptr, nullptr, nullptr};
    uint64_t gver[3] = {0, 0, 0};
    int64_t glaunches[3] = {0, 0, 0};
    double* d_dtp = nullptr;   // (dt_fixed, cfl) of a replayed step

    // subcycling (NEXT #4): per-level launch lists of every active patch (leaves, then covered patches with
    // LeafDesc.pad bit 0) with their own proxies, per-level C/F register tasks, accumulated registers
    std::vector<LeafDesc> sub_descs;
    std::vector<ProxyTask> sub_ptasks;
    std::vector<AccTask> acc_tasks;
    std::vector<int32_t> sub_off, sub_poff, acc_off, rt_off;   // per level [L+1]
    int sub_levels = 0;                                        // levels present in the (replicated) tree
    DevArray<LeafDesc> d_sub_descs;
    DevArray<ProxyTask> d_sub_ptasks;
    DevArray<AccTask> d_acc_tasks;
    DevArray<double> sub_proxy, facc;

    Comm comm;
    std::string err;
    amr_status sticky = AMR_OK;
};

