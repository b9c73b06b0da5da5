// debug_plan.cpp -- host-only planning API (include/amr_debug.h) for CPU tests of the multi-rank
// logic.  Uses the same PatchTree, partition and exchange planning as the device path; never calls CUDA.
#include "../../include/amr_debug.h"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "plan.h"
#include "tree.h"

struct amr_plan {
    amr::PatchTree tree;
    int levels = 1;
    int n = 8;
};

namespace {
std::vector<int32_t> canon_pos_of(const amr::PatchTree& t, std::vector<int32_t>& canon) {
    canon = t.canonical();
    std::vector<int32_t> pos(t.capacity, -1);
    for (size_t e = 0; e < canon.size(); ++e) pos[canon[e]] = (int32_t)e;
    return pos;
}
}  // namespace

extern "C" {

amr_status amr_plan_create(const amr_config* cfg, amr_plan** out) {
    if (!cfg || !out) return AMR_E_ARG;
    const amr_config& c = *cfg;
    int n = c.patch_cells;
    if (!(n == 8 || n == 16 || n == 32 || n == 64) || c.base_cells[0] % n || c.base_cells[1] % n || c.ratio != 2 ||
        c.num_levels < 1 || c.max_patches < 1)
        return AMR_E_CONFIG;
    int npx = c.base_cells[0] / n, npy = c.base_cells[1] / n;
    if ((int64_t)npx * npy > c.max_patches) return AMR_E_CAPACITY;
    amr_plan* p = new amr_plan();
    p->levels = c.num_levels;
    p->n = n;
    p->tree.init(npx, npy, c.num_levels, c.bc[0] == AMR_BC_PERIODIC, c.bc[2] == AMR_BC_PERIODIC, c.max_patches,
                 c.coarsen_rule);
    *out = p;
    return AMR_OK;
}

void amr_plan_destroy(amr_plan* p) { delete p; }

amr_status amr_plan_regrid(amr_plan* p, int32_t n, const int32_t* tree_index, const uint8_t* bits) {
    if (!p || n < 0 || (n && (!tree_index || !bits))) return AMR_E_ARG;
    std::vector<int32_t> canon;
    canon_pos_of(p->tree, canon);
    std::vector<uint8_t> ref(p->tree.capacity, 0), crs(p->tree.capacity, 0);
    for (int k = 0; k < n; ++k) {
        if (tree_index[k] < 0 || tree_index[k] >= (int)canon.size()) return AMR_E_ARG;
        ref[canon[tree_index[k]]] = bits[k] & 1;
        crs[canon[tree_index[k]]] = (bits[k] >> 1) & 1;
    }
    amr::PatchTree nt = p->tree;
    nt.begin_txn();   // the incremental check of the device path runs beside the full one
    std::string m;
    for (int id : canon) {
        if (!ref[id] || !nt.is_leaf(id) || nt.lev[id] >= p->levels - 1) continue;
        if (!nt.refine(id, m)) return m.find("capacity") != std::string::npos ? AMR_E_CAPACITY : AMR_E_MESH;
    }
    for (int l = p->levels - 2; l >= 0; --l)
        for (int id : canon)
            if (nt.lev[id] == l && crs[id] && nt.alive[id] && nt.coarsen_allowed(id)) nt.delete_children(id);
    std::string m2;
    const bool full = nt.validate(m), inc = nt.validate_txn(m2);
    if (full != inc) return AMR_E_STATE;   // validate_txn disagrees with validate: a bug, surfaced to the tests
    if (!full) return AMR_E_MESH;
    nt.commit();
    p->tree = nt;
    // the O(active) orders and neighbour table of build_plan against their definitions (sorts, neighbour())
    const amr::PatchTree& t = p->tree;
    const std::vector<int32_t> ca = t.canonical(), cs = t.canonical_sorted();
    if (ca != cs) return AMR_E_STATE;
    std::vector<std::vector<int32_t>> per;
    t.leaves_morton(per, [](int) { return true; });
    std::vector<std::pair<uint64_t, int32_t>> kv;
    for (int id : ca)
        if (t.is_leaf(id)) kv.push_back({(uint64_t(t.lev[id]) << t.morton_shift()) | amr::morton(t.pi[id], t.pj[id]), id});
    amr::radix_sort_pairs(kv);
    size_t e = 0;
    for (const auto& lv : per)
        for (int id : lv)
            if (e >= kv.size() || kv[e++].second != id) return AMR_E_STATE;
    if (e != kv.size()) return AMR_E_STATE;
    std::vector<int32_t> nb4;
    t.face_neighbours(ca, nb4);
    static const int d[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};
    for (int id : ca)
        for (int s2 = 0; s2 < 4; ++s2)
            if (nb4[4 * (size_t)id + s2] != t.neighbour(id, d[s2][0], d[s2][1])) return AMR_E_STATE;
    return AMR_OK;
}

amr_status amr_plan_tree(amr_plan* p, int32_t world, amr_patch_desc* out, int32_t cap, int32_t* count) {
    if (!p || !count || world < 1) return AMR_E_ARG;
    std::vector<int32_t> canon;
    std::vector<int32_t> pos = canon_pos_of(p->tree, canon);
    *count = (int32_t)canon.size();
    if (!out || cap < *count) return AMR_E_ARG;
    amr::Owners owner = amr::partition_owners(p->tree, world);
    static const int moore[8][2] = {{0, 1}, {1, 0}, {0, -1}, {-1, 0}, {1, 1}, {1, -1}, {-1, -1}, {-1, 1}};
    const amr::PatchTree& t = p->tree;
    for (size_t e = 0; e < canon.size(); ++e) {
        int id = canon[e];
        amr_patch_desc& d = out[e];
        d.level = t.lev[id];
        d.i = t.pi[id];
        d.j = t.pj[id];
        d.parent = t.parent[id] >= 0 ? pos[t.parent[id]] : -1;
        for (int q = 0; q < 4; ++q) d.child[q] = t.child[4 * id + q] >= 0 ? pos[t.child[4 * id + q]] : -1;
        for (int q = 0; q < 8; ++q) {
            int nb = t.neighbour(id, moore[q][0], moore[q][1]);
            d.nbr[q] = nb >= 0 ? pos[nb] : -1;
        }
        d.owner = owner[id];
        d.leaf = t.is_leaf(id);
        d.refine_req = d.coarsen_req = d.ambiguous = 0;
    }
    return AMR_OK;
}

amr_status amr_plan_exchange(amr_plan* p, int32_t world, int32_t rank, int32_t kind, int32_t* send_counts,
                             int32_t* send_index, int32_t* recv_counts, int32_t* recv_index, int32_t cap) {
    if (!p || world < 1 || rank < 0 || rank >= world || !send_counts || !recv_counts || !send_index || !recv_index)
        return AMR_E_ARG;
    std::vector<int32_t> canon;
    std::vector<int32_t> pos = canon_pos_of(p->tree, canon);
    amr::Owners owner = amr::partition_owners(p->tree, world);
    const bool raw = kind >= 1000;   // raw band items (tree index * 32 + code) instead of the slots they touch
    if (raw) kind -= 1000;
    amr::ExchangeLists L;
    if (kind == 0) L = amr::plan_halo(p->tree, owner, world, rank, p->n);
    else if (kind == 1) L = amr::plan_flux(p->tree, owner, world, rank);
    else {
        const int l = (kind - 2) / 3, which = (kind - 2) % 3;
        if (kind < 2 || l >= p->levels) return AMR_E_ARG;
        amr::SubLists S = amr::plan_subcycle(p->tree, owner, world, rank, p->n);
        L = which == 0 ? S.face[l] : (which == 1 ? S.coarse[l] : S.facc[l]);
    }
    // entries: slots (tree indices), or for band-item lists the distinct slots they touch (raw: the items)
    auto listed = [&](const std::vector<int32_t>& v) {
        std::vector<int32_t> o;
        for (int x : v) {
            if (!L.items) o.push_back(pos[x]);
            else if (raw) o.push_back(pos[x >> 5] * 32 + (x & 31));
            else if (o.empty() || o.back() != pos[x >> 5]) o.push_back(pos[x >> 5]);
        }
        if (L.items && !raw) {
            std::sort(o.begin(), o.end());
            o.erase(std::unique(o.begin(), o.end()), o.end());
        }
        return o;
    };
    int ns = 0, nr = 0;
    for (int q = 0; q < world; ++q) {
        std::vector<int32_t> sv = listed(L.send[q]), rv = listed(L.recv[q]);
        send_counts[q] = (int32_t)sv.size();
        recv_counts[q] = (int32_t)rv.size();
        for (int x : sv) {
            if (ns >= cap) return AMR_E_ARG;
            send_index[ns++] = x;
        }
        for (int x : rv) {
            if (nr >= cap) return AMR_E_ARG;
            recv_index[nr++] = x;
        }
    }
    return AMR_OK;
}

// Host plan work of one rank at a regrid (the replicated part of build_plan + Comm::replan), timed on this CPU:
// ms[0] partition, [1] this rank's roots and boundary roots, [2] leaf launch order, [3] face-neighbour table, [4] halo lists, [5] flux
// lists, [6] total; counts[0] active patches, [1] this rank's leaves, [2] halo items received, [3] sent.
amr_status amr_plan_profile(amr_plan* p, int32_t world, int32_t rank, int32_t reps, double* ms, int64_t* counts) {
    if (!p || world < 1 || rank < 0 || rank >= world || reps < 1 || !ms || !counts) return AMR_E_ARG;
    using clk = std::chrono::steady_clock;
    const amr::PatchTree& t = p->tree;
    for (int k = 0; k < 7; ++k) ms[k] = 0.0;
    for (int r = 0; r < reps; ++r) {
        auto t0 = clk::now();
        amr::Owners owner = amr::partition_owners(t, world);
        auto t1 = clk::now();
        // (as build_plan: the canonical order is not needed on the regrid path; this rank's roots and their boundary)
        const std::vector<int32_t> mine = owner.roots_of(rank);
        std::vector<int32_t> nbr = mine;
        for (int r2 : owner.boundary_roots(rank))
            if (owner.root_rank[(size_t)r2] != rank) nbr.push_back(r2);
        auto t2 = clk::now();
        std::vector<std::vector<int32_t>> per;
        t.leaves_morton_roots(per, [](int) { return true; }, [&](int root) { return owner[root] == rank; });
        auto t3 = clk::now();
        static std::vector<int32_t> nb4;   // (sized once, as the library's)
        t.face_neighbours_roots(nbr, nb4);
        auto t4 = clk::now();
        amr::ExchangeLists h = amr::plan_halo(t, owner, world, rank, p->n);
        auto t5 = clk::now();
        amr::ExchangeLists f = amr::plan_flux(t, owner, world, rank);
        auto t6 = clk::now();
        auto d = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        ms[0] += d(t0, t1); ms[1] += d(t1, t2); ms[2] += d(t2, t3); ms[3] += d(t3, t4); ms[4] += d(t4, t5);
        ms[5] += d(t5, t6); ms[6] += d(t0, t6);
        int64_t nl = 0;
        for (auto& v : per) nl += (int64_t)v.size();
        counts[0] = (int64_t)t.n_alive;
        counts[1] = nl;
        counts[2] = (int64_t)h.nrecv();
        counts[3] = (int64_t)h.nsend();
        (void)f;
    }
    for (int k = 0; k < 7; ++k) ms[k] /= reps;
    return AMR_OK;
}


// The plan phases of build_plan (leaf order, face-neighbour table, leaf descriptors: plan.h) of `rank` under a
// `world` partition, serially and on the armed host pool, reps times each; ms[0..2] serial, ms[3..5] pooled
// (milliseconds per run), *equal = 1 iff both give the same leaf order, nb4 entries of the planned patches and
// descriptor / proxy / reflux arrays byte for byte.  counts[0..2]: leaves, proxy tasks, reflux tasks; counts[3]:
// threads of the pool.
amr_status amr_plan_build_check(amr_plan* p, int32_t world, int32_t rank, int32_t halo_mode, int32_t reps, double* ms,
                                int64_t* counts, int32_t* equal) {
    if (!p || world < 1 || rank < 0 || rank >= world || reps < 1 || !ms || !counts || !equal) return AMR_E_ARG;
    using clk = std::chrono::steady_clock;
    const amr::PatchTree& t = p->tree;
    amr::Owners owner = amr::partition_owners(t, world);
    std::vector<int32_t> nb_roots = owner.roots_of(rank);
    for (int r2 : owner.boundary_roots(rank))
        if (owner.root_rank[(size_t)r2] != rank) nb_roots.push_back(r2);
    struct Out {
        std::vector<int32_t> ids, nb4;
        amr::DescOut d;
        std::string err;
        bool ok = true;
    } o[2];
    amr::HostPool& pool = amr::HostPool::get();
    auto d = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    for (int v = 0; v < 2; ++v) {
        pool.set_serial(v == 0);
        amr::PoolArm arm;
        double a0 = 0, a1 = 0, a2 = 0;
        for (int r = 0; r < reps; ++r) {
            auto t0 = clk::now();
            amr::plan_leaf_order(t, [&](int root) { return owner[root] == rank; }, o[v].ids);
            auto t1 = clk::now();
            amr::plan_face_neighbours(t, nb_roots, o[v].nb4);
            auto t2 = clk::now();
            o[v].ok = amr::plan_descriptors(t, o[v].nb4, o[v].ids, owner, world, rank, halo_mode, o[v].d, o[v].err);
            auto t3 = clk::now();
            a0 += d(t0, t1); a1 += d(t1, t2); a2 += d(t2, t3);
        }
        ms[3 * v] = a0 / reps; ms[3 * v + 1] = a1 / reps; ms[3 * v + 2] = a2 / reps;
    }
    pool.set_serial(false);
    auto same = [](const auto& a, const auto& b) {
        return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(a[0])) == 0);
    };
    bool eq = o[0].ok == o[1].ok && o[0].err == o[1].err && same(o[0].ids, o[1].ids) && same(o[0].d.leaves, o[1].d.leaves) &&
              same(o[0].d.ptasks, o[1].d.ptasks) && same(o[0].d.rtasks, o[1].d.rtasks);
    for (int id : o[0].ids)   // the planned leaves' neighbour entries (the rest of the table is scratch)
        for (int s2 = 0; s2 < 4; ++s2) eq = eq && o[0].nb4[(size_t)4 * id + s2] == o[1].nb4[(size_t)4 * id + s2];
    *equal = eq ? 1 : 0;
    counts[0] = (int64_t)o[1].ids.size();
    counts[1] = (int64_t)o[1].d.ptasks.size();
    counts[2] = (int64_t)o[1].d.rtasks.size();
    counts[3] = pool.threads();
    return o[0].ok ? AMR_OK : AMR_E_MESH;
}

}  // extern "C"
