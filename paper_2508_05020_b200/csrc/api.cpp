#include <chrono>
// api.cpp -- the C ABI of include/amr.h: context, host plan (descriptor build from
// the patch tree), step driver, regrid, state I/O, diagnostics and statistics.
// Every step of the numerical path runs in the kernels of kernels.cu; the host
// only orders launches and builds the descriptor lists (PAPER.md s3, Fig. 2).
#include "../../include/amr.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ctx.h"
#include "plan.h"

using namespace amr;

namespace {

amr_status fail(amr_ctx* c, amr_status s, const std::string& m) {
    if (c) {
        c->err = m;
        if (s == AMR_E_CUDA || s == AMR_E_COMM) c->sticky = s;
    }
    return s;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return fail(c, AMR_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

amr_status check(amr_ctx* c) {
    if (!c) return AMR_E_ARG;
    if (c->sticky != AMR_OK) {
        c->err = "context unusable after an earlier CUDA/NCCL error";
        return AMR_E_STATE;
    }
    return AMR_OK;
}

amr_status validate_config(const amr_config* cfg, std::string& m) {
    const amr_config& c = *cfg;
    int n = c.patch_cells;
    if (!(n == 8 || n == 16 || n == 32 || n == 64)) { m = "patch_cells must be 8, 16, 32 or 64"; return AMR_E_CONFIG; }
    if (c.base_cells[0] <= 0 || c.base_cells[1] <= 0 || c.base_cells[0] % n || c.base_cells[1] % n) {
        m = "base_cells must be positive multiples of patch_cells"; return AMR_E_CONFIG;
    }
    if (c.ratio != 2) { m = "refinement ratio must be 2 (quadtree)"; return AMR_E_CONFIG; }
    if (c.num_levels < 1 || c.num_levels > kMaxLevels - 1) { m = "num_levels out of range"; return AMR_E_CONFIG; }
    if ((int64_t)c.base_cells[0] << (c.num_levels - 1) >= (int64_t(1) << 30) ||
        (int64_t)c.base_cells[1] << (c.num_levels - 1) >= (int64_t(1) << 30)) { m = "mesh too large"; return AMR_E_CONFIG; }
    if (!(c.gamma > 1.0)) { m = "gamma must exceed 1"; return AMR_E_CONFIG; }
    for (int s = 0; s < 4; ++s)
        if (c.bc[s] < 0 || c.bc[s] > 2) { m = "bad boundary condition"; return AMR_E_CONFIG; }
    for (int ax = 0; ax < 2; ++ax)
        if ((c.bc[2 * ax] == AMR_BC_PERIODIC) != (c.bc[2 * ax + 1] == AMR_BC_PERIODIC)) {
            m = "periodic boundary must be set on both sides of an axis"; return AMR_E_CONFIG;
        }
    if (c.scheme != AMR_CENTRAL4 && c.scheme != AMR_WENO5_RUSANOV) { m = "bad scheme"; return AMR_E_CONFIG; }
    if (c.div_order != 2 && c.div_order != 4) { m = "div_order must be 2 or 4"; return AMR_E_CONFIG; }
    if (!(c.hi[0] > c.lo[0]) || !(c.hi[1] > c.lo[1])) { m = "empty domain"; return AMR_E_CONFIG; }
    if (c.dim != 1 && c.dim != 2) { m = "dim must be 1 or 2"; return AMR_E_CONFIG; }
    if (c.dim == 1 && (c.base_cells[1] != n || c.bc[2] != AMR_BC_PERIODIC)) {
        m = "dim 1 needs one periodic row of patches (strip embedding)"; return AMR_E_CONFIG;
    }
    if (c.world_size < 1 || c.rank < 0 || c.rank >= c.world_size) { m = "bad world_size / rank"; return AMR_E_CONFIG; }
    if (c.comm_backend < 0 || c.comm_backend > 2) { m = "comm_backend must be 0, 1 or 2"; return AMR_E_CONFIG; }
    if (c.world_size > 1 && c.comm_backend != 2 && !c.nccl_unique_id) {
        m = "world_size > 1 needs nccl_unique_id";
        return AMR_E_CONFIG;
    }
    if (c.world_size > 1 && c.comm_backend == 2 && !c.host_comm) { m = "comm_backend 2 needs host_comm"; return AMR_E_CONFIG; }
    if (c.refine_threshold < 0 || c.coarsen_fraction < 0) { m = "bad thresholds"; return AMR_E_CONFIG; }
    if (c.max_patches < 1) { m = "max_patches must be positive"; return AMR_E_CONFIG; }
    if (c.stage_kernel < 0 || c.stage_kernel > 3) { m = "stage_kernel must be 0..3"; return AMR_E_CONFIG; }
    if (c.halo_mode < 0 || c.halo_mode > 2) { m = "halo_mode must be 0, 1 or 2"; return AMR_E_CONFIG; }
    if (c.peer_map < 0 || c.peer_map > 1) { m = "peer_map must be 0 or 1"; return AMR_E_CONFIG; }
    if (c.peer_map == 1 && c.pool) { m = "peer_map 1 allocates the pool with ncclMemAlloc: cfg.pool must be NULL"; return AMR_E_CONFIG; }
    // halo_mode 2: the stage kernels that load remote face strips themselves -- the Central4 TMA kernel (n >= 32,
    // stage_kernel 0), the Central4 per-tile kernel (stage_kernel 1, every n; the n = 8 / 16 block-tile kernels of
    // stage_kernel 0 take their block-edge strips by TMA from the local pool only) and the WENO5 kernels (per-tile and
    // n = 8 block tiles); <= 8 ranks (3-bit owner field of LeafDesc.pad)
    if (c.halo_mode == 2 && c.world_size > 1 &&
        (c.world_size > 8 || c.stage_kernel > 1 ||
         (c.scheme == AMR_CENTRAL4 && c.patch_cells < 32 && c.stage_kernel != 1))) {
        m = "halo_mode 2 needs stage_kernel 0 / 1 (Central4 with patch_cells < 32: stage_kernel 1, the per-tile "
            "kernel), and <= 8 ranks";
        return AMR_E_CONFIG;
    }
    return AMR_OK;
}

// ------------------------------------------------------------------ plan
// host-side regrid phase timing (AMR_REGRID_PROF=1 in the environment; stderr)
struct PhaseClock {
    bool on = getenv("AMR_REGRID_PROF") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  [regrid] %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

// Subcycling plan (NEXT #4): for each level, the descriptors of every active patch of the level -- its leaves
// (launch order) and then its covered patches (pad bit 0; all same-level neighbours exist by R2) -- with proxies
// of their own (C/F ghosts prolonged in time per stage, physical BC), the C/F register tasks of the level's
// leaves, and per-level offsets of the reflux tasks (rtasks are in level-major leaf order).
void ensure_canon(amr_ctx* c);

amr_status build_subcycle_plan(amr_ctx* c) {
    const PatchTree& t = c->tree;
    const int L = c->cfg.num_levels;
    c->sub_descs.clear();
    c->sub_ptasks.clear();
    c->acc_tasks.clear();
    c->sub_off.assign(L + 1, 0);
    c->sub_poff.assign(L + 1, 0);
    c->acc_off.assign(L + 1, 0);
    c->rt_off.assign(L + 1, 0);
    int cpar = -1, cnb[9];   // the last C/F parent's 3 x 3 neighbourhood
    auto add = [&](int id, bool covered) -> amr_status {
        LeafDesc d{};
        d.slot = id;
        d.level = t.lev[id];
        d.pad = covered ? 1 : 0;
        for (int s = 0; s < 4; ++s) {
            int nb = c->nb4[(size_t)4 * id + s];
            if (nb >= 0) {
                d.side[s] = nb;
                if (!covered && t.has_children(nb)) d.cf |= 1 << s;
            } else {
                ProxyTask p{};
                p.proxy = (int)c->sub_ptasks.size();
                p.slot = id;
                p.side = s;
                p.level = t.lev[id];
                p.P = t.pi[id];
                p.Q = t.pj[id];
                if (nb == -2) {
                    p.kind = 0;
                    for (int q = 0; q < 9; ++q) p.coarse[q] = -1;
                } else {
                    if (covered) return fail(c, AMR_E_MESH, "subcycle: covered patch without a same-level neighbour");
                    p.kind = 1;
                    d.cf |= 1 << (4 + s);
                    int par = t.parent[id];
                    if (par != cpar) {   // siblings are consecutive (Morton leaf order): one lookup per parent
                        cpar = par;
                        for (int dy = -1; dy <= 1; ++dy)
                            for (int dx = -1; dx <= 1; ++dx) {
                                int q = (dx == 0 && dy == 0) ? par : t.neighbour(par, dx, dy);
                                if (q == -1) return fail(c, AMR_E_MESH, "R2 violated: coarse neighbourhood incomplete");
                                cnb[(dy + 1) * 3 + (dx + 1)] = q < 0 ? -1 : q;
                            }
                    }
                    for (int q = 0; q < 9; ++q) p.coarse[q] = cnb[q];
                }
                d.side[s] = -1 - p.proxy;
                c->sub_ptasks.push_back(p);
            }
        }
        if (!covered)
            for (int s = 0; s < 4; ++s) {
                if (d.cf & (1 << s)) c->acc_tasks.push_back(AccTask{id, s, 1});
                if (d.cf & (1 << (4 + s))) c->acc_tasks.push_back(AccTask{id, s, 2});
            }
        c->sub_descs.push_back(d);
        return AMR_OK;
    };
    size_t e = 0, r = 0, cp = 0;
    ensure_canon(c);
    for (int l = 0; l < L; ++l) {
        c->sub_off[l] = (int32_t)c->sub_descs.size();
        c->sub_poff[l] = (int32_t)c->sub_ptasks.size();
        c->acc_off[l] = (int32_t)c->acc_tasks.size();
        c->rt_off[l] = (int32_t)r;
        for (; e < c->leaf_ids.size() && t.lev[c->leaf_ids[e]] == l; ++e) {
            amr_status s = add(c->leaf_ids[e], false);
            if (s != AMR_OK) return s;
        }
        for (; cp < c->canon.size() && t.lev[c->canon[cp]] == l; ++cp) {   // canon is level-major: level l's run
            const int id = c->canon[cp];
            if (t.has_children(id) && c->comm.owns(c, id)) {
                amr_status s = add(id, true);
                if (s != AMR_OK) return s;
            }
        }
        while (r < c->rtasks.size() && c->rtasks[r].level == l) ++r;
    }
    // the one-pass walk above relies on canon being level-major (canon_key): every covered patch must have been seen
    if (cp != c->canon.size() || e != c->leaf_ids.size())
        return fail(c, AMR_E_STATE, "subcycle plan: canonical / leaf order not level-major");
    c->sub_levels = 0;
    for (int id : c->canon) c->sub_levels = std::max(c->sub_levels, t.lev[id] + 1);
    c->sub_off[L] = (int32_t)c->sub_descs.size();
    c->sub_poff[L] = (int32_t)c->sub_ptasks.size();
    c->acc_off[L] = (int32_t)c->acc_tasks.size();
    c->rt_off[L] = (int32_t)r;
    return AMR_OK;
}

// The canonical (level, j, i) order and its inverse, computed on first use after a plan change: the ABI's tree indices
// need them, the step / regrid path does not (O(active patches) on every rank otherwise)
void ensure_canon(amr_ctx* c) {
    if (c->canon_valid) return;
    const PatchTree& t = c->tree;
    if ((int)c->canon_pos.size() != t.capacity) c->canon_pos.assign(t.capacity, -1);
    else for (int id : c->canon) c->canon_pos[id] = -1;
    c->canon = t.canonical();
    for (size_t e = 0; e < c->canon.size(); ++e) c->canon_pos[c->canon[e]] = (int)e;
    c->canon_valid = true;
}

// peer_map 1: the state pool and the flux registers are NCCL symmetric-window memory, mapped by window registration
bool nccl_windows(const amr_ctx* c) {
    return c->cfg.peer_map == 1 && c->cfg.world_size > 1 && c->cfg.comm_backend == 0 && c->cfg.halo_mode >= 1;
}

// AMR_CHECK_PLAN=1 (tests; compute-sanitizer is closed on this GPU pool): every index a kernel dereferences through
// the plan's descriptors is checked against the tree and the buffer extents before the upload -- leaf slots alive
// leaves below the slot capacity, same-level side sources alive patches of the leaf's level at the face position,
// proxy numbers inside the proxy list, C/F parents' 3 x 3 sources alive level-(l-1) patches or -1, reflux fine
// slots alive level-(l+1) leaves, restriction parents / children alive with the parent-child links, sibling groups'
// leaf positions inside the leaf list and the children of their parent.  The kernels' addressing inside a patch is
// fixed by n and the tile shape; with these checks every global address they form is inside the pools.
bool plan_checks_on() {
    static const bool on = getenv("AMR_CHECK_PLAN") != nullptr;
    return on;
}
amr_status validate_plan(amr_ctx* c) {
    const PatchTree& t = c->tree;
    const int cap = t.capacity, L = c->cfg.num_levels;
    auto live = [&](int id) { return id >= 0 && id < cap && t.alive[id]; };
    auto bad = [&](const std::string& m) { return fail(c, AMR_E_STATE, "plan check: " + m); };
    static const int dx[4] = {-1, 1, 0, 0}, dy[4] = {0, 0, -1, 1};
    const int np = (int)c->ptasks.size();
    auto check_leaf = [&](const LeafDesc& d, bool covered_ok) -> bool {
        if (!live(d.slot) || d.level != t.lev[d.slot]) return false;
        if (!covered_ok && !t.is_leaf(d.slot)) return false;
        for (int s = 0; s < 4; ++s) {
            const int v = d.side[s];
            if (v >= 0) {
                if (!live(v) || t.lev[v] != d.level) return false;
                int i = t.pi[d.slot] + dx[s], j = t.pj[d.slot] + dy[s];
                if (!t.wrap(d.level, i, j) || t.pi[v] != i || t.pj[v] != j) return false;
            } else if (-1 - v >= np) {
                return false;
            }
        }
        return true;
    };
    for (const LeafDesc& d : c->leaves)
        if (!check_leaf(d, false)) return bad("leaf descriptor of slot " + std::to_string(d.slot));
    for (const LeafDesc& d : c->gleaves)
        if (!check_leaf(d, false)) return bad("block-tile member of slot " + std::to_string(d.slot));
    for (const LeafDesc& d : c->singles)
        if (!check_leaf(d, false)) return bad("single leaf of slot " + std::to_string(d.slot));
    for (int k = 0; k < np; ++k) {
        const ProxyTask& p = c->ptasks[k];
        if (p.proxy != k || !live(p.slot) || p.side < 0 || p.side > 3 || p.level != t.lev[p.slot])
            return bad("proxy task " + std::to_string(k));
        for (int q = 0; q < 9; ++q) {
            const int v = p.coarse[q];
            if (p.kind == 0 ? v != -1 : !(v == -1 || (live(v) && t.lev[v] == p.level - 1)))
                return bad("coarse source of proxy " + std::to_string(k));
        }
        if (p.kind == 1 && p.coarse[4] != t.parent[p.slot]) return bad("proxy parent " + std::to_string(k));
    }
    for (const RefluxTask& r : c->rtasks) {
        if (r.leaf < 0 || r.leaf >= (int)c->leaves.size() || c->leaves[r.leaf].slot != r.slot || !live(r.slot))
            return bad("reflux task of slot " + std::to_string(r.slot));
        for (int s = 0; s < 4; ++s)
            if (r.mask & (1 << s))
                for (int h = 0; h < 2; ++h)
                    if (!live(r.fine[s][h]) || !t.is_leaf(r.fine[s][h]) || t.lev[r.fine[s][h]] != r.level + 1)
                        return bad("reflux fine slot of " + std::to_string(r.slot));
    }
    for (int l = 1; l < L && l < (int)c->rlev.size(); ++l)
        for (const RestrictTask& r : c->rlev[l]) {
            if (!live(r.parent) || t.lev[r.parent] != l - 1) return bad("restriction parent");
            for (int q = 0; q < 4; ++q)
                if (!live(r.child[q]) || t.parent[r.child[q]] != r.parent || t.child[4 * r.parent + q] != r.child[q])
                    return bad("restriction child");
        }
    const int nl = (int)c->leaves.size();
    for (size_t g = 0; g + 4 < c->sib.size(); g += 5) {
        const int par = c->sib[g];
        if (!live(par)) return bad("sibling group parent");
        for (int q = 0; q < 4; ++q) {
            const int e = c->sib[g + 1 + q];
            if (e < 0 || e >= nl || c->leaves[e].slot != t.child[4 * par + q]) return bad("sibling group leaf position");
        }
    }
    if ((int64_t)c->proxy.cap < (int64_t)std::max(1, np) * (int64_t)c->PS) return bad("proxy buffer smaller than the proxy list");
    return AMR_OK;
}

amr_status build_plan(amr_ctx* c) {
    NvtxRange nv("build_plan");
    PhaseClock clk;
    PatchTree& t = c->tree;
    const int L = c->cfg.num_levels;
    // the plan phases run in parts on the host pool for large trees (its workers spin while armed; below ~8 k leaves
    // the parts' fixed cost and the spinning threads' competition for the cores cost more than they save: configs[2])
    std::unique_ptr<PoolArm> arm(t.n_leaves() >= kPoolMinLeaves ? new PoolArm() : nullptr);
    c->canon_valid = false;   // the canonical order is rebuilt on demand (ensure_canon)
    // id -> position maps sized once; the previous plan's entries are cleared instead of refilling all slots
    if ((int)c->leaf_pos.size() != t.capacity) c->leaf_pos.assign(t.capacity, -1);
    else for (int id : c->leaf_ids) c->leaf_pos[id] = -1;
    clk.mark("plan: reset maps");
    // this rank's roots (all of them on one rank) and the roots its patches read from across the partition
    // boundary: every loop below is over their subtrees, O(local)
    const std::vector<int32_t> my_roots = c->comm.owner.roots_of(c->comm.rank);
    std::vector<int32_t> nb_roots = my_roots;
    if (c->comm.world > 1) {
        for (int r : c->comm.owner.boundary_roots(c->comm.rank))
            if (c->comm.owner.root_rank[(size_t)r] != c->comm.rank) nb_roots.push_back(r);
    }

    // leaves in launch order: level, then Morton order of (i, j) for L2 locality of halos (a depth-first walk
    // from this rank's roots in Morton order, in parts over root ranges merged level by level -- plan.h; the planning
    // API checks it against the sort of (level, Morton) keys)
    static const bool check_incr = getenv("AMR_CHECK_INCR") != nullptr;   // (tests: incremental tables vs full ones)
    if (c->comm.world == 1 && c->nb4_incr && c->lo_full) {
        // one rank after a regrid: per level, drop the leaves it removed and merge in the ones it added (by key)
        if ((int)c->lo_mark.size() != t.capacity) c->lo_mark.assign(t.capacity, 0);
        for (const auto& r : c->lo_rm) c->lo_mark[r.second.second] = 1;
        std::sort(c->lo_add.begin(), c->lo_add.end());
        std::vector<std::pair<uint64_t, int32_t>> merged;
        size_t ia = 0;
        for (int l = 0; l < L; ++l) {
            auto& lst = c->lo_lvl[l];
            merged.clear();
            merged.reserve(lst.size() + 16);
            for (const auto& e : lst) {
                if (c->lo_mark[e.second]) continue;
                while (ia < c->lo_add.size() && c->lo_add[ia].first == l && c->lo_add[ia].second.first < e.first)
                    merged.push_back(c->lo_add[ia++].second);
                merged.push_back(e);
            }
            while (ia < c->lo_add.size() && c->lo_add[ia].first == l) merged.push_back(c->lo_add[ia++].second);
            lst.swap(merged);
        }
        for (const auto& r : c->lo_rm) c->lo_mark[r.second.second] = 0;
        c->leaf_ids.clear();
        for (int l = 0; l < L; ++l)
            for (const auto& e : c->lo_lvl[l]) c->leaf_ids.push_back(e.second);
        if (check_incr) {
            std::vector<int32_t> full;
            plan_leaf_order(t, [&](int root) { return c->comm.owns(c, root); }, full);
            if (full != c->leaf_ids) return fail(c, AMR_E_STATE, "incremental leaf order differs from the full walk");
        }
    } else {
        plan_leaf_order(t, [&](int root) { return c->comm.owns(c, root); }, c->leaf_ids);
        c->lo_full = c->comm.world == 1;
        if (c->lo_full) {
            c->lo_lvl.assign(L, {});
            for (int id : c->leaf_ids) c->lo_lvl[t.lev[id]].push_back({morton((uint32_t)t.pi[id], (uint32_t)t.pj[id]), id});
        }
    }
    for (size_t e = 0; e < c->leaf_ids.size(); ++e) c->leaf_pos[c->leaf_ids[e]] = (int)e;
    clk.mark("plan: leaf order");
    // owned parents whose 4 children are leaves: the coarsening candidates of a12; owned covered patches: the
    // restriction tasks per level (O9)
    c->sib.clear();
    c->rlev.assign(L, {});
    for (int r : my_roots)
        t.subtree(t.root_slot(r), [&](int id) {
            if (!t.has_children(id)) return;
            RestrictTask rt{};
            rt.parent = id;
            for (int q = 0; q < 4; ++q) rt.child[q] = t.child[4 * id + q];
            c->rlev[t.lev[id] + 1].push_back(rt);
            int q = 0;
            while (q < 4 && c->leaf_pos[t.child[4 * id + q]] >= 0) ++q;
            if (q < 4) return;
            c->sib.push_back(id);
            for (q = 0; q < 4; ++q) c->sib.push_back(c->leaf_pos[t.child[4 * id + q]]);
        });
    clk.mark("plan: sib + restriction");

    // face neighbours of the local patches and of those they read across the boundary, from the parents' entries
    // (subtree pre-order, no recursion): nb4[4 id + s]; after a regrid on one rank only the created / deleted slots
    // and their neighbours are updated (O(changes))
    if (c->comm.world == 1 && c->nb4_incr && c->nb4_full) {
        update_face_neighbours(t, c->nb4_created, c->nb4_deleted, c->nb4);
        if (check_incr) {
            std::vector<int32_t> full;
            plan_face_neighbours(t, nb_roots, full);
            for (int id : c->canon_valid ? c->canon : t.canonical())
                for (int s = 0; s < 4; ++s)
                    if (full[(size_t)4 * id + s] != c->nb4[(size_t)4 * id + s])
                        return fail(c, AMR_E_STATE, "incremental face-neighbour table differs from the full one");
        }
    } else {
        plan_face_neighbours(t, nb_roots, c->nb4);
        c->nb4_full = c->comm.world == 1;
    }
    c->nb4_incr = false;
    clk.mark("plan: face neighbours");
    {   // leaf descriptors, proxy strips (numbered in leaf order) and reflux tasks, in parts of the leaf order
        static thread_local DescOut dout;
        DescOut& D = dout;
        std::string m;
        if (!plan_descriptors(t, c->nb4, c->leaf_ids, c->comm.owner, c->comm.world, c->comm.rank, c->comm.halo_mode,
                              D, m))
            return fail(c, AMR_E_MESH, m);
        c->leaves.swap(D.leaves);
        c->ptasks.swap(D.ptasks);
        c->rtasks.swap(D.rtasks);
    }
    clk.mark("plan: leaf descriptors");
    c->leaf_cells = (int64_t)c->leaf_ids.size() * c->n * c->n;
    // Central4 with n = 8, 16: complete aligned B x B blocks of same-level leaves (consecutive in level-Morton
    // order, B = 32/n) form the 32 x 32 tiles of the TMA group kernel; the other leaves take the per-tile kernel
    c->gleaves.clear();
    c->singles.clear();
    const bool group_c4 = c->cfg.scheme == AMR_CENTRAL4 && (c->n == 8 || c->n == 16);
    const bool group_weno = c->cfg.scheme != AMR_CENTRAL4 && c->n == 8;   // n = 16 WENO: one CTA per patch (DESIGN s5)
    if (c->cfg.stage_kernel == 0 && (group_c4 || group_weno) && !c->cfg.subcycle) {
        const int B = 32 / c->n, K = B * B;
        for (size_t e = 0; e < c->leaves.size();) {
            const int id0 = c->leaf_ids[e];
            bool ok = t.pi[id0] % B == 0 && t.pj[id0] % B == 0 && e + K <= c->leaves.size();
            for (int m = 0; ok && m < K; ++m) {
                const int id = c->leaf_ids[e + m];
                const int mx = (m & 1) | ((m >> 1) & 2), my = ((m >> 1) & 1) | ((m >> 2) & 2);
                ok = t.lev[id] == t.lev[id0] && t.pi[id] == t.pi[id0] + mx && t.pj[id] == t.pj[id0] + my;
            }
            if (ok) {
                c->gleaves.insert(c->gleaves.end(), c->leaves.begin() + e, c->leaves.begin() + e + K);
                bool contig = true;   // members in consecutive slots: the block is one contiguous run of the pool
                for (int m = 1; m < K; ++m) contig = contig && c->leaf_ids[e + m] == id0 + m;
                if (contig) c->gleaves[c->gleaves.size() - K].pad |= 2;
                e += K;
            } else {
                c->singles.push_back(c->leaves[e]);
                e += 1;
            }
        }
    }
    if (c->cfg.subcycle) {
        amr_status ss = build_subcycle_plan(c);
        if (ss != AMR_OK) return ss;
    }
    clk.mark("plan: descriptors");

    cudaStream_t s = c->stream;
    {   // one packed upload of the per-plan descriptor arrays (each 256-byte aligned in the arena)
        size_t total = 0;   // the arena layout first (each array 256-byte aligned), then one pinned staging fill
        auto span = [&](size_t bytes) { total = ((total + 255) & ~(size_t)255) + bytes; };
        span(c->leaves.size() * sizeof(LeafDesc));
        span(c->gleaves.size() * sizeof(LeafDesc));
        span(c->singles.size() * sizeof(LeafDesc));
        span(c->ptasks.size() * sizeof(ProxyTask));
        span(c->rtasks.size() * sizeof(RefluxTask));
        for (int l = 0; l < L; ++l) span(c->rlev[l].size() * sizeof(RestrictTask));
        span(c->sib.size() * sizeof(int32_t));
        // the previous plan's DMA out of the pinned arena must be done before it is refilled (build_plan does not
        // wait for its own upload: the host goes on to the prolongation launches while it runs)
        if (c->arena_ev) CU(cudaEventSynchronize(c->arena_ev));
        if (total > c->arena_host_cap) {
            if (c->arena_host) cudaFreeHost(c->arena_host);
            c->arena_host = nullptr;
            c->arena_host_cap = 0;
            const size_t cap = std::max<size_t>(total + total / 2, 4096);
            CU(cudaMallocHost(reinterpret_cast<void**>(&c->arena_host), cap));
            c->arena_host_cap = cap;
        }
        size_t used = 0;
        std::vector<size_t> offs;
        auto add = [&](const void* src, size_t bytes) {
            const size_t o = (used + 255) & ~(size_t)255;
            if (bytes) std::memcpy(c->arena_host + o, src, bytes);
            used = o + bytes;
            offs.push_back(o);
        };
        add(c->leaves.data(), c->leaves.size() * sizeof(LeafDesc));
        add(c->gleaves.data(), c->gleaves.size() * sizeof(LeafDesc));
        add(c->singles.data(), c->singles.size() * sizeof(LeafDesc));
        add(c->ptasks.data(), c->ptasks.size() * sizeof(ProxyTask));
        add(c->rtasks.data(), c->rtasks.size() * sizeof(RefluxTask));
        for (int l = 0; l < L; ++l) add(c->rlev[l].data(), c->rlev[l].size() * sizeof(RestrictTask));
        add(c->sib.data(), c->sib.size() * sizeof(int32_t));
        // the views must not alias the arena while it is re-allocated
        c->d_leaves.release(); c->d_gleaves.release(); c->d_singles.release(); c->d_ptasks.release();
        c->d_rtasks.release(); c->d_sib.release();
        for (auto& d : c->d_rlev) d.release();
        CU(c->arena_dev.reserve(std::max<size_t>(used, 256)));
        if (used) CU(cudaMemcpyAsync(c->arena_dev.p, c->arena_host, used, cudaMemcpyHostToDevice, s));
        if (!c->arena_ev) CU(cudaEventCreateWithFlags(&c->arena_ev, cudaEventDisableTiming));
        CU(cudaEventRecord(c->arena_ev, s));
        char* base = c->arena_dev.p;
        size_t k = 0;
        c->d_leaves.view(reinterpret_cast<LeafDesc*>(base + offs[k++]), c->leaves.size());
        c->d_gleaves.view(reinterpret_cast<LeafDesc*>(base + offs[k++]), c->gleaves.size());
        c->d_singles.view(reinterpret_cast<LeafDesc*>(base + offs[k++]), c->singles.size());
        c->d_ptasks.view(reinterpret_cast<ProxyTask*>(base + offs[k++]), c->ptasks.size());
        c->d_rtasks.view(reinterpret_cast<RefluxTask*>(base + offs[k++]), c->rtasks.size());
        c->d_rlev.resize(L);
        for (int l = 0; l < L; ++l) c->d_rlev[l].view(reinterpret_cast<RestrictTask*>(base + offs[k++]), c->rlev[l].size());
        c->d_sib.view(reinterpret_cast<int32_t*>(base + offs[k++]), c->sib.size());
    }
    if (c->cfg.subcycle) {
        CU(c->d_sub_descs.upload(c->sub_descs, s));
        CU(c->d_sub_ptasks.upload(c->sub_ptasks, s));
        CU(c->d_acc_tasks.upload(c->acc_tasks, s));
        CU(c->sub_proxy.reserve(std::max<size_t>(1, c->sub_ptasks.size()) * c->PS));
        CU(c->facc.reserve((size_t)t.capacity * 16 * c->n, false));
    }

    CU(c->proxy.reserve(std::max<size_t>(1, c->ptasks.size()) * c->PS));
    if (nccl_windows(c) && !c->freg_nccl) {   // peer_map 1: the flux registers are NCCL window memory too (fixed size)
        const size_t cnt = (size_t)t.capacity * 16 * c->n;
        std::string e;
        c->freg_nccl = comm_nccl_mem_alloc(cnt * sizeof(double), e);
        if (!c->freg_nccl) return fail(c, AMR_E_COMM, "flux registers: " + e);
        c->freg.view(reinterpret_cast<double*>(c->freg_nccl), cnt);
        c->freg.cap = cnt;
    }
    CU(c->freg.reserve((size_t)t.capacity * 16 * c->n, false));   // indexed by slot (remote fine leaves arrive by exchange)
    CU(c->d_maxeta.reserve(std::max<size_t>(1, c->leaves.size())));
    CU(c->d_amb.reserve(std::max<size_t>(1, c->leaves.size())));
    CU(c->d_flist.reserve(2 * (c->leaves.size() + c->sib.size() / 5) + 2));
    CU(c->d_fcount.reserve(1));
    CU(c->d_partial.reserve(4 * std::max<size_t>(1, c->leaves.size())));
    // no stream synchronisation: the descriptors travel from the pinned arena (guarded by arena_ev) and the
    // subcycling lists' pageable copies are staged by the driver before cudaMemcpyAsync returns
    clk.mark("plan: uploads");

    c->st.leaves = t.n_leaves();
    c->st.patches = (int64_t)t.n_alive;
    c->st.leaf_cells = c->leaf_cells;
    c->st.proxies = (int64_t)c->ptasks.size();
    if (c->cfg.stage_kernel == 2)
        CU(c->unf_scratch.reserve(unfused_scratch_doubles(c->n, std::max<int>(1, (int)c->leaves.size()))));
    c->lambda_valid = false;
    c->ghost_valid = false;
    c->plan_version++;
    c->plan_steps = 0;
    c->comm.replan(t);
    if (plan_checks_on()) return validate_plan(c);
    return AMR_OK;
}

AuxArgs aux(amr_ctx* c, const double* Ur, double* Uw) {
    AuxArgs a{};
    a.U = Ur;
    a.Uc = Ur;
    a.Uw = Uw;
    a.proxy = c->proxy.p;
    a.freg = c->freg.p;
    a.dt = c->d_dt;
    a.gamma = c->cfg.gamma;
    a.theta = c->cfg.refine_threshold;
    a.coarsen_fraction = c->cfg.coarsen_fraction;
    a.lambda_bits = c->d_lambda;
    a.err = c->d_err;
    a.check = c->cfg.check_positivity;
    a.geo = c->geo;
    return a;
}

// Launch timeline for performance work (AMR_TRACE=<file>, not for capture): an event before and after every
// launch; written as "name start_us duration_us" lines (relative to the first event) at amr_destroy.
void trace_pre(amr_ctx* c) {
    if (!c->trace_on || c->capturing) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c->stream);
    c->trace_ev.push_back(e);
}
void trace_post(amr_ctx* c, const char* what) {
    if (!c->trace_on || c->capturing || c->trace_ev.size() % 2 == 0) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c->stream);
    c->trace_ev.push_back(e);
    c->trace_name.push_back(what);
}
void trace_dump(amr_ctx* c) {
    if (!c->trace_on || c->trace_ev.empty()) return;
    cudaStreamSynchronize(c->stream);
    FILE* f = std::fopen(getenv("AMR_TRACE"), "a");
    if (!f) return;
    for (size_t k = 0; k + 1 < c->trace_ev.size(); k += 2) {
        float t0 = 0.f, t1 = 0.f;
        cudaEventElapsedTime(&t0, c->trace_ev[0], c->trace_ev[k]);
        cudaEventElapsedTime(&t1, c->trace_ev[k], c->trace_ev[k + 1]);
        std::fprintf(f, "%s %.2f %.2f\n", c->trace_name[k / 2].c_str(), t0 * 1e3, t1 * 1e3);
    }
    std::fclose(f);
    for (auto e : c->trace_ev) cudaEventDestroy(e);
    c->trace_ev.clear();
    c->trace_name.clear();
}

amr_status count_launch(amr_ctx* c, cudaError_t e, const char* what) {
    trace_post(c, what);
    if (e != cudaSuccess) return fail(c, AMR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    c->st.launches++;
    return AMR_OK;
}

#define LAUNCH(expr, what)                                         \
    do {                                                           \
        trace_pre(c);                                              \
        amr_status s_ = count_launch(c, (expr), what);             \
        if (s_ != AMR_OK) return s_;                               \
    } while (0)

// restriction of every non-leaf patch, finest level first (O9)
amr_status restrict_all(amr_ctx* c, double* Ubuf) {
    AuxArgs a = aux(c, Ubuf, Ubuf);
    for (int l = c->cfg.num_levels - 1; l >= 1; --l)
        if (!c->rlev[l].empty()) LAUNCH(launch_restrict(c->d_rlev[l].p, (int)c->rlev[l].size(), a, c->stream), "restrict");
    return AMR_OK;
}

amr_status fill_ghosts(amr_ctx* c, const double* Ubuf) {
    if (c->ptasks.empty()) return AMR_OK;
    AuxArgs a = aux(c, Ubuf, nullptr);
    LAUNCH(launch_ghost(c->d_ptasks.p, (int)c->ptasks.size(), c->g, a, c->stream), "ghost");
    return AMR_OK;
}

amr_status seed_lambda(amr_ctx* c) {
    CU(cudaMemsetAsync(c->d_lambda, 0, sizeof(unsigned long long), c->stream));
    amr_status s = c->comm.exchange_halos(c, c->U[c->un]);
    if (s != AMR_OK) return s;
    AuxArgs a = aux(c, c->U[c->un], nullptr);
    a.lam0 = c->cfg.subcycle;
    LAUNCH(launch_lambda(c->d_leaves.p, (int)c->leaves.size(), a, c->stream), "lambda");
    s = c->comm.allreduce_max_u64(c, c->d_lambda);
    if (s != AMR_OK) return s;
    c->lambda_valid = true;
    return AMR_OK;
}

cudaEvent_t take_event(amr_ctx* c) {
    if (c->ev_free.empty()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    cudaEvent_t e = c->ev_free.back();
    c->ev_free.pop_back();
    return e;
}

amr_status harvest_events(amr_ctx* c) {
    if (c->ev_pending.empty()) return AMR_OK;
    CU(cudaStreamSynchronize(c->stream));
    for (size_t k = 0; k + 1 < c->ev_pending.size(); k += 2) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, c->ev_pending[k], c->ev_pending[k + 1]));
        c->st.stage_ms += ms;
        c->st.stage_timed++;
        c->st.stage_cells += c->ev_cells[k / 2];
        c->st.stage_bytes += c->ev_bytes[k / 2];
        c->ev_free.push_back(c->ev_pending[k]);
        c->ev_free.push_back(c->ev_pending[k + 1]);
    }
    c->ev_pending.clear();
    c->ev_cells.clear();
    c->ev_bytes.clear();
    return AMR_OK;
}

// The work after a stage kernel as one cooperative post-stage launch (one rank: no flux / halo exchange sits
// between reflux, restriction and the next ghost fill).  AMR_POST_FUSE=0 selects the separate launches (A/B).
bool post_fused(const amr_ctx* c) {
    static const bool on = [] { const char* e = getenv("AMR_POST_FUSE"); return !(e && e[0] == '0'); }();
    return on && c->comm.world == 1;
}

// one SSP-RK3 step, queued on the stream without host synchronisation
amr_status enqueue_step(amr_ctx* c, double dt, double cfl) {
    if (!c->lambda_valid && !(dt > 0.0)) {
        amr_status s = seed_lambda(c);
        if (s != AMR_OK) return s;
    }
    if (c->capturing) LAUNCH(launch_dt_dev(c->d_dt, c->d_lambda, c->d_err, c->d_dtp, c->stream), "dt");
    else LAUNCH(launch_dt(c->d_dt, c->d_lambda, c->d_err, dt, cfl, c->stream), "dt");
    const int A = (c->un + 1) % 3, B = (c->un + 2) % 3;
    const bool fused = post_fused(c);
    const double as[3] = {0.0, 0.75, 1.0 / 3.0};
    const double bs[3] = {1.0, 0.25, 2.0 / 3.0};
    static const char* const kStageName[3] = {"stage 1", "stage 2", "stage 3"};
    for (int s = 1; s <= 3; ++s) {
        NvtxRange nv(kStageName[s - 1]);
        double* Uin = s == 1 ? c->U[c->un] : (s == 2 ? c->U[A] : c->U[B]);
        double* Uout = s == 2 ? c->U[B] : c->U[A];
        amr_status cs = AMR_OK;
        // one rank: the previous stage's post kernel filled the ghost strips of this stage's input; stage 1 fills
        // them here unless the last step's stage 3 already did (and nothing has changed U^n or the plan since)
        if (!fused || (s == 1 && !(c->ghost_valid && !c->capturing))) {
            cs = c->comm.exchange_halos_stage(c, Uin);
            if (cs != AMR_OK) return cs;
            cs = fill_ghosts(c, Uin);
            if (cs != AMR_OK) return cs;
        }
        StageArgs a{};
        a.leaves = c->d_leaves.p;
        a.nleaves = (int)c->leaves.size();
        a.tiles = c->n > 32 ? c->n / 32 : 1;
        a.Uin = Uin;
        a.Un = c->U[c->un];
        a.Uout = Uout;
        a.proxy = c->proxy.p;
        a.freg = c->freg.p;
        a.dt = c->d_dt;
        a.a = as[s - 1];
        a.b = bs[s - 1];
        a.stage = s;
        a.div_order = c->cfg.div_order;
        a.characteristic = c->cfg.weno_characteristic;
        a.check = c->cfg.check_positivity;
        a.want_lambda = s == 3;
        a.gamma = c->cfg.gamma;
        a.eps = c->cfg.weno_eps;
        a.lambda_bits = c->d_lambda;
        a.err = c->d_err;
        a.nslots = c->cfg.max_patches;
        a.nproxy = (int32_t)(c->proxy.cap / c->PS);
        a.variant = c->cfg.stage_kernel;
        a.scratch = c->unf_scratch.p;   // variant 2: reserved by build_plan (no allocation inside a graph capture)
        if (!c->gleaves.empty()) {      // Central4 n = 8, 16: block tiles, then the remaining single leaves
            const int K = (32 / c->n) * (32 / c->n);
            a.gleaves = c->d_gleaves.p;
            a.ngroups = (int32_t)(c->gleaves.size() / K);
            a.leaves = c->d_singles.p;
            a.nleaves = (int32_t)c->singles.size();
        }
        a.geo = c->geo;
        if (c->comm.world > 1 && c->comm.halo_mode == 2) {   // remote face strips: TMA straight from the owners' pools
            a.npeers = c->comm.world;
            const size_t off = (size_t)(Uin - (double*)c->comm.pool_base);
            for (int q = 0; q < c->comm.world; ++q) a.peer_in[q] = c->comm.peer_pool[q] + off;
        }
        int scheme = c->cfg.scheme == AMR_CENTRAL4 ? 0 : (c->cfg.weno_characteristic ? 1 : 2);
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (c->timing && !c->leaves.empty()) {
            e0 = take_event(c);
            e1 = take_event(c);
            CU(cudaEventRecord(e0, c->stream));
        }
        LAUNCH(launch_stage(scheme, a, c->stream), "stage");
        c->st.launches += stage_launches_per_stage(a.variant, a.nleaves) - 1 + (a.gleaves && a.nleaves > 0 ? 1 : 0);
        c->st.stage_launches++;
        if (e1) {
            CU(cudaEventRecord(e1, c->stream));
            c->ev_pending.push_back(e0);
            c->ev_pending.push_back(e1);
            c->ev_cells.push_back(c->leaf_cells);
            c->ev_bytes.push_back((double)c->leaf_cells * (s == 1 ? 64.0 : 96.0));
        }
        if (fused) {   // reflux + restriction + the next stage's ghost strips in one cooperative launch
            PostArgs p{};
            p.a = aux(c, Uout, Uout);
            p.a.b = bs[s - 1];
            p.a.stage = s;
            p.a.want_lambda = s == 3;
            p.rtasks = c->d_rtasks.p;
            p.nr = (int32_t)c->rtasks.size();
            p.levels = c->cfg.num_levels;
            bool work = p.nr > 0;
            for (int l = 1; l < p.levels; ++l) {
                p.rl[l] = c->d_rlev[l].p;
                p.nrl[l] = (int32_t)c->rlev[l].size();
                work = work || p.nrl[l] > 0;
            }
            p.ptasks = c->d_ptasks.p;
            p.np = (s < 3 || !c->capturing) ? (int32_t)c->ptasks.size() : 0;   // a graph refills at its stage 1
            p.g = c->g;
            work = work || p.np > 0;
            if (work) LAUNCH(launch_post_stage(p, c->stream), "post stage");
        } else {
            cs = c->comm.exchange_fluxes(c);
            if (cs != AMR_OK) return cs;
            if (!c->rtasks.empty()) {
                AuxArgs x = aux(c, Uout, Uout);
                x.b = bs[s - 1];
                x.stage = s;
                x.want_lambda = s == 3;
                LAUNCH(launch_reflux(c->d_rtasks.p, (int)c->rtasks.size(), x, c->stream), "reflux");
            }
            cs = restrict_all(c, Uout);
            if (cs != AMR_OK) return cs;
        }
    }
    c->ghost_valid = fused && !c->capturing;   // the ghost strips of U^(n+1) are in the proxies
    amr_status cs = c->comm.allreduce_max_u64(c, c->d_lambda);
    if (cs != AMR_OK) return cs;
    c->un = A;
    c->st.steps++;
    c->lambda_valid = true;   // stage 3 (and the reflux) accumulated Lambda of U^(n+1)
    if (c->timing && c->ev_pending.size() > 4096) return harvest_events(c);
    return AMR_OK;
}

// read {err, dt}; on a device-reported error roll back to the pre-step buffer
amr_status finish_step(amr_ctx* c, int prev_un, double* dt_used) {
    int32_t* he = (int32_t*)c->h_pinned;
    double* hdt = (double*)((char*)c->h_pinned + 16);
    amr_status cs = c->comm.allreduce_max_i32(c, c->d_err, 1);   // every rank sees an error anywhere
    if (cs != AMR_OK) return cs;
    CU(cudaMemcpyAsync(he, c->d_err, 16, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(hdt, c->d_dt, 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (he[0] != 0) {
        int32_t e0 = he[0], slot = he[1], stage = he[2], cell = he[3];
        CU(cudaMemsetAsync(c->d_err, 0, 16, c->stream));
        if (prev_un >= 0) {
            c->un = prev_un;
            c->st.steps--;
            c->sim_time_fix -= *hdt;   // the rolled-back step's dt was added on the device
        }
        c->lambda_valid = false;
    c->ghost_valid = false;
        char b[256];
        if (e0 == 2) std::snprintf(b, sizeof b, "non-positive or non-finite time step (wave speed)");
        else if (slot >= 0 && slot < c->tree.capacity && c->tree.alive[slot])
            std::snprintf(b, sizeof b, "non-physical state at stage %d, patch (level %d, i %d, j %d), cell %d", stage,
                          c->tree.lev[slot], c->tree.pi[slot], c->tree.pj[slot], cell);
        else std::snprintf(b, sizeof b, "non-physical state at stage %d", stage);
        return fail(c, AMR_E_NONPHYSICAL, b);
    }
    c->last_dt = *hdt;
    if (dt_used) *dt_used = *hdt;
    return AMR_OK;
}

// flags on the current state (ghost-filled U^n): per-leaf max eta and ambiguity
amr_status evaluate_flags(amr_ctx* c) {
    double* Un = c->U[c->un];
    amr_status s = c->comm.exchange_halos(c, Un);
    if (s != AMR_OK) return s;
    s = fill_ghosts(c, Un);
    if (s != AMR_OK) return s;
    AuxArgs a = aux(c, Un, nullptr);
    LAUNCH(launch_flags(c->d_leaves.p, (int)c->leaves.size(), a, c->d_maxeta.p, c->d_amb.p, c->stream), "flags");
    std::vector<double> me(c->leaves.size());
    std::vector<int32_t> am(c->leaves.size());
    if (!me.empty()) {
        CU(cudaMemcpyAsync(me.data(), c->d_maxeta.p, me.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(am.data(), c->d_amb.p, am.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    }
    CU(cudaStreamSynchronize(c->stream));
    PatchTree& t = c->tree;
    // per-id arrays sized once to the slot capacity; only the entries of active patches are (re)written and read
    ensure_canon(c);
    std::vector<double>& eta = c->fl_eta_raw;
    std::vector<uint8_t>& amb = c->fl_amb_raw;
    if ((int)eta.size() != t.capacity) { eta.assign(t.capacity, std::nan("")); amb.assign(t.capacity, 0); }
    for (int id : c->canon) { eta[id] = std::nan(""); amb[id] = 0; }
    for (size_t e = 0; e < c->leaf_ids.size(); ++e) { eta[c->leaf_ids[e]] = me[e]; amb[c->leaf_ids[e]] = (uint8_t)am[e]; }
    s = c->comm.allgather_flags(c, eta, amb);
    if (s != AMR_OK) return s;
    if ((int)c->fl_eta.size() != t.capacity) {
        c->fl_eta.assign(t.capacity, std::nan(""));
        c->fl_ref.assign(t.capacity, 0);
        c->fl_crs.assign(t.capacity, 0);
        c->fl_amb.assign(t.capacity, 0);
    }
    for (int id : c->canon) { c->fl_eta[id] = std::nan(""); c->fl_ref[id] = c->fl_crs[id] = c->fl_amb[id] = 0; }
    const double th = c->cfg.refine_threshold, tc = th * c->cfg.coarsen_fraction;
    for (int id : c->canon) {
        if (t.is_leaf(id)) {
            c->fl_eta[id] = eta[id];
            c->fl_amb[id] = amb[id];
            c->fl_ref[id] = t.lev[id] < c->cfg.num_levels - 1 && eta[id] > th;
        } else {
            bool all_leaves = true;
            double m = 0.0;
            uint8_t a = 0;
            for (int q = 0; q < 4; ++q) {
                int ch = t.child[4 * id + q];
                if (!t.is_leaf(ch)) { all_leaves = false; break; }
                if (!(eta[ch] <= m)) m = eta[ch];
                a |= amb[ch];
            }
            if (all_leaves) {
                c->fl_eta[id] = m;
                c->fl_amb[id] = a;
                c->fl_crs[id] = m < tc;
            }
        }
    }
    return AMR_OK;
}

// Refine / coarsen requests of the current state with device-side compaction (single rank): the flag kernel's
// per-leaf eta stays on the device and only the (slot, bits) list of actual requests comes back.  The requests
// equal evaluate_flags' fl_ref / fl_crs (same comparisons on the same doubles); gpu test test_regrid_compact_*.
amr_status flag_requests(amr_ctx* c, std::vector<uint8_t>& ref, std::vector<uint8_t>& crs) {
    double* Un = c->U[c->un];
    amr_status s = c->comm.exchange_halos(c, Un);   // the indicator reads neighbours (remote ones on N > 1)
    if (s != AMR_OK) return s;
    if (!c->ghost_valid) {   // (the last step's post-stage kernel already filled U^n's strips: ghost_valid)
        s = fill_ghosts(c, Un);
        if (s != AMR_OK) return s;
    }
    AuxArgs a = aux(c, Un, nullptr);
    const int nl = (int)c->leaves.size(), ns = (int)c->sib.size() / 5;
    LAUNCH(launch_flags(c->d_leaves.p, nl, a, c->d_maxeta.p, c->d_amb.p, c->stream), "flags");
    const double th = c->cfg.refine_threshold, tc = th * c->cfg.coarsen_fraction;
    LAUNCH(launch_flags_compact(c->d_leaves.p, nl, c->d_sib.p, ns, c->d_maxeta.p, th, tc, c->cfg.num_levels - 1,
                                c->d_flist.p, c->d_fcount.p, c->stream), "flags compact");
    int32_t cnt = 0;
    CU(cudaMemcpyAsync(&cnt, c->d_fcount.p, 4, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (cnt < 0 || cnt > nl + ns) return fail(c, AMR_E_CUDA, "flags compact: bad request count");
    std::vector<int32_t> lst(2 * (size_t)cnt);
    if (cnt) {
        CU(cudaMemcpyAsync(lst.data(), c->d_flist.p, lst.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    s = c->comm.allgather_requests(c, lst);   // N > 1: every rank's owned requests, on every rank
    if (s != AMR_OK) return s;
    cnt = (int32_t)(lst.size() / 2);
    if ((int)ref.size() != c->tree.capacity) {
        ref.assign(c->tree.capacity, 0);
        crs.assign(c->tree.capacity, 0);
        c->rq_set.clear();
    }
    for (int id : c->rq_set) ref[id] = crs[id] = 0;   // the previous regrid's requests
    c->rq_set.clear();
    for (int32_t k = 0; k < cnt; ++k) {
        const int id = lst[2 * k], b = lst[2 * k + 1];
        if (id < 0 || id >= c->tree.capacity) return fail(c, AMR_E_CUDA, "flags compact: bad slot");
        if (b & 1) ref[id] = 1;
        if (b & 2) crs[id] = 1;
        c->rq_set.push_back(id);
    }
    return AMR_OK;
}

// refinement pass, coarsening pass, validation, new-patch prolongation, restriction
amr_status apply_regrid(amr_ctx* c, const std::vector<uint8_t>& ref, const std::vector<uint8_t>& crs,
                        const std::vector<int32_t>& req, int32_t* nr, int32_t* nc) {
    PhaseClock clk;
    PatchTree& nt = c->tree;   // modified in place inside a transaction (rolled back on any failure)
    // the requested patches in canonical order: the passes below visit exactly the patches a walk over the whole
    // canonical list would act on, in the same order, in O(requests log requests)
    std::vector<std::pair<uint64_t, int32_t>>& order = c->rq_order;
    order.clear();
    for (int id : req) order.push_back({nt.canon_key(PatchTree::key(nt.lev[id], nt.pi[id], nt.pj[id])), id});
    radix_sort_pairs(order);
    order.erase(std::unique(order.begin(), order.end()), order.end());
    nt.begin_txn();
    std::string m;
    int n_rq_ref = 0, n_rq_crs = 0, n_crs_done = 0;   // (AMR_REGRID_PROF: request statistics)
    for (const auto& o : order) {
        const int id = o.second;
        if (!ref[id] || !nt.is_leaf(id) || nt.lev[id] >= c->cfg.num_levels - 1) continue;
        ++n_rq_ref;
        if (!nt.refine(id, m)) {
            nt.rollback();
            amr_status s = m.find("capacity") != std::string::npos ? AMR_E_CAPACITY : AMR_E_MESH;
            return fail(c, s, "regrid: " + m + " (mesh unchanged)");
        }
    }
    for (int l = c->cfg.num_levels - 2; l >= 0; --l)
        for (const auto& o : order) {
            const int id = o.second;
            if (nt.lev[id] != l || !crs[id] || !nt.alive[id]) continue;
            ++n_rq_crs;
            if (nt.coarsen_allowed(id)) { nt.delete_children(id); ++n_crs_done; }
        }
    clk.mark("refine + coarsen");
    if (clk.on)
        std::fprintf(stderr, "  [regrid] requests %zu: refine %d, coarsen %d (%d done), patches %d\n", order.size(),
                     n_rq_ref, n_rq_crs, n_crs_done, nt.n_alive);
    if (!nt.validate_txn(m)) {   // O(changes); amr_plan_regrid checks it against the full validate()
        nt.rollback();
        return fail(c, AMR_E_MESH, "regrid produced an invalid mesh: " + m);
    }
    clk.mark("validate");
    int n_new = 0, n_del = 0;
    const int W = c->comm.world, R = c->comm.rank;
    std::vector<int32_t>& new_ids = c->rq_new_ids;
    new_ids.clear();
    for (const auto& sn : nt.journal()) {   // created / deleted slots, from the transaction journal
        if (nt.alive[sn.id] && !sn.alive) { new_ids.push_back(sn.id); ++n_new; }
        if (!nt.alive[sn.id] && sn.alive) ++n_del;
    }
    std::sort(new_ids.begin(), new_ids.end());
    // created / deleted slots for the incremental face-neighbour table (created in level order)
    c->nb4_created = new_ids;
    std::stable_sort(c->nb4_created.begin(), c->nb4_created.end(), [&](int a, int b) { return nt.lev[a] < nt.lev[b]; });
    c->nb4_deleted.clear();
    c->lo_rm.clear();
    c->lo_add.clear();
    for (const auto& sn : nt.journal()) {
        if (!nt.alive[sn.id] && sn.alive) c->nb4_deleted.push_back(sn.id);
        // leaves removed (refined or deleted) / added (created leaves, coarsened parents): every change of a slot's
        // leaf status is journaled (refine, alloc, release and delete_children touch the slot)
        const bool was = sn.alive && sn.child[0] < 0, now = nt.is_leaf(sn.id);
        if (was && !now) c->lo_rm.push_back({sn.lev, {morton((uint32_t)sn.pi, (uint32_t)sn.pj), sn.id}});
        if (now && !was)
            c->lo_add.push_back({nt.lev[sn.id], {morton((uint32_t)nt.pi[sn.id], (uint32_t)nt.pj[sn.id]), sn.id}});
    }
    c->nb4_incr = W == 1;
    nt.commit();
    // ownership of the new tree under the OLD partition (roots never change): the old owner of a
    // root prolongs the new patches of that root, since it holds their parents' data
    const Owners old_owner = c->comm.owner;   // root ranks of the old partition (valid for the new tree's patches)
    std::vector<std::vector<ProlongTask>> pro(c->cfg.num_levels);
    for (int id : new_ids) {
        if (W > 1 && old_owner[id] != R) continue;
        ProlongTask p{};
        p.slot = id;
        p.level = nt.lev[id];
        p.P = nt.pi[id];
        p.Q = nt.pj[id];
        int par = nt.parent[id];
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int q = (dx == 0 && dy == 0) ? par : nt.neighbour(par, dx, dy);
                if (q == -1) return fail(c, AMR_E_MESH, "prolongation: coarse neighbourhood incomplete");
                p.coarse[(dy + 1) * 3 + (dx + 1)] = q < 0 ? -1 : q;
            }
        pro[p.level].push_back(p);
    }
    clk.mark("new patches / owners");
    amr_status s = build_plan(c);
    if (s != AMR_OK) return s;
    clk.mark("build_plan");
    double* Un = c->U[c->un];
    for (int l = 1; l < c->cfg.num_levels; ++l) {
        if (W > 1) {
            ExchangeLists xl = plan_coarse(nt, new_ids, l, old_owner, W, R);
            s = c->comm.exchange_lists(c, xl, Un, (int)c->PS, "coarse exchange");
            if (s != AMR_OK) return s;
        }
        if (pro[l].empty()) continue;
        CU(c->d_prolong.upload(pro[l], c->stream));
        AuxArgs a = aux(c, Un, Un);
        LAUNCH(launch_prolong(c->d_prolong.p, (int)pro[l].size(), a, c->stream), "prolong");
        // (no synchronisation per level: the next level's upload into d_prolong is stream-ordered after this launch;
        // a growing d_prolong is freed by cudaFree, which waits for the device)
    }
    s = restrict_all(c, Un);
    if (s != AMR_OK) return s;
    clk.mark("prolong + restrict");
    if (W > 1) {
        // repartition the new tree and migrate every patch whose owner changed
        Owners new_owner = partition_owners(nt, W);
        ExchangeLists mig = plan_migration(nt, old_owner, new_owner, W, R);
        s = c->comm.exchange_lists(c, mig, Un, (int)c->PS, "migration");
        if (s != AMR_OK) return s;
        c->comm.owner = new_owner;
        s = build_plan(c);
        if (s != AMR_OK) return s;
    }
    CU(cudaStreamSynchronize(c->stream));
    c->lambda_valid = false;
    c->ghost_valid = false;
    if ((int)c->fl_eta.size() == nt.capacity) {   // no requests on the new mesh until the next flag evaluation
        ensure_canon(c);
        for (int id : c->canon) { c->fl_eta[id] = std::nan(""); c->fl_ref[id] = c->fl_crs[id] = c->fl_amb[id] = 0; }
    }
    if (nr) *nr = n_new;
    if (nc) *nc = n_del;
    clk.mark("finish");
    return AMR_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int32_t amr_abi_version(void) { return AMR_ABI_VERSION; }

amr_status amr_default_config(amr_config* cfg) {
    if (!cfg) return AMR_E_ARG;
    std::memset(cfg, 0, sizeof *cfg);
    cfg->dim = 2;
    cfg->lo[0] = cfg->lo[1] = 0.0;
    cfg->hi[0] = cfg->hi[1] = 1.0;
    cfg->base_cells[0] = cfg->base_cells[1] = 64;
    cfg->patch_cells = 16;
    cfg->num_levels = 1;
    cfg->ratio = 2;
    cfg->gamma = 1.4;
    for (int s = 0; s < 4; ++s) cfg->bc[s] = AMR_BC_PERIODIC;
    cfg->scheme = AMR_CENTRAL4;
    cfg->weno_characteristic = 1;
    cfg->div_order = 4;
    cfg->weno_eps = 1e-6;
    cfg->refine_threshold = 0.1;
    cfg->coarsen_fraction = 0.25;
    cfg->coarsen_rule = AMR_COARSEN_R2_EXACT;
    cfg->max_patches = 4096;
    cfg->device = -1;
    cfg->world_size = 1;
    cfg->rank = 0;
    cfg->check_positivity = 1;
    cfg->use_graphs = 0;
    cfg->stage_kernel = 0;
    return AMR_OK;
}

amr_status amr_query_pool_bytes(const amr_config* cfg, uint64_t* bytes) {
    if (!cfg || !bytes) return AMR_E_ARG;
    *bytes = 3ull * (uint64_t)cfg->max_patches * 4ull * (uint64_t)cfg->patch_cells * cfg->patch_cells * 8ull;
    return AMR_OK;
}

amr_status amr_create(const amr_config* cfg, amr_ctx** out) {
    if (!cfg || !out) return AMR_E_ARG;
    *out = nullptr;
    std::string m;
    amr_status vs = validate_config(cfg, m);
    if (vs != AMR_OK) {
        std::fprintf(stderr, "amr_create: %s\n", m.c_str());
        return vs;
    }
    std::unique_ptr<amr_ctx> h(new amr_ctx());
    amr_ctx* c = h.get();
    c->cfg = *cfg;
    c->n = cfg->patch_cells;
    c->PS = 4ull * c->n * c->n;
    const int npx = cfg->base_cells[0] / c->n, npy = cfg->base_cells[1] / c->n;
    if ((int64_t)npx * npy > cfg->max_patches) {
        std::fprintf(stderr, "amr_create: %d roots exceed max_patches %d\n", npx * npy, cfg->max_patches);
        return AMR_E_CAPACITY;
    }
    if (cfg->device >= 0) CU(cudaSetDevice(cfg->device));
    c->tree.init(npx, npy, cfg->num_levels, cfg->bc[0] == AMR_BC_PERIODIC, cfg->bc[2] == AMR_BC_PERIODIC,
                 cfg->max_patches, cfg->coarsen_rule);
    Geometry& G = c->geo;
    G.n = c->n;
    for (int s = 0; s < 4; ++s) G.bc[s] = cfg->bc[s];
    for (int l = 0; l < kMaxLevels; ++l) {
        G.nc[0][l] = l < cfg->num_levels ? cfg->base_cells[0] << l : 0;
        G.nc[1][l] = l < cfg->num_levels ? cfg->base_cells[1] << l : 0;
        // O1: dx_l = (hi - lo) / (N * 2^l)
        G.dx[l] = (cfg->hi[0] - cfg->lo[0]) / ((double)cfg->base_cells[0] * (double)(1 << std::min(l, 30)));
        G.dy[l] = (cfg->hi[1] - cfg->lo[1]) / ((double)cfg->base_cells[1] * (double)(1 << std::min(l, 30)));
        G.inv_dx[l] = 1.0 / G.dx[l];
        G.inv_dy[l] = 1.0 / G.dy[l];
    }
    if (cfg->cuda_stream) c->stream = (cudaStream_t)cfg->cuda_stream;
    else {
        CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    uint64_t need = 0;
    amr_query_pool_bytes(cfg, &need);
    char* base = nullptr;
    if (cfg->pool) {
        if (cfg->pool_bytes < need) {
            std::fprintf(stderr, "amr_create: pool too small (%llu < %llu bytes)\n", (unsigned long long)cfg->pool_bytes,
                         (unsigned long long)need);
            return AMR_E_ARG;
        }
        base = (char*)cfg->pool;
    } else if (nccl_windows(c)) {   // symmetric NCCL window memory (peer_map 1)
        std::string e;
        c->own_pool = comm_nccl_mem_alloc(need, e);
        if (!c->own_pool) { std::fprintf(stderr, "amr_create: %s\n", e.c_str()); return AMR_E_COMM; }
        c->own_pool_nccl = true;
        base = (char*)c->own_pool;
    } else {
        CU(cudaMalloc(&c->own_pool, need));
        base = (char*)c->own_pool;
    }
    for (int b = 0; b < 3; ++b) c->U[b] = (double*)(base + (size_t)b * (need / 3));
    CU(cudaMemsetAsync(base, 0, need, c->stream));
    CU(cudaMalloc(&c->d_dt, 8 * (kMaxLevels + 1)));   // dt per level (subcycling; dt[0] otherwise), simulated time
    CU(cudaMemset(c->d_dt, 0, 8 * (kMaxLevels + 1)));
    CU(cudaMalloc(&c->d_lambda, 8));
    CU(cudaMalloc(&c->d_tmp, 8));
    CU(cudaMalloc(&c->d_err, 16));
    CU(cudaMalloc(&c->d_dtp, 16));
    CU(cudaMemsetAsync(c->d_err, 0, 16, c->stream));
    CU(cudaMallocHost(&c->h_pinned, 64));
    amr_status s = c->comm.init(c);
    if (s == AMR_OK && c->comm.world > 1 && c->comm.halo_mode >= 1) s = c->comm.map_pool(c, base, need);
    if (s != AMR_OK) {
        std::fprintf(stderr, "amr_create: %s\n", c->err.c_str());
        return s;
    }
    s = build_plan(c);
    if (s != AMR_OK) {
        std::fprintf(stderr, "amr_create: %s\n", c->err.c_str());
        return s;
    }
    *out = h.release();
    return AMR_OK;
}

void amr_destroy(amr_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    trace_dump(c);
    c->comm.finalize(c);
    c->d_leaves.release(); c->d_gleaves.release(); c->d_singles.release(); c->d_ptasks.release(); c->d_rtasks.release(); c->d_prolong.release();
    for (auto& d : c->d_rlev) d.release();
    c->proxy.release(); c->freg.release(); c->staging.release(); c->d_maxeta.release(); c->d_partial.release();
    c->unf_scratch.release();
    c->d_slots.release(); c->d_amb.release(); c->d_sib.release(); c->d_flist.release(); c->d_fcount.release();
    c->arena_dev.release();
    if (c->freg_nccl) { c->freg.release(); comm_nccl_mem_free(c->freg_nccl); }
    if (c->own_pool) { if (c->own_pool_nccl) comm_nccl_mem_free(c->own_pool); else cudaFree(c->own_pool); }
    cudaFree(c->d_dt); cudaFree(c->d_lambda); cudaFree(c->d_err); cudaFree(c->d_tmp); cudaFree(c->d_dtp);
    for (auto& g : c->gexec) if (g) cudaGraphExecDestroy(g);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->arena_host) cudaFreeHost(c->arena_host);
    if (c->arena_ev) cudaEventDestroy(c->arena_ev);
    for (auto e : c->ev_free) cudaEventDestroy(e);
    for (auto e : c->ev_pending) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}

static amr_status select_local(amr_ctx* c, int32_t npatch, const int32_t* tree_index, std::vector<int32_t>& slots,
                               std::vector<int32_t>& which) {
    ensure_canon(c);
    slots.clear();
    which.clear();
    for (int k = 0; k < npatch; ++k) {
        int ti = tree_index[k];
        if (ti < 0 || ti >= (int)c->canon.size()) return fail(c, AMR_E_ARG, "tree_index out of range");
        int id = c->canon[ti];
        if (!c->comm.owns(c, id)) continue;
        slots.push_back(id);
        which.push_back(k);
    }
    return AMR_OK;
}

amr_status amr_set_state_fn(amr_ctx* c, amr_ic_fn fn, void* user) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (!fn) return fail(c, AMR_E_ARG, "set_state_fn: null callback");
    // every locally owned active patch (leaves and covered patches), sampled at its cell centres (A33)
    const PatchTree& t = c->tree;
    const int n = c->n;
    const size_t PS = c->PS, nn = (size_t)n * n;
    ensure_canon(c);
    std::vector<int32_t> idx;
    for (size_t e = 0; e < c->canon.size(); ++e)
        if (c->comm.owns(c, c->canon[e])) idx.push_back((int32_t)e);
    std::vector<double> U(idx.size() * PS), x(nn), y(nn);
    for (size_t k = 0; k < idx.size(); ++k) {
        const int id = c->canon[idx[k]];
        const int l = t.lev[id];
        const double dx = c->geo.dx[l], dy = c->geo.dy[l];
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                x[(size_t)j * n + i] = c->cfg.lo[0] + ((double)t.pi[id] * n + i + 0.5) * dx;
                y[(size_t)j * n + i] = c->cfg.lo[1] + ((double)t.pj[id] * n + j + 0.5) * dy;
            }
        fn((int32_t)nn, x.data(), y.data(), U.data() + k * PS, user);
    }
    return amr_set_state(c, (int32_t)idx.size(), idx.data(), U.data());
}

amr_status amr_set_state(amr_ctx* c, int32_t npatch, const int32_t* tree_index, const double* U) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (npatch < 0 || (npatch > 0 && (!tree_index || !U))) return fail(c, AMR_E_ARG, "set_state: bad arguments");
    std::vector<int32_t> slots, which;
    s = select_local(c, npatch, tree_index, slots, which);
    if (s != AMR_OK) return s;
    const size_t PS = c->PS;
    const size_t chunk = 8192;   // patches per staging round
    for (size_t b = 0; b < slots.size(); b += chunk) {
        size_t m = std::min(chunk, slots.size() - b);
        CU(c->staging.reserve(m * PS));
        CU(c->d_slots.reserve(m));
        bool contiguous = true;
        for (size_t k = 1; k < m; ++k) contiguous &= which[b + k] == which[b] + (int)k;
        if (contiguous) {
            CU(cudaMemcpyAsync(c->staging.p, U + (size_t)which[b] * PS, m * PS * 8, cudaMemcpyHostToDevice, c->stream));
        } else {
            for (size_t k = 0; k < m; ++k)
                CU(cudaMemcpyAsync(c->staging.p + k * PS, U + (size_t)which[b + k] * PS, PS * 8, cudaMemcpyHostToDevice,
                                   c->stream));
        }
        CU(cudaMemcpyAsync(c->d_slots.p, slots.data() + b, m * 4, cudaMemcpyHostToDevice, c->stream));
        LAUNCH(launch_scatter(c->staging.p, c->d_slots.p, (int)m, c->U[c->un], (int)PS, c->stream), "scatter");
        CU(cudaStreamSynchronize(c->stream));
    }
    s = c->comm.exchange_children(c, c->U[c->un]);
    if (s != AMR_OK) return s;
    s = restrict_all(c, c->U[c->un]);
    if (s != AMR_OK) return s;
    CU(cudaStreamSynchronize(c->stream));
    c->lambda_valid = false;
    c->ghost_valid = false;
    return AMR_OK;
}

amr_status amr_set_state_device(amr_ctx* c, int32_t npatch, const int32_t* tree_index, const double* dU) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (npatch < 0 || (npatch > 0 && (!tree_index || !dU))) return fail(c, AMR_E_ARG, "set_state_device: bad arguments");
    std::vector<int32_t> slots, which;
    s = select_local(c, npatch, tree_index, slots, which);
    if (s != AMR_OK) return s;
    const size_t PS = c->PS;
    std::vector<int32_t> src_slots(slots.size());
    // scatter row k of dU (packed) into its slot: a packed index list per chunk
    const size_t chunk = 1 << 20;
    for (size_t b = 0; b < slots.size(); b += chunk) {
        size_t m = std::min(chunk, slots.size() - b);
        bool contiguous = true;
        for (size_t k = 1; k < m; ++k) contiguous &= which[b + k] == which[b] + (int)k;
        if (!contiguous) return fail(c, AMR_E_ARG, "set_state_device: tree_index rows of local patches must be contiguous");
        CU(c->d_slots.reserve(m));
        CU(cudaMemcpyAsync(c->d_slots.p, slots.data() + b, m * 4, cudaMemcpyHostToDevice, c->stream));
        LAUNCH(launch_scatter(dU + (size_t)which[b] * PS, c->d_slots.p, (int)m, c->U[c->un], (int)PS, c->stream), "scatter");
        CU(cudaStreamSynchronize(c->stream));
    }
    s = c->comm.exchange_children(c, c->U[c->un]);
    if (s != AMR_OK) return s;
    s = restrict_all(c, c->U[c->un]);
    if (s != AMR_OK) return s;
    c->lambda_valid = false;
    c->ghost_valid = false;
    return AMR_OK;
}

amr_status amr_get_state_device(amr_ctx* c, int32_t npatch, const int32_t* tree_index, double* dU_out) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (npatch < 0 || (npatch > 0 && (!tree_index || !dU_out))) return fail(c, AMR_E_ARG, "get_state_device: bad arguments");
    std::vector<int32_t> slots, which;
    s = select_local(c, npatch, tree_index, slots, which);
    if (s != AMR_OK) return s;
    for (size_t k = 1; k < which.size(); ++k)
        if (which[k] != which[0] + (int)k) return fail(c, AMR_E_ARG, "get_state_device: local rows must be contiguous");
    if (slots.empty()) return AMR_OK;
    CU(c->d_slots.reserve(slots.size()));
    CU(cudaMemcpyAsync(c->d_slots.p, slots.data(), slots.size() * 4, cudaMemcpyHostToDevice, c->stream));
    LAUNCH(launch_gather(c->U[c->un], c->d_slots.p, (int)slots.size(), dU_out + (size_t)which[0] * c->PS, (int)c->PS,
                         c->stream), "gather");
    CU(cudaStreamSynchronize(c->stream));
    return AMR_OK;
}

amr_status amr_get_state(amr_ctx* c, int32_t npatch, const int32_t* tree_index, double* U_out) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (npatch < 0 || (npatch > 0 && (!tree_index || !U_out))) return fail(c, AMR_E_ARG, "get_state: bad arguments");
    std::vector<int32_t> slots, which;
    s = select_local(c, npatch, tree_index, slots, which);
    if (s != AMR_OK) return s;
    const size_t PS = c->PS;
    const size_t chunk = 8192;
    std::vector<double> host;
    for (size_t b = 0; b < slots.size(); b += chunk) {
        size_t m = std::min(chunk, slots.size() - b);
        CU(c->staging.reserve(m * PS));
        CU(c->d_slots.reserve(m));
        CU(cudaMemcpyAsync(c->d_slots.p, slots.data() + b, m * 4, cudaMemcpyHostToDevice, c->stream));
        LAUNCH(launch_gather(c->U[c->un], c->d_slots.p, (int)m, c->staging.p, (int)PS, c->stream), "gather");
        bool contiguous = true;
        for (size_t k = 1; k < m; ++k) contiguous &= which[b + k] == which[b] + (int)k;
        if (contiguous) {
            CU(cudaMemcpyAsync(U_out + (size_t)which[b] * PS, c->staging.p, m * PS * 8, cudaMemcpyDeviceToHost, c->stream));
        } else {
            for (size_t k = 0; k < m; ++k)
                CU(cudaMemcpyAsync(U_out + (size_t)which[b + k] * PS, c->staging.p + k * PS, PS * 8,
                                   cudaMemcpyDeviceToHost, c->stream));
        }
        CU(cudaStreamSynchronize(c->stream));
    }
    return AMR_OK;
}

// ---------------------------------------------------------------- subcycled step (NEXT #4, S1-S6)
// Buffer rotation: every level starts the coarse step in buffer un and must end it in (un + 1) % 3.  A level-l
// step moves its current buffer by +1 or +2 (stage outputs in the two other buffers); level l takes 2^l steps, so
// the increments are chosen with sum = 1 (mod 3): 2^l - k ones then k twos, k = (1 - 2^l) mod 3.  Levels own
// disjoint slots, so a level's old (step start) and new buffers stay intact while the next level interpolates.
struct SubRun {
    amr_ctx* c;
    int L;
    int cur[kMaxLevels], start[kMaxLevels], nstep[kMaxLevels];
    int inc(int l) const {
        const int m = 1 << l, k = ((1 - m) % 3 + 3) % 3;
        return nstep[l] >= m - k ? 2 : 1;
    }
    // a level takes part in the recursion when it exists anywhere in the replicated tree (every rank must make the
    // same sequence of collective exchanges, whether or not it owns patches of the level)
    bool has_level(int l) const { return l < L && l < c->sub_levels; }
    amr_status xchg(const ExchangeLists& x, double* buf, int per, const char* what) {
        return c->comm.world > 1 ? c->comm.exchange_lists(c, x, buf, per, what, true) : AMR_OK;   // (plan lists)
    }

    amr_status advance(int l, bool final, int sub_i) {
        static const double as[3] = {0.0, 0.75, 1.0 / 3.0}, bs[3] = {1.0, 0.25, 2.0 / 3.0};
        static const double cs[3] = {0.0, 1.0, 0.5}, ws[3] = {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0};
        const int P = (cur[l] + inc(l)) % 3, Q = 3 - cur[l] - P;
        start[l] = cur[l];
        double* Un = c->U[cur[l]];
        const int n0 = c->sub_off[l], nl = c->sub_off[l + 1] - n0;
        const int p0 = c->sub_poff[l], pl = c->sub_poff[l + 1] - p0;
        const int a0 = c->acc_off[l], al = c->acc_off[l + 1] - a0;
        for (int s = 1; s <= 3; ++s) {
            double* Uin = s == 1 ? Un : (s == 2 ? c->U[P] : c->U[Q]);
            double* Uout = s == 2 ? c->U[Q] : c->U[P];
            amr_status xs = xchg(c->comm.sub.face.empty() ? ExchangeLists() : c->comm.sub.face[l], Uin, (int)c->PS,
                                 "subcycle face halo");
            if (xs != AMR_OK) return xs;
            if (pl > 0) {   // ghosts: physical BC from the stage input, C/F from level l-1 in time (S2)
                AuxArgs g = aux(c, Uin, nullptr);
                g.proxy = c->sub_proxy.p;
                if (l > 0) {
                    g.Uc = c->U[cur[l - 1]];
                    g.Uold = c->U[start[l - 1]];
                    g.tfrac = (sub_i + cs[s - 1]) * 0.5;
                }
                LAUNCH(launch_ghost(c->d_sub_ptasks.p + p0, pl, c->g, g, c->stream), "ghost");
            }
            StageArgs a{};
            a.leaves = c->d_sub_descs.p + n0;
            a.nleaves = nl;
            a.tiles = c->n > 32 ? c->n / 32 : 1;
            a.Uin = Uin;
            a.Un = Un;
            a.Uout = Uout;
            a.proxy = c->sub_proxy.p;
            a.freg = c->freg.p;
            a.dt = c->d_dt + l;
            a.a = as[s - 1];
            a.b = bs[s - 1];
            a.stage = s;
            a.div_order = c->cfg.div_order;
            a.characteristic = c->cfg.weno_characteristic;
            a.check = c->cfg.check_positivity;
            a.want_lambda = final && s == 3;
            a.lam0 = 1;
            a.gamma = c->cfg.gamma;
            a.eps = c->cfg.weno_eps;
            a.lambda_bits = c->d_lambda;
            a.err = c->d_err;
            a.nslots = c->cfg.max_patches;
            a.nproxy = (int32_t)(c->sub_proxy.cap / c->PS);
            a.variant = c->cfg.stage_kernel;
            a.scratch = c->unf_scratch.p;
            a.geo = c->geo;
            const int scheme = c->cfg.scheme == AMR_CENTRAL4 ? 0 : (c->cfg.weno_characteristic ? 1 : 2);
            LAUNCH(launch_stage(scheme, a, c->stream), "stage");
            c->st.launches += stage_launches_per_stage(a.variant, a.nleaves) - 1;
            c->st.stage_launches++;
            if (al > 0)
                LAUNCH(launch_accumulate(c->d_acc_tasks.p + a0, al, c->n, c->freg.p, c->facc.p, ws[s - 1], 0.5 * ws[s - 1],
                                         s == 1, s == 1 && sub_i == 0, c->stream), "accumulate");
        }
        cur[l] = P;
        nstep[l]++;
        if (!has_level(l + 1)) return AMR_OK;
        if (c->comm.world > 1) {   // coarse sources of level l+1's C/F ghosts, at the start and the end of this step
            amr_status xs = xchg(c->comm.sub.coarse[l + 1], c->U[cur[l]], (int)c->PS, "subcycle coarse sources (new)");
            if (xs == AMR_OK) xs = xchg(c->comm.sub.coarse[l + 1], c->U[start[l]], (int)c->PS, "subcycle coarse sources (old)");
            if (xs != AMR_OK) return xs;
        }
        amr_status st = advance(l + 1, false, 0);
        if (st != AMR_OK) return st;
        st = advance(l + 1, final, 1);
        if (st != AMR_OK) return st;
        const int r0 = c->rt_off[l], rl = c->rt_off[l + 1] - r0;
        if (c->comm.world > 1) {   // accumulated registers of remote fine leaves on this level's C/F faces
            st = xchg(c->comm.sub.facc[l], c->facc.p, 16 * c->n, "subcycle flux registers");
            if (st != AMR_OK) return st;
        }
        if (rl > 0) {   // S4
            AuxArgs x = aux(c, c->U[cur[l]], c->U[cur[l]]);
            x.freg = c->facc.p;
            x.dt = c->d_dt + l;
            x.b = 1.0;
            x.stage = 3;
            x.want_lambda = final;
            x.lam0 = 1;
            LAUNCH(launch_reflux(c->d_rtasks.p + r0, rl, x, c->stream), "reflux");
        }
        if (!c->rlev[l + 1].empty()) {   // O9: level l+1 into the covered level-l patches
            AuxArgs r = aux(c, c->U[cur[l + 1]], c->U[cur[l]]);
            LAUNCH(launch_restrict(c->d_rlev[l + 1].p, (int)c->rlev[l + 1].size(), r, c->stream), "restrict");
        }
        return AMR_OK;
    }
};

amr_status enqueue_step_subcycled(amr_ctx* c, double dt, double cfl) {
    if (!c->lambda_valid && !(dt > 0.0)) {
        amr_status s = seed_lambda(c);
        if (s != AMR_OK) return s;
    }
    LAUNCH(launch_dt(c->d_dt, c->d_lambda, c->d_err, dt, cfl, c->stream), "dt");
    LAUNCH(launch_dt_levels(c->d_dt, c->cfg.num_levels, c->stream), "dt levels");
    SubRun r{};
    r.c = c;
    r.L = c->cfg.num_levels;
    for (int l = 0; l < kMaxLevels; ++l) { r.cur[l] = r.start[l] = c->un; r.nstep[l] = 0; }
    amr_status s = r.advance(0, true, 0);
    if (s != AMR_OK) return s;
    s = c->comm.allreduce_max_u64(c, c->d_lambda);   // Lambda of U^(n+1) over all ranks
    if (s != AMR_OK) return s;
    for (int l = 0; l < r.L; ++l)
        if (r.has_level(l) && r.cur[l] != (c->un + 1) % 3)
            return fail(c, AMR_E_STATE, "subcycle: buffer rotation out of step");
    c->un = (c->un + 1) % 3;
    c->st.steps++;
    c->lambda_valid = true;
    c->ghost_valid = false;
    return AMR_OK;
}

// One step as a CUDA graph replay (use_graphs, one rank, kernel timing off): the launch sequence of
// enqueue_step is captured once per position of U^n in the buffer rotation and per plan, and replayed with the
// step's (dt, cfl) written to device memory first.  Host bookkeeping is the same as enqueue_step's.
amr_status enqueue_step_graph(amr_ctx* c, double dt, double cfl) {
    if (!c->lambda_valid && !(dt > 0.0)) {
        amr_status s = seed_lambda(c);
        if (s != AMR_OK) return s;
    }
    const int u = c->un;
    if (!c->gexec[u] || c->gver[u] != c->plan_version) {
        if (c->gexec[u]) { cudaGraphExecDestroy(c->gexec[u]); c->gexec[u] = nullptr; }
        const int64_t l0 = c->st.launches, sl0 = c->st.stage_launches, st0 = c->st.steps;
        const bool lv = c->lambda_valid;
        cudaGraph_t g = nullptr;
        CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        c->capturing = true;
        amr_status s = enqueue_step(c, dt, cfl);
        c->capturing = false;
        cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        c->glaunches[u] = c->st.launches - l0;
        c->st.launches = l0;
        c->st.stage_launches = sl0;
        c->st.steps = st0;
        c->un = u;
        c->lambda_valid = lv;
        if (s != AMR_OK) { if (g) cudaGraphDestroy(g); return s; }
        if (e != cudaSuccess) return fail(c, AMR_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        e = cudaGraphInstantiate(&c->gexec[u], g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(c, AMR_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
        c->gver[u] = c->plan_version;
    }
    LAUNCH(launch_set2(c->d_dtp, dt, cfl, c->stream), "dt params");
    CU(cudaGraphLaunch(c->gexec[u], c->stream));
    c->st.launches += c->glaunches[u];
    c->st.stage_launches += 3;
    c->un = (u + 1) % 3;
    c->st.steps++;
    c->lambda_valid = true;
    c->ghost_valid = false;   // the captured stage 3 does not refill (its stage 1 always does)
    return AMR_OK;
}

// graphs pay off only when a plan is replayed many times: capture once the current plan has served kGraphAfter
// stream-launched steps (a regrid every few steps would otherwise re-capture all the time)
constexpr int kGraphAfter = 3;
bool use_graph(const amr_ctx* c) {
    return c->cfg.use_graphs && c->cfg.world_size == 1 && !c->timing && c->plan_steps >= kGraphAfter &&
           !c->cfg.subcycle;
}
amr_status enqueue_any_step(amr_ctx* c, double dt, double cfl) {
    if (c->cfg.subcycle) return enqueue_step_subcycled(c, dt, cfl);
    return use_graph(c) ? enqueue_step_graph(c, dt, cfl) : enqueue_step(c, dt, cfl);
}

amr_status amr_step(amr_ctx* c, double dt, double cfl, double* dt_used) {
    NvtxRange nv("amr_step");
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (!(dt > 0.0) && !(cfl > 0.0)) return fail(c, AMR_E_ARG, "step: need dt > 0 or cfl > 0");
    int prev = c->un;
    s = enqueue_any_step(c, dt, cfl);
    c->plan_steps++;
    if (s != AMR_OK) return s;
    if (c->cfg.check_positivity || dt_used) return finish_step(c, prev, dt_used);
    return AMR_OK;
}

amr_status amr_steps(amr_ctx* c, int32_t nsteps, double dt, double cfl) {
    NvtxRange nv("amr_steps");
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (nsteps < 0 || (!(dt > 0.0) && !(cfl > 0.0))) return fail(c, AMR_E_ARG, "steps: bad arguments");
    for (int k = 0; k < nsteps; ++k) {
        s = enqueue_any_step(c, dt, cfl);
        if (s != AMR_OK) return s;
        c->plan_steps++;
    }
    return AMR_OK;
}

amr_status amr_sync(amr_ctx* c) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    s = harvest_events(c);
    if (s != AMR_OK) return s;
    return finish_step(c, -1, nullptr);
}

amr_status amr_get_flags(amr_ctx* c, int32_t cap, double* maxeta, uint8_t* bits) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    ensure_canon(c);
    if (cap < (int)c->canon.size() || !maxeta || !bits) return fail(c, AMR_E_ARG, "get_flags: capacity");
    s = evaluate_flags(c);
    if (s != AMR_OK) return s;
    for (size_t e = 0; e < c->canon.size(); ++e) {
        int id = c->canon[e];
        maxeta[e] = c->fl_eta[id];
        bits[e] = (uint8_t)(c->fl_ref[id] | (c->fl_crs[id] << 1) | (c->fl_amb[id] << 2));
    }
    return AMR_OK;
}

amr_status amr_regrid(amr_ctx* c, int32_t* n_refined, int32_t* n_coarsened) {
    NvtxRange nv("amr_regrid");
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    PhaseClock clk;
    std::vector<uint8_t>& ref = c->rq_ref;
    std::vector<uint8_t>& crs = c->rq_crs;
    s = flag_requests(c, ref, crs);   // device-compacted requests; on N > 1 the ranks' lists are exchanged
    if (s != AMR_OK) return s;
    clk.mark("flags");
    return apply_regrid(c, ref, crs, c->rq_set, n_refined, n_coarsened);
}

amr_status amr_regrid_with_flags(amr_ctx* c, int32_t n, const int32_t* tree_index, const uint8_t* bits,
                                 int32_t* n_refined, int32_t* n_coarsened) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (n < 0 || (n > 0 && (!tree_index || !bits))) return fail(c, AMR_E_ARG, "regrid_with_flags: bad arguments");
    ensure_canon(c);
    std::vector<uint8_t> ref(c->tree.capacity, 0), crs(c->tree.capacity, 0);
    std::vector<int32_t> req(n);
    for (int k = 0; k < n; ++k) {
        int ti = tree_index[k];
        if (ti < 0 || ti >= (int)c->canon.size()) return fail(c, AMR_E_ARG, "regrid_with_flags: tree_index");
        ref[c->canon[ti]] = bits[k] & 1;
        crs[c->canon[ti]] = (bits[k] >> 1) & 1;
        req[k] = c->canon[ti];
    }
    CU(cudaStreamSynchronize(c->stream));
    return apply_regrid(c, ref, crs, req, n_refined, n_coarsened);
}

amr_status amr_get_patch_tree(amr_ctx* c, amr_patch_desc* out, int32_t cap, int32_t* count) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (!count) return fail(c, AMR_E_ARG, "get_patch_tree: count is NULL");
    ensure_canon(c);
    *count = (int32_t)c->canon.size();
    if (!out || cap < *count) return fail(c, AMR_E_ARG, "get_patch_tree: capacity smaller than the patch count");
    const PatchTree& t = c->tree;
    static const int moore[8][2] = {{0, 1}, {1, 0}, {0, -1}, {-1, 0}, {1, 1}, {1, -1}, {-1, -1}, {-1, 1}};
    auto tix = [&](int id) { return id >= 0 ? c->canon_pos[id] : -1; };
    for (size_t e = 0; e < c->canon.size(); ++e) {
        int id = c->canon[e];
        amr_patch_desc& d = out[e];
        d.level = t.lev[id];
        d.i = t.pi[id];
        d.j = t.pj[id];
        d.parent = tix(t.parent[id]);
        for (int q = 0; q < 4; ++q) d.child[q] = tix(t.child[4 * id + q]);
        for (int q = 0; q < 8; ++q) {
            int nb = t.neighbour(id, moore[q][0], moore[q][1]);
            d.nbr[q] = nb >= 0 ? tix(nb) : -1;
        }
        d.owner = c->comm.owner_of(c, id);
        d.leaf = t.is_leaf(id);
        d.refine_req = id < (int)c->fl_ref.size() ? c->fl_ref[id] : 0;
        d.coarsen_req = id < (int)c->fl_crs.size() ? c->fl_crs[id] : 0;
        d.ambiguous = id < (int)c->fl_amb.size() ? c->fl_amb[id] : 0;
    }
    return AMR_OK;
}

amr_status amr_diagnostics(amr_ctx* c, double totals[4], double* lambda_max) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    CU(cudaStreamSynchronize(c->stream));
    AuxArgs a = aux(c, c->U[c->un], nullptr);
    if (totals) {
        LAUNCH(launch_totals(c->d_leaves.p, (int)c->leaves.size(), a, c->d_partial.p, c->stream), "totals");
        std::vector<double> part(4 * c->leaves.size());
        if (!part.empty())
            CU(cudaMemcpyAsync(part.data(), c->d_partial.p, part.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        // combine in canonical order (deterministic), long double accumulation
        ensure_canon(c);
        std::vector<int32_t> order(c->leaves.size());
        for (size_t e = 0; e < order.size(); ++e) order[e] = (int32_t)e;
        std::sort(order.begin(), order.end(),
                  [&](int x, int y) { return c->canon_pos[c->leaf_ids[x]] < c->canon_pos[c->leaf_ids[y]]; });
        long double acc[4] = {0, 0, 0, 0};
        for (int e : order)
            for (int k = 0; k < 4; ++k) acc[k] += part[4 * (size_t)e + k];
        double loc[4];
        for (int k = 0; k < 4; ++k) loc[k] = (double)acc[k];
        s = c->comm.allreduce_sum4(c, loc);
        if (s != AMR_OK) return s;
        for (int k = 0; k < 4; ++k) totals[k] = loc[k];
    }
    if (lambda_max) {
        AuxArgs b = a;
        b.lambda_bits = c->d_tmp;
        CU(cudaMemsetAsync(c->d_tmp, 0, 8, c->stream));
        LAUNCH(launch_lambda(c->d_leaves.p, (int)c->leaves.size(), b, c->stream), "lambda");
        s = c->comm.allreduce_max_u64(c, c->d_tmp);
        if (s != AMR_OK) return s;
        unsigned long long bits = 0;
        CU(cudaMemcpyAsync(&bits, c->d_tmp, 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        std::memcpy(lambda_max, &bits, 8);
    }
    return AMR_OK;
}

amr_status amr_set_kernel_timing(amr_ctx* c, int32_t enable) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    c->timing = enable != 0;
    return AMR_OK;
}

amr_status amr_get_stats(amr_ctx* c, amr_stats* out) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    if (!out) return fail(c, AMR_E_ARG, "get_stats: NULL");
    s = harvest_events(c);
    if (s != AMR_OK) return s;
    double t = 0.0;
    CU(cudaMemcpyAsync(&t, c->d_dt + kMaxLevels, 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    c->st.sim_time = t + c->sim_time_fix;
    *out = c->st;
    return AMR_OK;
}

amr_status amr_reset_stats(amr_ctx* c) {
    amr_status s = check(c);
    if (s != AMR_OK) return s;
    s = harvest_events(c);
    if (s != AMR_OK) return s;
    amr_stats keep = c->st;
    std::memset(&c->st, 0, sizeof c->st);
    c->st.leaf_cells = keep.leaf_cells;
    c->st.leaves = keep.leaves;
    c->st.patches = keep.patches;
    c->st.proxies = keep.proxies;
    CU(cudaMemsetAsync(c->d_dt + kMaxLevels, 0, 8, c->stream));
    c->sim_time_fix = 0.0;
    return AMR_OK;
}

const char* amr_last_error(const amr_ctx* c) { return c ? c->err.c_str() : "null context"; }

}  // extern "C"
