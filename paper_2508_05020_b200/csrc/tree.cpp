// tree.cpp -- see tree.h.  Citations: PAPER.md (P:Lnn), DESIGN.md s3 readings.
#include "tree.h"

#include <algorithm>
#include <functional>

namespace amr {

namespace {
// Fig. 2 nbr order: N, E, S, W, NE, SE, SW, NW
const int kMoore[8][2] = {{0, 1}, {1, 0}, {0, -1}, {-1, 0}, {1, 1}, {1, -1}, {-1, -1}, {-1, 1}};
inline int pmod(int a, int b) { int r = a % b; return r < 0 ? r + b : r; }
uint64_t spread(uint32_t v) {
    uint64_t x = v;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}
uint64_t morton_key(uint32_t x, uint32_t y) { return spread(x) | (spread(y) << 1); }
}  // namespace

void PatchTree::init(int npx, int npy, int nlev, bool perx, bool pery, int cap, int rule) {
    np0[0] = npx; np0[1] = npy; levels = nlev;
    periodic[0] = perx; periodic[1] = pery;
    capacity = cap; coarsen_rule = rule;
    for (int ax = 0; ax < 2; ++ax) {
        kb[ax] = 0;
        while ((int64_t(1) << kb[ax]) < (int64_t(ax ? npy : npx) << (nlev - 1))) ++kb[ax];
    }
    lev.assign(cap, -1); pi.assign(cap, 0); pj.assign(cap, 0); parent.assign(cap, -1);
    child.assign(4 * (size_t)cap, -1); alive.assign(cap, 0);
    node_.assign(cap, Node{-1, 0, 0, -1, {-1, -1, -1, -1}});
    n_alive = 0;
    index_.clear();
    index_.reserve((size_t)npx * npy * 2);
    free_.clear();
    for (int s = cap - 1; s >= 0; --s) free_.push_back(s);
    std::make_heap(free_.begin(), free_.end(), std::greater<int32_t>());
    // R1: the permanent root scaffold, allocated in Morton order of (i, j) so that every aligned 2^k x 2^k block
    // of roots occupies consecutive slots (the Central4 group kernel then moves a block with one bulk copy)
    std::vector<std::pair<uint64_t, int32_t>> kv;
    kv.reserve((size_t)npx * npy);
    for (int j = 0; j < npy; ++j)
        for (int i = 0; i < npx; ++i) kv.push_back({morton_key(i, j), j * npx + i});
    radix_sort_pairs(kv);
    root_.assign((size_t)npx * npy, -1);
    root_morton_.clear();
    for (const auto& e : kv) {
        root_[e.second] = alloc(0, e.second % npx, e.second / npx);
        root_morton_.push_back(root_[e.second]);
    }
    root_leaves_.assign((size_t)npx * npy, 1);
    n_leaves_ = (int64_t)npx * npy;
}

void PatchTree::recount_leaves() {
    std::fill(root_leaves_.begin(), root_leaves_.end(), 0);
    n_leaves_ = 0;
    for (int id = 0; id < capacity; ++id)
        if (alive[id] && child[4 * id] < 0) { ++root_leaves_[root_index(id)]; ++n_leaves_; }
}

void PatchTree::touch(int id) {
    if (!txn_ || touched_[id]) return;
    touched_[id] = 1;
    SlotSnap sn{id, lev[id], pi[id], pj[id], parent[id], {child[4 * id], child[4 * id + 1], child[4 * id + 2], child[4 * id + 3]},
                alive[id]};
    journal_.push_back(sn);
}

void PatchTree::begin_txn() {
    journal_.clear();
    released_parent_ = false;
    if ((int)touched_.size() != capacity) touched_.assign(capacity, 0);
    txn_ = true;
}

void PatchTree::commit() {
    for (const auto& sn : journal_) touched_[sn.id] = 0;
    txn_ = false;
}

void PatchTree::rollback() {
    for (const auto& sn : journal_)
        if (alive[sn.id]) { index_.erase(key(lev[sn.id], pi[sn.id], pj[sn.id])); --n_alive; }
    for (auto it = journal_.rbegin(); it != journal_.rend(); ++it) {
        const SlotSnap& sn = *it;
        lev[sn.id] = sn.lev; pi[sn.id] = sn.pi; pj[sn.id] = sn.pj; parent[sn.id] = sn.parent; alive[sn.id] = sn.alive;
        for (int c = 0; c < 4; ++c) child[4 * sn.id + c] = sn.child[c];
        sync(sn.id);
    }
    for (const auto& sn : journal_)
        if (sn.alive) { index_.set(key(sn.lev, sn.pi, sn.pj), sn.id); ++n_alive; }
    free_.clear();   // rare path: rebuild the free-slot heap
    for (int s = 0; s < capacity; ++s)
        if (!alive[s]) free_.push_back(s);
    std::make_heap(free_.begin(), free_.end(), std::greater<int32_t>());
    for (const auto& sn : journal_) touched_[sn.id] = 0;
    journal_.clear();
    txn_ = false;
    recount_leaves();   // rare path
}

int PatchTree::alloc(int l, int i, int j) {
    std::pop_heap(free_.begin(), free_.end(), std::greater<int32_t>());
    int id = free_.back();
    free_.pop_back();
    touch(id);
    lev[id] = l; pi[id] = i; pj[id] = j; parent[id] = -1; alive[id] = 1;
    for (int c = 0; c < 4; ++c) child[4 * id + c] = -1;
    sync(id);
    index_.set(key(l, i, j), id);
    ++n_alive;
    return id;
}

void PatchTree::release(int id) {
    touch(id);
    if (child[4 * id] >= 0) released_parent_ = true;
    index_.erase(key(lev[id], pi[id], pj[id]));
    alive[id] = 0; lev[id] = -1; parent[id] = -1;
    for (int c = 0; c < 4; ++c) child[4 * id + c] = -1;
    sync(id);
    free_.push_back(id);
    std::push_heap(free_.begin(), free_.end(), std::greater<int32_t>());
    --n_alive;
}

bool PatchTree::wrap(int l, int& i, int& j) const {
    int nx = npatch(0, l), ny = npatch(1, l);
    if (i < 0 || i >= nx) { if (!periodic[0]) return false; i = pmod(i, nx); }
    if (j < 0 || j >= ny) { if (!periodic[1]) return false; j = pmod(j, ny); }
    return true;
}

int PatchTree::find(int l, int i, int j) const {
    if (l < 0 || l >= levels || !wrap(l, i, j)) return -1;
    return index_.find(key(l, i, j));
}

int PatchTree::neighbour(int id, int dx, int dy) const {
    const Node& n = node_[id];
    if (n.lev == 0) {
        int i = n.pi + dx, j = n.pj + dy;
        if (!wrap(0, i, j)) return -2;
        return root_[(size_t)j * np0[0] + i];
    }
    int a = (n.pi & 1) + dx, b = (n.pj & 1) + dy;   // position relative to the parent's children, -1 .. 2
    if (a >= 0 && a <= 1 && b >= 0 && b <= 1) return node_[n.parent].child[a + 2 * b];   // a sibling
    const int DX = a < 0 ? -1 : (a > 1 ? 1 : 0), DY = b < 0 ? -1 : (b > 1 ? 1 : 0);
    const int pn = neighbour(n.parent, DX, DY);         // same-level neighbour of the parent (recursion by level)
    if (pn < 0) return pn;                              // outside the domain, or missing
    const Node& p = node_[pn];
    if (p.child[0] < 0) return -1;
    return p.child[(a - 2 * DX) + 2 * (b - 2 * DY)];
}

// Alg. 1 RefinePatch: before creating p's children make every
// Moore position of p active, refining the corresponding neighbour of p's
// parent (which exists by R2) recursively.
bool PatchTree::refine(int id, std::string& err) {
    if (has_children(id)) return true;
    int l = lev[id];
    if (l + 1 >= levels) { err = "refine beyond the finest level"; return false; }
    for (int d = 0; d < 8; ++d) {
        int q = neighbour(id, kMoore[d][0], kMoore[d][1]);
        if (q != -1) continue;          // exists, or outside the domain (ghost patch)
        int i = pi[id] + kMoore[d][0], j = pj[id] + kMoore[d][1];
        wrap(l, i, j);
        int r = find(l - 1, i >> 1, j >> 1);
        if (l == 0 || r < 0) { err = "R2 violated: no coarse support for refinement"; return false; }
        if (!refine(r, err)) return false;
    }
    if ((int)free_.size() < 4) { err = "slot capacity exceeded"; return false; }
    touch(id);
    root_leaves_[root_index(id)] += 3;
    n_leaves_ += 3;
    for (int c = 0; c < 4; ++c) {
        int a = c & 1, b = c >> 1;
        int k = alloc(l + 1, 2 * pi[id] + a, 2 * pj[id] + b);
        parent[k] = id;
        child[4 * id + c] = k;
        sync(k);
    }
    sync(id);
    return true;
}

// IsCoarseningAllowed (Alg. 2) -- rule 1 literal; rule 0 the prose
// condition of P:L259 (A16): children are leaves and none of them serves as a
// Moore neighbour of a level-(l+1) patch that has children.
bool PatchTree::coarsen_allowed(int id) const {
    if (!has_children(id)) return false;
    for (int c = 0; c < 4; ++c)
        if (has_children(child[4 * id + c])) return false;
    if (coarsen_rule == 1) {
        if (lev[id] == 0) return false;
        for (int d = 0; d < 8; ++d) {
            int q = neighbour(id, kMoore[d][0], kMoore[d][1]);
            if (q >= 0 && has_children(q)) return false;
        }
        return true;
    }
    // R2-exact rule: no Moore neighbour q of a child (same level, parent[q] != id) may have children.  Those q are the
    // 12 level-(l+1) cells around the 2 x 2 block: the children of id's 8 Moore neighbours that touch it, so they are
    // found from 8 neighbour() calls at level l instead of 20 at level l+1 (each of which recursed to level l anyway)
    for (int d = 0; d < 8; ++d) {
        const int DX = kMoore[d][0], DY = kMoore[d][1];
        const int pn = neighbour(id, DX, DY);
        if (pn < 0 || pn == id || node_[pn].child[0] < 0) continue;   // (pn == id: periodic self-wrap, q are siblings)
        const Node& p = node_[pn];
        for (int qb = 0; qb < 2; ++qb) {
            if ((DY == 1 && qb != 0) || (DY == -1 && qb != 1)) continue;   // the row of pn's children facing id
            for (int qa = 0; qa < 2; ++qa) {
                if ((DX == 1 && qa != 0) || (DX == -1 && qa != 1)) continue;
                if (has_children(p.child[qa + 2 * qb])) return false;
            }
        }
    }
    return true;
}

void PatchTree::delete_children(int id) {
    touch(id);
    if (child[4 * id] >= 0) {   // (coarsening: the 4 children are leaves)
        root_leaves_[root_index(id)] -= 3;
        n_leaves_ -= 3;
    }
    for (int c = 0; c < 4; ++c) {
        int k = child[4 * id + c];
        if (k >= 0) release(k);
        child[4 * id + c] = -1;
    }
    sync(id);
}

bool PatchTree::validate(std::string& err) const {
    for (int j = 0; j < np0[1]; ++j)
        for (int i = 0; i < np0[0]; ++i) {   // R1: the root table's slots are alive roots at their position
            const int r = root_[(size_t)j * np0[0] + i];
            if (r < 0 || !alive[r] || lev[r] != 0 || pi[r] != i || pj[r] != j) { err = "R1 violated: root missing"; return false; }
        }
    static thread_local std::vector<std::pair<uint64_t, int32_t>> kv;   // the active patches (O(active))
    index_.dump(kv);
    for (const auto& e : kv) {
        const int id = e.second;
        if (!alive[id]) { err = "index refers to a free slot"; return false; }
        if (lev[id] > 0) {
            int p = parent[id];
            if (p < 0 || !alive[p]) { err = "orphan patch"; return false; }
        }
        int nc = 0;
        for (int c = 0; c < 4; ++c) nc += child[4 * id + c] >= 0;
        if (nc != 0 && nc != 4) { err = "children not all-or-none"; return false; }
        if (nc == 4) {
            for (int d = 0; d < 8; ++d)
                if (neighbour(id, kMoore[d][0], kMoore[d][1]) == -1) { err = "R2 violated"; return false; }
        }
    }
    return true;
}

bool PatchTree::validate_txn(std::string& err) const {
    if (released_parent_) { err = "orphan patch"; return false; }
    auto r2 = [&](int id) {
        for (int d = 0; d < 8; ++d)
            if (neighbour(id, kMoore[d][0], kMoore[d][1]) == -1) return false;
        return true;
    };
    for (const SlotSnap& sn : journal_) {
        const int id = sn.id;
        if (sn.alive && sn.lev == 0 && !(alive[id] && lev[id] == 0 && pi[id] == sn.pi && pj[id] == sn.pj)) {
            err = "R1 violated: root missing";
            return false;
        }
        if (alive[id]) {   // a created or modified patch: the per-patch checks of validate()
            if (lev[id] > 0 && (parent[id] < 0 || !alive[parent[id]])) { err = "orphan patch"; return false; }
            int nc = 0;
            for (int c = 0; c < 4; ++c) nc += child[4 * id + c] >= 0;
            if (nc != 0 && nc != 4) { err = "children not all-or-none"; return false; }
            if (nc == 4 && !r2(id)) { err = "R2 violated"; return false; }
        }
        if (sn.alive && find(sn.lev, sn.pi, sn.pj) < 0) {   // a removed position: its refined Moore neighbours
            for (int d = 0; d < 8; ++d) {
                const int q = find(sn.lev, sn.pi + kMoore[d][0], sn.pj + kMoore[d][1]);
                if (q >= 0 && has_children(q)) { err = "R2 violated"; return false; }
            }
        }
    }
    return true;
}

std::vector<int32_t> PatchTree::canonical() const {
    std::vector<int32_t> ids;
    ids.reserve((size_t)n_alive);
    for (int j = 0; j < np0[1]; ++j)
        for (int i = 0; i < np0[0]; ++i) ids.push_back(root_[(size_t)j * np0[0] + i]);
    size_t b = 0, e = ids.size();   // [b, e): level l in (j, i) order
    while (b < e) {
        for (size_t r = b; r < e;) {   // one row J of level l: rows 2J (children 0, 1) and 2J + 1 (children 2, 3)
            size_t q = r;
            while (q < e && node_[ids[q]].pj == node_[ids[r]].pj) ++q;
            for (int half = 0; half < 2; ++half)
                for (size_t k = r; k < q; ++k) {
                    const Node& nd = node_[ids[k]];
                    if (nd.child[0] < 0) continue;
                    ids.push_back(nd.child[2 * half]);
                    ids.push_back(nd.child[2 * half + 1]);
                }
            r = q;
        }
        b = e;
        e = ids.size();
    }
    return ids;
}

void PatchTree::face_neighbours(const std::vector<int32_t>& canon, std::vector<int32_t>& nb4) const {
    if (nb4.size() != (size_t)4 * capacity) nb4.assign((size_t)4 * capacity, -1);
    static const int d[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};   // W, E, S, N
    auto one = [&](int id) {
        const Node& nd = node_[id];
        int32_t* o = &nb4[(size_t)4 * id];
        if (nd.lev == 0) {
            for (int s = 0; s < 4; ++s) {
                int i = nd.pi + d[s][0], j = nd.pj + d[s][1];
                o[s] = wrap(0, i, j) ? root_[(size_t)j * np0[0] + i] : -2;
            }
            return;
        }
        const Node& pa = node_[nd.parent];
        const int32_t* pn = &nb4[(size_t)4 * nd.parent];
        const int a = nd.pi & 1, b = nd.pj & 1;
        auto across = [&](int side, int cidx) {   // child cidx of the parent's neighbour on `side`, else -1 / -2
            const int q = pn[side];
            if (q < 0) return q;
            return node_[q].child[0] < 0 ? -1 : node_[q].child[cidx];
        };
        o[0] = a == 1 ? pa.child[0 + 2 * b] : across(0, 1 + 2 * b);
        o[1] = a == 0 ? pa.child[1 + 2 * b] : across(1, 0 + 2 * b);
        o[2] = b == 1 ? pa.child[a] : across(2, a + 2);
        o[3] = b == 0 ? pa.child[a + 2] : across(3, a);
    };
    for (int id : canon) one(id);   // level-major: a patch's parent is done before it
}

void PatchTree::face_neighbours_roots(const std::vector<int32_t>& roots, std::vector<int32_t>& nb4) const {
    if (nb4.size() != (size_t)4 * capacity) nb4.assign((size_t)4 * capacity, -1);
    face_neighbours_span(roots.data(), roots.size(), nb4, walk_);
}

void PatchTree::face_neighbours_span(const int32_t* roots, size_t nr, std::vector<int32_t>& nb4,
                                     std::vector<int32_t>& st) const {
    for (size_t k = 0; k < nr; ++k) {
        st.clear();
        st.push_back(root_[(size_t)roots[k]]);
        while (!st.empty()) {   // pre-order: a patch's parent is done before it
            const int id = st.back();
            st.pop_back();
            const Node& nd = node_[id];
            if (nd.child[0] >= 0)
                for (int q = 3; q >= 0; --q) st.push_back(nd.child[q]);
            face_neighbours_one(id, nb4);
        }
    }
}

void PatchTree::face_neighbours_one(int id, std::vector<int32_t>& nb4) const {
    static const int d[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};   // W, E, S, N
    const Node& nd = node_[id];
    int32_t* o = &nb4[(size_t)4 * id];
    if (nd.lev == 0) {
        for (int s = 0; s < 4; ++s) {
            int i = nd.pi + d[s][0], j = nd.pj + d[s][1];
            o[s] = wrap(0, i, j) ? root_[(size_t)j * np0[0] + i] : -2;
        }
        return;
    }
    const Node& pa = node_[nd.parent];
    const int32_t* pn = &nb4[(size_t)4 * nd.parent];
    const int a = nd.pi & 1, b = nd.pj & 1;
    auto across = [&](int side, int cidx) {
        const int q = pn[side];
        if (q < 0) return q;
        return node_[q].child[0] < 0 ? -1 : node_[q].child[cidx];
    };
    o[0] = a == 1 ? pa.child[0 + 2 * b] : across(0, 1 + 2 * b);
    o[1] = a == 0 ? pa.child[1 + 2 * b] : across(1, 0 + 2 * b);
    o[2] = b == 1 ? pa.child[a] : across(2, a + 2);
    o[3] = b == 0 ? pa.child[a + 2] : across(3, a);
}

std::vector<int32_t> PatchTree::canonical_sorted() const {
    static thread_local std::vector<std::pair<uint64_t, int32_t>> kv;   // key (level, j, i) = the map key
    index_.dump(kv);
    for (auto& e : kv) e.first = canon_key(e.first);
    radix_sort_pairs(kv);
    std::vector<int32_t> ids(kv.size());
    for (size_t e = 0; e < kv.size(); ++e) ids[e] = kv[e].second;
    return ids;
}

}  // namespace amr
