// tree.h -- host-side quadtree of patches (PAPER.md s3.2-3.3, Fig. 2).
//
// Flat structure-of-arrays indexed by patch id (= device slot), a hash map from
// (level, i, j) to id, and lowest-free-first slot recycling.  Enforces R1
// and R2 through Alg. 1 (recursive refinement)
// and the coarsening pass of Alg. 2 / its prose condition.
// Independent of oracle/ (no shared code).
#pragma once
#include <algorithm>
#include <cstdint>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

namespace amr {

// Open-addressing hash map uint64 key -> int32 id (linear probing, backward-shift deletion): the patch index of the
// tree.  Keys are never ~0ull (the empty marker); the table stays at most half full.
class FlatIndex {
  public:
    void clear() { keys_.assign(keys_.size(), kEmpty); size_ = 0; }
    void reserve(size_t n) {
        size_t cap = 16;
        while (cap < 2 * n) cap <<= 1;
        if (cap > keys_.size()) rehash(cap);
    }
    int32_t find(uint64_t k) const {
        if (keys_.empty()) return -1;
        for (size_t i = hash(k) & mask(); ; i = (i + 1) & mask()) {
            if (keys_[i] == k) return vals_[i];
            if (keys_[i] == kEmpty) return -1;
        }
    }
    void set(uint64_t k, int32_t v) {
        if (2 * (size_ + 1) > keys_.size()) rehash(keys_.empty() ? 16 : 2 * keys_.size());
        size_t i = hash(k) & mask();
        while (keys_[i] != kEmpty && keys_[i] != k) i = (i + 1) & mask();
        if (keys_[i] == kEmpty) ++size_;
        keys_[i] = k;
        vals_[i] = v;
    }
    void erase(uint64_t k) {
        if (keys_.empty()) return;
        size_t i = hash(k) & mask();
        while (keys_[i] != k) {
            if (keys_[i] == kEmpty) return;
            i = (i + 1) & mask();
        }
        // backward-shift deletion keeps every probe chain contiguous
        size_t j = i;
        for (;;) {
            j = (j + 1) & mask();
            if (keys_[j] == kEmpty) break;
            const size_t h = hash(keys_[j]) & mask();
            const bool move = (j > i) ? (h <= i || h > j) : (h <= i && h > j);
            if (move) { keys_[i] = keys_[j]; vals_[i] = vals_[j]; i = j; }
        }
        keys_[i] = kEmpty;
        --size_;
    }
    size_t size() const { return size_; }
    template <class F>
    void for_each(F f) const {
        for (size_t i = 0; i < keys_.size(); ++i)
            if (keys_[i] != kEmpty) f(keys_[i], vals_[i]);
    }
    // every (key, id) entry into out, in table order; branch-free (a half-full table defeats the branch predictor)
    void dump(std::vector<std::pair<uint64_t, int32_t>>& out) const {
        out.resize(size_ + 1);
        size_t n = 0;
        for (size_t i = 0; i < keys_.size(); ++i) {
            out[n] = {keys_[i], vals_[i]};
            n += keys_[i] != kEmpty;
        }
        out.resize(n);
    }

  private:
    static constexpr uint64_t kEmpty = ~0ull;
    std::vector<uint64_t> keys_;
    std::vector<int32_t> vals_;
    size_t size_ = 0;
    size_t mask() const { return keys_.size() - 1; }
    static size_t hash(uint64_t k) { k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; return (size_t)k; }
    void rehash(size_t cap) {
        std::vector<uint64_t> ok;
        std::vector<int32_t> ov;
        ok.swap(keys_);
        ov.swap(vals_);
        keys_.assign(cap, kEmpty);
        vals_.assign(cap, -1);
        size_ = 0;
        for (size_t i = 0; i < ok.size(); ++i)
            if (ok[i] != kEmpty) set(ok[i], ov[i]);
    }
};

// LSD radix sort of (key, id) pairs by key.  Only the bit span in which the keys differ is sorted, in the fewest
// passes of digits of at most 8 bits (under 2 k pairs), 12 bits (under 64 k) or 16 bits, split evenly (a compact
// 22-bit patch key takes two passes).  Keys are unique in every use (patch keys, level-Morton keys), so the order
// is the plain key order.
inline uint64_t spread_bits(uint32_t v) {
    uint64_t x = v;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}
inline uint64_t morton(uint32_t x, uint32_t y) { return spread_bits(x) | (spread_bits(y) << 1); }

inline void radix_sort_pairs(std::vector<std::pair<uint64_t, int32_t>>& v) {
    if (v.size() < 2) return;
    uint64_t diff = 0;   // bits in which some key differs from the first: only that span needs passes
    for (const auto& e : v) diff |= e.first ^ v[0].first;
    if (!diff) return;
    const int lo = __builtin_ctzll(diff), span = 64 - __builtin_clzll(diff) - lo;
    const int maxb = v.size() < 2048 ? 8 : (v.size() < 65536 ? 12 : 16);
    const int passes = (span + maxb - 1) / maxb, bits = (span + passes - 1) / passes;
    const uint64_t mask = (1ull << bits) - 1;
    // scratch kept across calls (per thread): a fresh 100 KB+ buffer is an mmap plus page faults on every regrid
    static thread_local std::vector<std::pair<uint64_t, int32_t>> tmp;
    static thread_local std::vector<uint32_t> cnt;
    tmp.resize(v.size());
    cnt.resize(size_t(1) << bits);
    for (int p = 0, shift = lo; p < passes; ++p, shift += bits) {
        std::fill(cnt.begin(), cnt.end(), 0u);
        for (const auto& e : v) ++cnt[(e.first >> shift) & mask];
        uint32_t sum = 0;
        for (auto& c : cnt) { const uint32_t x = c; c = sum; sum += x; }
        for (const auto& e : v) tmp[cnt[(e.first >> shift) & mask]++] = e;
        v.swap(tmp);
    }
}

struct PatchTree {
    // geometry
    int np0[2] = {0, 0};     // level-0 patches per axis
    int levels = 1;
    bool periodic[2] = {false, false};
    int capacity = 0;
    int coarsen_rule = 0;    // 0 R2-exact, 1 Alg. 2 literal

    // per slot
    std::vector<int32_t> lev, pi, pj, parent;
    std::vector<int32_t> child;      // 4 per slot, -1 if none
    std::vector<uint8_t> alive;
    int n_alive = 0;

    void init(int npx, int npy, int nlev, bool perx, bool pery, int cap, int rule);
    static uint64_t key(int l, int i, int j) {
        return (uint64_t(uint32_t(l)) << 56) | (uint64_t(uint32_t(j)) << 28) | uint64_t(uint32_t(i));
    }
    // bits of a finest-level patch coordinate per axis: (level, j, i) and (level, Morton(i, j)) packed above
    // kb[0] + kb[1] (resp. 2 max(kb)) bits sort in few radix passes
    int kb[2] = {0, 0};
    uint64_t canon_key(uint64_t k) const {   // key(l, i, j) -> same order, compact
        return ((k >> 56) << (kb[0] + kb[1])) | (((k >> 28) & 0xFFFFFFFull) << kb[0]) | (k & 0xFFFFFFFull);
    }
    int morton_shift() const { return 2 * std::max(kb[0], kb[1]); }   // level above a Morton key of (i, j)
    int npatch(int ax, int l) const { return np0[ax] << l; }
    // wrap a level-l patch position; false when outside a non-periodic boundary
    bool wrap(int l, int& i, int& j) const;
    int find(int l, int i, int j) const;          // id or -1 (position wrapped first)
    // id, -1 missing, -2 outside domain (|dx|, |dy| <= 1): by the parent/child links -- a sibling, else the child of
    // the parent's neighbour (roots from a table) -- with no hash probe
    int neighbour(int id, int dx, int dy) const;
    bool has_children(int id) const { return node_[id].child[0] >= 0; }
    // root (row-major index) of the tree holding slot id
    int root_index(int id) const { const Node& nd = node_[id]; return (nd.pj >> nd.lev) * np0[0] + (nd.pi >> nd.lev); }
    int root_slot(int r) const { return root_[(size_t)r]; }
    int nroots() const { return np0[0] * np0[1]; }
    const std::vector<int32_t>& root_morton() const { return root_morton_; }   // root slots in Morton order
    // leaves per root (row-major), maintained by refine / delete_children (+3 / -3), recomputed by rollback
    const std::vector<int32_t>& root_leaves() const { return root_leaves_; }
    int64_t n_leaves() const { return n_leaves_; }
    // pre-order walk of the subtree of a slot (parents before children), f(id)
    template <class F>
    void subtree(int top, F f) const {
        std::vector<int32_t>& st = walk_;
        st.clear();
        st.push_back(top);
        while (!st.empty()) {
            const int id = st.back();
            st.pop_back();
            f(id);
            const Node& nd = node_[id];
            if (nd.child[0] >= 0)
                for (int q = 3; q >= 0; --q) st.push_back(nd.child[q]);
        }
    }
    bool is_leaf(int id) const { return node_[id].lev >= 0 && node_[id].child[0] < 0; }   // alive <=> lev >= 0

    // Alg. 1 on a copy-on-write basis; returns false (tree unchanged by caller's
    // transaction) on capacity overflow.
    bool refine(int id, std::string& err);
    bool coarsen_allowed(int id) const;
    void delete_children(int id);
    bool validate(std::string& err) const;
    // The same checks restricted to what the open transaction changed (journaled slots, the Moore neighbours of
    // removed positions, released slots with children): equal to validate() when the tree was valid at
    // begin_txn(), in O(changes).
    bool validate_txn(std::string& err) const;
    // ids of active patches in canonical order (level, j, i): generated level by level from the parent rows (a
    // level-(l+1) row 2J / 2J+1 is the SW,SE / NW,NE children of level-l row J, left to right), O(active)
    std::vector<int32_t> canonical() const;
    // the same order by sorting the packed keys of the index (the definition; the planning API checks the two agree)
    std::vector<int32_t> canonical_sorted() const;
    // leaves per level in Morton order of their position (depth-first from the roots in Morton order, children in
    // Morton order a + 2b): the launch order of build_plan without a sort; keep(id) filters (ownership)
    template <class Keep>
    void leaves_morton(std::vector<std::vector<int32_t>>& per_level, Keep keep) const {
        leaves_morton_roots(per_level, keep, [](int) { return true; });
    }
    // the same walk over the roots with root_ok(root slot) only (a rank's own roots: O(local))
    template <class Keep, class RootOk>
    void leaves_morton_roots(std::vector<std::vector<int32_t>>& per_level, Keep keep, RootOk root_ok) const {
        leaves_morton_span(0, root_morton_.size(), per_level, keep, root_ok, dfs_);
    }
    // the same walk over the roots root_morton()[r0, r1) with a caller-owned stack (parts of a parallel plan)
    template <class Keep, class RootOk>
    void leaves_morton_span(size_t r0, size_t r1, std::vector<std::vector<int32_t>>& per_level, Keep keep,
                            RootOk root_ok, std::vector<int32_t>& st) const {
        per_level.resize(levels);
        for (auto& v : per_level) v.clear();
        st.clear();
        for (size_t r = r1; r-- > r0;)
            if (root_ok(root_morton_[r])) st.push_back(root_morton_[r]);
        while (!st.empty()) {
            const int id = st.back();
            st.pop_back();
            const Node& nd = node_[id];
            if (nd.child[0] < 0) {
                if (keep(id)) per_level[nd.lev].push_back(id);
            } else {
                for (int q = 3; q >= 0; --q) st.push_back(nd.child[q]);
            }
        }
    }
    // face neighbours W, E, S, N of every active patch (nb4[4 id + s]: id, -1 missing, -2 outside the domain), top
    // down over `canon` (level-major) from the parents' entries: equal to neighbour(id, +-1 / 0) without recursion
    void face_neighbours(const std::vector<int32_t>& canon, std::vector<int32_t>& nb4) const;
    // the same table for the subtrees of the given roots only (row-major root indices; each subtree pre-order, a patch
    // needs only its parent's entries); nb4 is sized once to the capacity
    void face_neighbours_roots(const std::vector<int32_t>& roots, std::vector<int32_t>& nb4) const;
    // the same for roots[0, nr) with a caller-owned stack, into an nb4 already sized to 4 x capacity (parts of a
    // parallel plan: a patch's entries depend only on its parent's, so root subtrees are independent)
    void face_neighbours_span(const int32_t* roots, size_t nr, std::vector<int32_t>& nb4, std::vector<int32_t>& st) const;
    // the entries of one patch from its parent's (level 0: the root table); nb4 sized to 4 x capacity
    void face_neighbours_one(int id, std::vector<int32_t>& nb4) const;

    // Transactions (regrid is atomic): between begin_txn() and commit()/rollback() every modified slot
    // is journaled once with its prior state, so a failed regrid is undone in O(changes) -- no copy of the
    // capacity-sized arrays -- and the journal tells which slots were created or deleted.
    struct SlotSnap {
        int32_t id, lev, pi, pj, parent, child[4];
        uint8_t alive;
    };
    void begin_txn();
    void commit();
    void rollback();
    const std::vector<SlotSnap>& journal() const { return journal_; }

  private:
    std::vector<SlotSnap> journal_;
    std::vector<uint8_t> touched_;
    bool txn_ = false;
    bool released_parent_ = false;   // a slot with children was released inside the transaction (orphans)
    void touch(int id);
    FlatIndex index_;
    // packed copy of (lev, pi, pj, parent, child[4]) per slot, for neighbour(): one 32-byte line per node visited
    // instead of five arrays (1.8x faster lookups); written only by sync(), after every change of a slot
    struct Node {
        int32_t lev, pi, pj, parent, child[4];
    };
    std::vector<Node> node_;
    void sync(int id) {
        node_[id] = Node{lev[id], pi[id], pj[id], parent[id], {child[4 * id], child[4 * id + 1], child[4 * id + 2], child[4 * id + 3]}};
    }
    std::vector<int32_t> root_;   // root (i, j) -> slot, row-major (R1: roots are permanent)
    std::vector<int32_t> root_morton_;   // root slots in Morton order of (i, j)
    mutable std::vector<int32_t> dfs_;   // leaves_morton's stack
    mutable std::vector<int32_t> walk_;  // subtree()'s stack
    std::vector<int32_t> root_leaves_;   // leaves per root (row-major)
    int64_t n_leaves_ = 0;
    void recount_leaves();
    std::vector<int32_t> free_;   // min-heap of free slots
    int alloc(int l, int i, int j);
    void release(int id);
};

}  // namespace amr
