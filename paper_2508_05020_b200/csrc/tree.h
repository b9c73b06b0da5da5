// tree.h -- host-side quadtree of patches (PAPER.md s3.2-3.3, Fig. 2).
//
// Flat structure-of-arrays indexed by patch id (= device slot), a hash map from
// (level, i, j) to id, and lowest-free-first slot recycling.  Enforces R1
// and R2 through Alg. 1 (recursive refinement)
// and the coarsening pass of Alg. 2 / its prose condition.
// Independent of oracle/ (no shared code).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

namespace amr {

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
    int npatch(int ax, int l) const { return np0[ax] << l; }
    // wrap a level-l patch position; false when outside a non-periodic boundary
    bool wrap(int l, int& i, int& j) const;
    int find(int l, int i, int j) const;          // id or -1 (position wrapped first)
    int neighbour(int id, int dx, int dy) const;  // id, -1 missing, -2 outside domain
    bool has_children(int id) const { return child[4 * id] >= 0; }
    bool is_leaf(int id) const { return alive[id] && child[4 * id] < 0; }

    // Alg. 1 on a copy-on-write basis; returns false (tree unchanged by caller's
    // transaction) on capacity overflow.
    bool refine(int id, std::string& err);
    bool coarsen_allowed(int id) const;
    void delete_children(int id);
    bool validate(std::string& err) const;
    // ids of active patches in canonical order (level, j, i)
    std::vector<int32_t> canonical() const;

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
    void touch(int id);
    std::unordered_map<uint64_t, int32_t> index_;
    std::vector<int32_t> free_;   // min-heap of free slots
    int alloc(int l, int i, int j);
    void release(int id);
};

}  // namespace amr
