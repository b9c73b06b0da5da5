// comm.h -- multi-GPU plumbing of one node.
//
// Every rank holds the same (replicated) patch tree and the same global slot numbering.  Patches
// are owned by root tree: roots in Morton order, weighted by their leaf count, are cut into
// world_size contiguous chunks, and every patch belongs to the owner of its root, so restriction
// is always local.  Each rank advances its own leaves; the data its kernels read from patches
// owned elsewhere (same-level face neighbours, the coarse 3x3 neighbourhood of C/F ghost strips,
// fine flux registers of a C/F face, the coarse sources of new patches) is copied into the same
// global slots of the local pool by grouped point-to-point exchanges; Lambda is a max-allreduce.
// Transports: NCCL (one process per GPU, torch's libnccl.so.2 loaded with dlopen) or an
// in-process loopback (virtual ranks as host threads on one GPU; test-only).
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <vector>

#include "../../include/amr.h"
#include "tree.h"

struct amr_ctx;

namespace amr {

// per-peer slot lists (sorted); send[r]: my slots that rank r needs; recv[r]: slots owned by r I need.
// items = true: the entries are BAND ITEMS, slot * 32 + code -- the g-wide strips a halo reader needs instead of whole
// patches: code < 16 the row band 4 code .. 4 code + 3 (code 0 = the S strip, n/4 - 1 = the N
// strip), 16 the W strip (columns 0..3), 17 the E strip (columns n-4..n-1); a whole patch is its n/4 row bands
constexpr int kBandW = 16, kBandE = 17;
struct ExchangeLists {
    std::vector<std::vector<int32_t>> send, recv;
    bool items = false;
    void reset(int world) { send.assign(world, {}); recv.assign(world, {}); }
    size_t nsend() const { size_t s = 0; for (auto& v : send) s += v.size(); return s; }
    size_t nrecv() const { size_t s = 0; for (auto& v : recv) s += v.size(); return s; }
};

// ---- pure host planning (no CUDA): testable on CPU
// Ownership by root tree: owner(id) = root_rank[root of id] -- O(1) per query, O(roots) per repartition (no
// capacity-sized array); the tree must outlive the object
struct Owners {
    const PatchTree* t = nullptr;
    int world = 1;
    std::vector<int32_t> root_rank;   // per root, row-major
    int operator[](int id) const { return world == 1 ? 0 : root_rank[(size_t)t->root_index(id)]; }
    // roots whose subtrees can hold leaves that read from, or are read by, `rank` across a partition boundary: the
    // roots of `rank` with a Moore-neighbour root of another rank, and the other ranks' roots Moore-adjacent to one of
    // `rank` (a patch reads only its own root and the 8 around it: face neighbours, parent's 3 x 3 neighbourhood)
    const std::vector<int32_t>& boundary_roots(int rank) const;   // (cached per rank until the partition changes)
    std::vector<int32_t> roots_of(int rank) const;   // row-major indices of rank's roots

  private:
    mutable int bnd_rank_ = -1;
    mutable std::vector<int32_t> bnd_;
};
Owners partition_owners(const PatchTree& t, int world);
// band items read by the stage / flags / ghost kernels of leaf `id` that may live on another rank (patch size n): of a
// face neighbour the strip facing id, of a coarse source of a C/F ghost strip (the parent's 3 x 3 neighbourhood) the
// whole patch (faces = false: only the coarse sources -- halo_mode 2 reads face strips in the stage kernel)
void halo_sources(const PatchTree& t, int id, int n, std::vector<int32_t>& out, bool faces = true);
// the per-rank lists are built from the leaves of owner.boundary_roots(rank) only: O(partition boundary)
ExchangeLists plan_halo(const PatchTree& t, const Owners& owner, int world, int rank, int n, bool faces = true);
ExchangeLists plan_flux(const PatchTree& t, const Owners& owner, int world, int rank);
// coarse sources of new level-l patches prolonged by the (old) owner of their root
ExchangeLists plan_coarse(const PatchTree& nt, const std::vector<int32_t>& new_ids, int level, const Owners& owner,
                          int world, int rank);
// subcycling (NEXT #4) across ranks, per level l: the remote slots a level-l stage reads (same-level face
// neighbours of every advanced level-l patch, leaves and covered ones), the remote coarse sources of the level's
// C/F ghosts (read at two times: the coarse step's start and end buffers), and the remote fine leaves whose
// accumulated registers the level-l reflux reads
struct SubLists {
    std::vector<ExchangeLists> face, coarse, facc;
};
SubLists plan_subcycle(const PatchTree& t, const Owners& owner, int world, int rank, int n);
// patches of the roots whose owner changed (O(changed subtrees))
ExchangeLists plan_migration(const PatchTree& nt, const Owners& old_owner, const Owners& new_owner, int world, int rank);

struct Transport;

struct Comm {
    int world = 1, rank = 0;
    int n = 0;                         // patch size (band items)
    std::unique_ptr<Transport> tr;
    Owners owner;                      // root-tree ownership of every active patch
    ExchangeLists halo, flux, halo_cf;
    bool subcycle = false;
    SubLists sub;                      // subcycle: per-level lists (plan_subcycle)
    uint64_t lists_version = 0;        // bumped by replan
    int64_t bytes_sent = 0;

    // halo_mode 1 (NEXT #3): every rank's state pool and flux-register buffer mapped into this process; halo and
    // flux exchanges become a stream-ordered cross-rank fence plus one peer_pull_kernel launch
    int halo_mode = 0;
    void* pool_base = nullptr;               // local pool (the 3 RK buffers)
    const void* mapped_freg = nullptr;       // local flux-register buffer the peer table was built for
    double** d_pool_bases = nullptr;         // device [world]: every rank's pool base as seen here
    double** d_freg_bases = nullptr;
    std::vector<double*> peer_pool;          // host copy of the peer pool bases (halo_mode 2 tensor maps)
    struct PullList {
        uint64_t version = ~0ull;
        int n = 0;
        int32_t* slots = nullptr;            // device
        int32_t* peers = nullptr;
    } pull_halo, pull_flux, pull_halo_cf;

    Comm();
    ~Comm();
    amr_status init(amr_ctx* c);
    void finalize(amr_ctx* c);
    bool owns(const amr_ctx*, int id) const { return world == 1 || owner[id] == rank; }
    int owner_of(const amr_ctx*, int id) const { return world == 1 ? 0 : owner[id]; }
    void repartition(const PatchTree& t);      // owner <- partition_owners(t)
    void replan(const PatchTree& t);           // halo / flux lists for the current owner

    amr_status exchange_halos(amr_ctx* c, double* U);
    // before a stage kernel: halo_mode 2 pulls only the C/F coarse sources (face strips are read in the kernel)
    amr_status exchange_halos_stage(amr_ctx* c, double* U);
    amr_status exchange_fluxes(amr_ctx* c);
    // persistent = true: L lives until the next replan, so its index lists stay on the device (keyed by &L)
    amr_status exchange_lists(amr_ctx* c, const ExchangeLists& L, double* U, int per_slot, const char* what,
                              bool persistent = false);
    struct DevLists {
        uint64_t version = ~0ull;
        int32_t *send = nullptr, *recv = nullptr;
        size_t ns = 0, nr = 0;
    };
    std::map<const ExchangeLists*, DevLists> dev_lists;   // per-plan index lists on the device (freed at replan)
    void free_dev_lists();
    amr_status exchange_children(amr_ctx*, double*) { return AMR_OK; }   // root-tree ownership: local
    amr_status map_pool(amr_ctx* c, void* base, size_t bytes);   // collective (amr_create)
    amr_status peer_pull(amr_ctx* c, const ExchangeLists& L, PullList& P, double* dst, bool freg, const char* what);
    amr_status allreduce_max_u64(amr_ctx* c, unsigned long long* d);
    amr_status allreduce_max_i32(amr_ctx* c, int32_t* d, int n);
    amr_status allreduce_sum4(amr_ctx* c, double* h4);
    amr_status allgather_flags(amr_ctx* c, std::vector<double>& eta, std::vector<uint8_t>& amb);
    // regrid requests: every rank's compact (slot, bits) list appended to `lst` on every rank (p2p; O(requests))
    amr_status allgather_requests(amr_ctx* c, std::vector<int32_t>& lst);
    amr_status agree_error(amr_ctx* c, int32_t* h_err4);
};

// NCCL symmetric-window memory (peer_map 1): ncclMemAlloc / ncclMemFree through the dlopen'ed library (nullptr and
// a message when NCCL or the symbol is unavailable)
void* comm_nccl_mem_alloc(size_t bytes, std::string& err);
void comm_nccl_mem_free(void* p);

}  // namespace amr
