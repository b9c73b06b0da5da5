// comm.cpp -- see comm.h.  Host planning (pure functions), the NCCL and loopback transports, and
// the exchange / collective hooks called by the step driver (api.cpp).
#include "comm.h"

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>

#include "ctx.h"

#ifdef AMR_HAVE_NCCL_H
#include <nccl.h>
#include <nccl_device.h>   // ncclDevComm / ncclDevCommRequirements (the LSA-barrier fence of peer_map 1)
#endif

namespace amr {

// =====================================================================================  planning
namespace {
const int kSideDir[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};   // W, E, S, N

ExchangeLists from_needs(const std::vector<std::map<int, std::set<int32_t>>>& need, int world, int rank) {
    // need[o][p] = slots owned by p that rank o needs
    ExchangeLists L;
    L.reset(world);
    for (int p = 0; p < world; ++p) {
        auto it = need[rank].find(p);
        if (it != need[rank].end()) L.recv[p].assign(it->second.begin(), it->second.end());
    }
    for (int o = 0; o < world; ++o) {
        auto it = need[o].find(rank);
        if (it != need[o].end()) L.send[o].assign(it->second.begin(), it->second.end());
    }
    return L;
}
}  // namespace

Owners partition_owners(const PatchTree& t, int world) {
    Owners o;
    o.t = &t;
    o.world = world;
    const int nr = t.nroots();
    o.root_rank.assign((size_t)nr, 0);
    if (world <= 1) return o;
    // roots in Morton order, weighted by their (incrementally maintained) leaf counts, cut into world chunks
    const std::vector<int32_t>& w = t.root_leaves();
    int64_t total = 0;
    for (int r = 0; r < nr; ++r) total += w[(size_t)r];
    int64_t prefix = 0;
    for (int slot : t.root_morton()) {
        const int r = t.root_index(slot);
        const int64_t wr = w[(size_t)r];
        const int64_t k = ((2 * prefix + wr) * (int64_t)world) / (2 * std::max<int64_t>(total, 1));
        o.root_rank[(size_t)r] = (int32_t)std::min<int64_t>(k, world - 1);
        prefix += wr;
    }
    return o;
}

std::vector<int32_t> Owners::roots_of(int rank) const {
    std::vector<int32_t> out;
    for (size_t r = 0; r < root_rank.size(); ++r)
        if (world == 1 || root_rank[r] == rank) out.push_back((int32_t)r);
    return out;
}

const std::vector<int32_t>& Owners::boundary_roots(int rank) const {
    if (bnd_rank_ == rank) return bnd_;
    bnd_.clear();
    bnd_rank_ = rank;
    if (world <= 1) return bnd_;
    // from this rank's roots and their 8 neighbours only: O(local roots)
    const int npx = t->np0[0], npy = t->np0[1];
    std::vector<uint8_t> mark;   // (sparse set over the roots touched)
    std::vector<int32_t> cand;
    for (int J = 0; J < npy; ++J)
        for (int I = 0; I < npx; ++I) {
            if (root_rank[(size_t)J * npx + I] != rank) continue;
            bool edge = false;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int i = I + dx, j = J + dy;
                    if (!t->wrap(0, i, j)) continue;
                    if (root_rank[(size_t)j * npx + i] != rank) { edge = true; cand.push_back(j * npx + i); }
                }
            if (edge) cand.push_back(J * npx + I);
        }
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    bnd_.swap(cand);
    return bnd_;
}

void halo_sources(const PatchTree& t, int id, int n, std::vector<int32_t>& out, bool faces) {
    out.clear();
    const int nb4 = n / 4;
    auto whole = [&](int q) { for (int b = 0; b < nb4; ++b) out.push_back(q * 32 + b); };
    // of the neighbour on side s (W, E, S, N of id) the strip facing id: its E columns, W columns, N rows, S rows
    const int facing[4] = {kBandE, kBandW, nb4 - 1, 0};
    for (int s = 0; s < 4; ++s) {
        int nb = t.neighbour(id, kSideDir[s][0], kSideDir[s][1]);
        if (nb >= 0) {
            if (faces) out.push_back(nb * 32 + facing[s]);
        } else if (nb == -1) {
            int par = t.parent[id];
            if (par < 0) continue;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int q = (dx == 0 && dy == 0) ? par : t.neighbour(par, dx, dy);
                    if (q >= 0) whole(q);
                }
        }
    }
}

namespace {
// f(id) for every active patch (leaves_only: every leaf) in the subtrees of `rank`'s boundary roots
template <class F>
void for_boundary(const PatchTree& t, const Owners& owner, int rank, bool leaves_only, F f) {
    for (int r : owner.boundary_roots(rank))
        t.subtree(t.root_slot(r), [&](int id) {
            if (!leaves_only || t.is_leaf(id)) f(id);
        });
}
}  // namespace

ExchangeLists plan_halo(const PatchTree& t, const Owners& owner, int world, int rank, int n, bool faces) {
    std::vector<std::map<int, std::set<int32_t>>> need(world);
    std::vector<int32_t> src;
    for_boundary(t, owner, rank, true, [&](int id) {
        const int o = owner[id];
        halo_sources(t, id, n, src, faces);
        for (int q : src) {
            const int oq = owner[q >> 5];
            if (oq != o && (o == rank || oq == rank)) need[o][oq].insert(q);
        }
    });
    ExchangeLists L = from_needs(need, world, rank);
    L.items = true;
    return L;
}

ExchangeLists plan_flux(const PatchTree& t, const Owners& owner, int world, int rank) {
    static const int cidx[4][2] = {{1, 3}, {0, 2}, {2, 3}, {0, 1}};
    std::vector<std::map<int, std::set<int32_t>>> need(world);
    for_boundary(t, owner, rank, true, [&](int id) {
        const int o = owner[id];
        for (int s = 0; s < 4; ++s) {
            int nb = t.neighbour(id, kSideDir[s][0], kSideDir[s][1]);
            if (nb < 0 || !t.has_children(nb)) continue;
            for (int h = 0; h < 2; ++h) {
                const int f = t.child[4 * nb + cidx[s][h]];
                const int of = owner[f];
                if (of != o && (o == rank || of == rank)) need[o][of].insert(f);
            }
        }
    });
    return from_needs(need, world, rank);
}

ExchangeLists plan_coarse(const PatchTree& nt, const std::vector<int32_t>& new_ids, int level, const Owners& owner,
                          int world, int rank) {
    std::vector<std::map<int, std::set<int32_t>>> need(world);
    for (int id : new_ids) {
        if (!nt.alive[id] || nt.lev[id] != level) continue;
        int o = owner[id], par = nt.parent[id];
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int q = (dx == 0 && dy == 0) ? par : nt.neighbour(par, dx, dy);
                if (q >= 0 && owner[q] != o && (o == rank || owner[q] == rank)) need[o][owner[q]].insert(q);
            }
    }
    return from_needs(need, world, rank);
}

SubLists plan_subcycle(const PatchTree& t, const Owners& owner, int world, int rank, int n) {
    static const int cidx[4][2] = {{1, 3}, {0, 2}, {2, 3}, {0, 1}};   // children of a W/E/S/N neighbour on the face
    const int L = t.levels;
    std::vector<std::vector<std::map<int, std::set<int32_t>>>> face(L), coarse(L), facc(L);
    for (int l = 0; l < L; ++l) {
        face[l].resize(world);
        coarse[l].resize(world);
        facc[l].resize(world);
    }
    auto keep = [&](int o, int q) { return q != o && (o == rank || q == rank); };
    for_boundary(t, owner, rank, false, [&](int id) {   // every active patch is advanced (leaves and covered ones)
        const int l = t.lev[id], o = owner[id];
        const bool leaf = t.is_leaf(id);
        for (int s = 0; s < 4; ++s) {
            const int nb = t.neighbour(id, kSideDir[s][0], kSideDir[s][1]);
            if (nb >= 0) {
                // the strip of nb facing id (band item, as plan_halo)
                const int facing[4] = {kBandE, kBandW, n / 4 - 1, 0};
                if (keep(o, owner[nb])) face[l][o][owner[nb]].insert(nb * 32 + facing[s]);
                if (leaf && t.has_children(nb))
                    for (int h = 0; h < 2; ++h) {
                        const int f = t.child[4 * nb + cidx[s][h]];
                        if (f >= 0 && keep(o, owner[f])) facc[l][o][owner[f]].insert(f);
                    }
            } else if (nb == -1 && leaf) {
                const int par = t.parent[id];
                if (par < 0) continue;
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int q = (dx == 0 && dy == 0) ? par : t.neighbour(par, dx, dy);
                        if (q >= 0 && keep(o, owner[q])) coarse[l][o][owner[q]].insert(q);
                    }
            }
        }
    });
    SubLists out;
    for (int l = 0; l < L; ++l) {
        out.face.push_back(from_needs(face[l], world, rank));
        out.face.back().items = true;
        out.coarse.push_back(from_needs(coarse[l], world, rank));
        out.facc.push_back(from_needs(facc[l], world, rank));
    }
    return out;
}

ExchangeLists plan_migration(const PatchTree& nt, const Owners& old_owner, const Owners& new_owner, int world,
                             int rank) {
    std::vector<std::map<int, std::set<int32_t>>> need(world);
    for (int r = 0; r < nt.nroots(); ++r) {
        const int a = old_owner.root_rank[(size_t)r], b = new_owner.root_rank[(size_t)r];
        if (a == b || (a != rank && b != rank)) continue;
        nt.subtree(nt.root_slot(r), [&](int id) { need[b][a].insert(id); });
    }
    return from_needs(need, world, rank);
}

// Host <-> device copies ordered on the library stream s and completed on return.  A plain cudaMemcpy runs on the
// legacy default stream, which does not order against the (non-blocking) library stream, and an H2D copy from
// pageable memory may still be in flight when it returns: a later kernel on s could read the old bytes.
inline cudaError_t h2d_sync(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    return e != cudaSuccess ? e : cudaStreamSynchronize(s);
}
inline cudaError_t d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
    return e != cudaSuccess ? e : cudaStreamSynchronize(s);
}

// =====================================================================================  transports
struct Xfer {
    int peer;
    void* buf;
    size_t bytes;
};

struct Transport {
    virtual ~Transport() {}
    virtual std::string p2p(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) = 0;
    // in-place allreduce on a device buffer; kind 0: max u64, 1: max f64, 2: sum f64, 3: max i32
    virtual std::string allreduce(void* d, size_t count, int kind, cudaStream_t s) = 0;
    // halo_mode 1: map every rank's device buffer [base, base + bytes) into this process (out[rank] = base)
    // tag: 0 the state pool, 1 the flux registers -- a re-map of a tag first closes that tag's previous mappings
    virtual std::string map_peers(void* base, size_t bytes, std::vector<void*>& out, cudaStream_t s, int tag = 0) = 0;
    // stream-ordered cross-rank fence: work queued after it on s runs after every rank's work queued before it
    virtual std::string fence(cudaStream_t s) = 0;
};

// ---- NCCL (torch's libnccl.so.2, resolved at run time)
#ifdef AMR_HAVE_NCCL_H
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    // symmetric memory windows (NCCL >= 2.27; optional: only peer_map 1 needs them)
    ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
    ncclResult_t (*MemFree)(void*) = nullptr;
    ncclResult_t (*CommWindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
    ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
    // device communicator (NCCL >= 2.28; optional: the LSA-barrier fence of peer_map 1)
    ncclResult_t (*DevCommCreate)(ncclComm_t, const ncclDevCommRequirements_t*, ncclDevComm_t*) = nullptr;
    ncclResult_t (*DevCommDestroy)(ncclComm_t, const ncclDevComm_t*) = nullptr;
    bool load(std::string& err) {
        if (h) return true;
        const char* env = getenv("AMR_NCCL_LIB");
        const char* names[] = {env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) { err = "cannot dlopen libnccl.so.2 (import torch first or set AMR_NCCL_LIB)"; return false; }
#define SYM(f, name) f = reinterpret_cast<decltype(f)>(dlsym(h, name)); if (!f) { err = std::string("missing NCCL symbol ") + name; return false; }
        SYM(CommInitRank, "ncclCommInitRank");
        SYM(CommDestroy, "ncclCommDestroy");
        SYM(GetUniqueId, "ncclGetUniqueId");
        SYM(Send, "ncclSend");
        SYM(Recv, "ncclRecv");
        SYM(GroupStart, "ncclGroupStart");
        SYM(GroupEnd, "ncclGroupEnd");
        SYM(AllReduce, "ncclAllReduce");
        SYM(GetErrorString, "ncclGetErrorString");
        SYM(CommUserRank, "ncclCommUserRank");
#undef SYM
        MemAlloc = reinterpret_cast<decltype(MemAlloc)>(dlsym(h, "ncclMemAlloc"));
        MemFree = reinterpret_cast<decltype(MemFree)>(dlsym(h, "ncclMemFree"));
        CommWindowRegister = reinterpret_cast<decltype(CommWindowRegister)>(dlsym(h, "ncclCommWindowRegister"));
        CommWindowDeregister = reinterpret_cast<decltype(CommWindowDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
        DevCommCreate = reinterpret_cast<decltype(DevCommCreate)>(dlsym(h, "ncclDevCommCreate"));
        DevCommDestroy = reinterpret_cast<decltype(DevCommDestroy)>(dlsym(h, "ncclDevCommDestroy"));
        return true;
    }
};
NcclApi& nccl_api() {
    static NcclApi api;
    return api;
}

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    bool windows = false;           // peer_map 1: map_peers registers NCCL symmetric windows instead of CUDA IPC
    ncclWindow_t win[2] = {nullptr, nullptr};   // per tag
    void** d_ptrs = nullptr;        // device scratch for the peer addresses read from a window
    // peer_map 1: a device communicator with one LSA barrier, made (collectively) with the first window; when its LSA
    // team is the whole world (one NVLink domain) the stage fence is an in-kernel LSA barrier session instead of the
    // one-word allreduce
    ncclDevComm dc{};
    bool have_dc = false, lsa_fence = false;
    long long lsa_fences = 0;       // fences issued as LSA barrier kernels (the self-test reports it)
    std::string err(ncclResult_t r) { return std::string("NCCL: ") + nccl_api().GetErrorString(r); }
    std::string p2p(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) override {
        NcclApi& A = nccl_api();
        ncclResult_t r = A.GroupStart();
        if (r != ncclSuccess) return err(r);
        for (auto& x : sends)
            if (x.bytes && (r = A.Send(x.buf, x.bytes, ncclChar, x.peer, comm, s)) != ncclSuccess) return err(r);
        for (auto& x : recvs)
            if (x.bytes && (r = A.Recv(x.buf, x.bytes, ncclChar, x.peer, comm, s)) != ncclSuccess) return err(r);
        r = A.GroupEnd();
        return r == ncclSuccess ? std::string() : err(r);
    }
    std::string allreduce(void* d, size_t count, int kind, cudaStream_t s) override {
        ncclDataType_t t = kind == 0 ? ncclUint64 : (kind == 3 ? ncclInt32 : ncclFloat64);
        ncclRedOp_t op = kind == 2 ? ncclSum : ncclMax;
        ncclResult_t r = nccl_api().AllReduce(d, d, count, t, op, comm, s);
        return r == ncclSuccess ? std::string() : err(r);
    }
    // peer mapping by CUDA IPC: each rank publishes (handle of the allocation holding base, offset of base in it);
    // the W records are combined by a byte-wise sum allreduce (every record is zero except on its owner)
    std::vector<void*> opened[2];   // IPC mappings per tag
    int32_t* d_fence = nullptr;
    // peer mapping by an NCCL symmetric window (peer_map 1; base from ncclMemAlloc, the same size on every rank):
    // ncclCommWindowRegister maps every rank's buffer into one load/store-accessible range, and the peers' addresses
    // are read on the device with ncclGetPeerPointer (launch_window_peer_ptrs); this rank keeps its own base
    std::string map_peers_window(void* base, size_t bytes, std::vector<void*>& out, cudaStream_t s, int tag,
                                 std::vector<void*>* aliases = nullptr) {
        NcclApi& A = nccl_api();
        if (!A.CommWindowRegister || !A.CommWindowDeregister) return "NCCL without ncclCommWindowRegister (need >= 2.27)";
        if (win[tag]) { A.CommWindowDeregister(comm, win[tag]); win[tag] = nullptr; }
        ncclResult_t r = A.CommWindowRegister(comm, base, bytes, &win[tag], NCCL_WIN_COLL_SYMMETRIC);
        if (r != ncclSuccess) { win[tag] = nullptr; return "ncclCommWindowRegister: " + std::string(A.GetErrorString(r)); }
        if (!have_dc && A.DevCommCreate && A.DevCommDestroy) {   // collective, like the registration (same lib on all ranks)
            ncclDevCommRequirements req{};
            req.lsaBarrierCount = 1;
            r = A.DevCommCreate(comm, &req, &dc);
            if (r != ncclSuccess) return "ncclDevCommCreate: " + std::string(A.GetErrorString(r));
            have_dc = true;
            lsa_fence = dc.lsaSize == dc.nRanks;
        }
        const int world = (int)out.size();
        if (!d_ptrs && cudaMalloc(&d_ptrs, 64 * sizeof(void*)) != cudaSuccess) return "window: cudaMalloc";
        if (world > 64) return "window: more than 64 ranks";
        if (launch_window_peer_ptrs(win[tag], world, d_ptrs, s) != cudaSuccess) return "window: peer-pointer kernel";
        std::vector<void*> h(world, nullptr);
        if (cudaMemcpyAsync(h.data(), d_ptrs, world * sizeof(void*), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return "window: peer pointers";
        int me = 0;
        A.CommUserRank(comm, &me);
        for (int q = 0; q < world; ++q) out[q] = q == me ? base : h[q];
        if (aliases) *aliases = h;
        return std::string();
    }
    std::string map_peers(void* base, size_t bytes, std::vector<void*>& out, cudaStream_t s, int tag = 0) override {
        if (windows) return map_peers_window(base, bytes, out, s, tag);
        (void)bytes;
        for (void* p : opened[tag]) cudaIpcCloseMemHandle(p);   // the tag's previous buffer (re-allocated)
        opened[tag].clear();
        using RangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
        static RangeFn range = nullptr;
        if (!range) {
            void* p = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                return "cuMemGetAddressRange unavailable";
            range = reinterpret_cast<RangeFn>(p);
        }
        unsigned long long alloc = 0;
        size_t asz = 0;
        if (range(&alloc, &asz, (unsigned long long)(uintptr_t)base) != 0) return "cuMemGetAddressRange failed";
        struct Rec { cudaIpcMemHandle_t h; uint64_t off; };
        int me = 0;
        nccl_api().CommUserRank(comm, &me);
        const int world = (int)out.size();
        std::vector<Rec> recs(world);
        std::memset(recs.data(), 0, recs.size() * sizeof(Rec));
        if (cudaIpcGetMemHandle(&recs[me].h, (void*)(uintptr_t)alloc) != cudaSuccess) return "cudaIpcGetMemHandle failed";
        recs[me].off = (uint64_t)((uintptr_t)base - alloc);
        void* d = nullptr;
        const size_t nb = recs.size() * sizeof(Rec);
        if (cudaMalloc(&d, nb) != cudaSuccess) return "map_peers: cudaMalloc";
        cudaMemcpyAsync(d, recs.data(), nb, cudaMemcpyHostToDevice, s);
        ncclResult_t r = nccl_api().AllReduce(d, d, nb, ncclUint8, ncclSum, comm, s);
        if (r != ncclSuccess) { cudaFree(d); return err(r); }
        cudaMemcpyAsync(recs.data(), d, nb, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        cudaFree(d);
        for (int q = 0; q < world; ++q) {
            if (q == me) { out[q] = base; continue; }
            void* p = nullptr;
            if (cudaIpcOpenMemHandle(&p, recs[q].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
                return "cudaIpcOpenMemHandle failed";
            opened[tag].push_back(p);
            out[q] = (char*)p + recs[q].off;
        }
        return std::string();
    }
    std::string fence(cudaStream_t s) override {   // a one-word allreduce completes only after every rank reached it
        if (windows && lsa_fence) {   // peer_map 1 in one NVLink domain: the LSA barrier session, in-kernel
            if (launch_lsa_fence(&dc, s) != cudaSuccess) return "fence: LSA barrier kernel";
            ++lsa_fences;
            return std::string();
        }
        if (!d_fence && cudaMalloc(&d_fence, sizeof(int32_t)) != cudaSuccess) return "fence: cudaMalloc";
        ncclResult_t r = nccl_api().AllReduce(d_fence, d_fence, 1, ncclInt32, ncclMax, comm, s);
        return r == ncclSuccess ? std::string() : err(r);
    }
    ~NcclTransport() override {
        for (auto& v : opened)
            for (void* p : v) cudaIpcCloseMemHandle(p);
        if (have_dc && comm) nccl_api().DevCommDestroy(comm, &dc);
        for (auto& w : win)
            if (w && comm) nccl_api().CommWindowDeregister(comm, w);
        if (d_fence) cudaFree(d_fence);
        if (d_ptrs) cudaFree(d_ptrs);
        if (comm) nccl_api().CommDestroy(comm);
    }
};
#endif

// ---- host collectives (comm_backend 2, test-only): one process per rank, possibly several on one GPU; data moves
// through host memory with the caller's allgather, peer pools are mapped with CUDA IPC exactly as over NCCL.
struct HostTransport : Transport {
    const amr_host_comm* hc = nullptr;
    int world = 1, rank = 0;
    std::vector<void*> opened[2];   // IPC mappings per tag
    std::string gather(const void* send, size_t bytes, void* recv) {
        return hc->allgather(send, (uint64_t)bytes, recv, hc->user) == 0 ? std::string() : "host allgather failed";
    }
    std::string p2p(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) override {
        // every rank publishes its per-peer byte counts, then all its outgoing messages back to back
        std::vector<uint64_t> mine(world, 0), counts((size_t)world * world);
        for (auto& x : sends) mine[x.peer] = x.bytes;
        std::string e = gather(mine.data(), world * 8, counts.data());
        if (!e.empty()) return e;
        uint64_t maxtot = 0;
        for (int q = 0; q < world; ++q) {
            uint64_t t = 0;
            for (int p = 0; p < world; ++p) t += counts[(size_t)q * world + p];
            maxtot = std::max(maxtot, t);
        }
        std::vector<unsigned char> out(std::max<uint64_t>(maxtot, 1), 0), all((size_t)world * std::max<uint64_t>(maxtot, 1));
        cudaStreamSynchronize(s);
        for (auto& x : sends) {
            uint64_t off = 0;
            for (int p = 0; p < x.peer; ++p) off += mine[p];
            if (x.bytes && d2h_sync(out.data() + off, x.buf, x.bytes, s) != cudaSuccess)
                return "host p2p: download";
        }
        e = gather(out.data(), out.size(), all.data());
        if (!e.empty()) return e;
        for (auto& rv : recvs) {
            if (!rv.bytes) continue;
            const uint64_t* cq = &counts[(size_t)rv.peer * world];
            if (cq[rank] != rv.bytes) return "host p2p: unmatched receive";
            uint64_t off = 0;
            for (int p = 0; p < rank; ++p) off += cq[p];
            if (h2d_sync(rv.buf, all.data() + (size_t)rv.peer * out.size() + off, rv.bytes, s) != cudaSuccess)
                return "host p2p: upload";
        }
        return std::string();
    }
    std::string allreduce(void* d, size_t count, int kind, cudaStream_t s) override {
        const size_t esz = kind == 3 ? 4 : 8, bytes = count * esz;
        std::vector<unsigned char> mine(bytes), all(bytes * world);
        cudaStreamSynchronize(s);
        if (d2h_sync(mine.data(), d, bytes, s) != cudaSuccess) return "host allreduce: download";
        std::string e = gather(mine.data(), bytes, all.data());
        if (!e.empty()) return e;
        for (size_t k = 0; k < count; ++k)
            for (int q = 1; q < world; ++q) {
                unsigned char* a = all.data() + k * esz;
                const unsigned char* b = all.data() + (size_t)q * bytes + k * esz;
                if (kind == 0) { uint64_t x, y; std::memcpy(&x, a, 8); std::memcpy(&y, b, 8); x = std::max(x, y); std::memcpy(a, &x, 8); }
                else if (kind == 1 || kind == 2) {
                    double x, y; std::memcpy(&x, a, 8); std::memcpy(&y, b, 8);
                    x = kind == 1 ? (y > x ? y : x) : x + y; std::memcpy(a, &x, 8);
                } else { int32_t x, y; std::memcpy(&x, a, 4); std::memcpy(&y, b, 4); x = std::max(x, y); std::memcpy(a, &x, 4); }
            }
        return h2d_sync(d, all.data(), bytes, s) == cudaSuccess ? std::string() : "host allreduce: upload";
    }
    std::string map_peers(void* base, size_t, std::vector<void*>& out, cudaStream_t, int tag = 0) override {
        for (void* p : opened[tag]) cudaIpcCloseMemHandle(p);   // the tag's previous buffer (re-allocated)
        opened[tag].clear();
        using RangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
        static RangeFn range = nullptr;
        if (!range) {
            void* p = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                return "cuMemGetAddressRange unavailable";
            range = reinterpret_cast<RangeFn>(p);
        }
        unsigned long long alloc = 0;
        size_t asz = 0;
        if (range(&alloc, &asz, (unsigned long long)(uintptr_t)base) != 0) return "cuMemGetAddressRange failed";
        struct Rec { cudaIpcMemHandle_t h; uint64_t off; } me{};
        if (cudaIpcGetMemHandle(&me.h, (void*)(uintptr_t)alloc) != cudaSuccess) return "cudaIpcGetMemHandle failed";
        me.off = (uint64_t)((uintptr_t)base - alloc);
        std::vector<Rec> recs(world);
        std::string e = gather(&me, sizeof me, recs.data());
        if (!e.empty()) return e;
        for (int q = 0; q < world; ++q) {
            if (q == rank) { out[q] = base; continue; }
            void* p = nullptr;
            if (cudaIpcOpenMemHandle(&p, recs[q].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
                return "cudaIpcOpenMemHandle failed";
            opened[tag].push_back(p);
            out[q] = (char*)p + recs[q].off;
        }
        return std::string();
    }
    std::string fence(cudaStream_t s) override {   // every rank's queued work done, then a host barrier
        if (cudaStreamSynchronize(s) != cudaSuccess) return "fence: stream";
        return hc->barrier(hc->user) == 0 ? std::string() : "host barrier failed";
    }
    ~HostTransport() override {
        for (auto& v : opened)
            for (void* p : v) cudaIpcCloseMemHandle(p);
    }
};

// ---- loopback: virtual ranks = host threads of one process on one GPU (test-only)
struct LoopGroup {
    int world = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<std::vector<Xfer>> sends;
    std::vector<cudaEvent_t> ready, done;
    std::vector<void*> bufs;
    int users = 0;
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
std::mutex g_loop_mu;
std::map<std::string, std::shared_ptr<LoopGroup>> g_loops;

struct LoopTransport : Transport {
    std::shared_ptr<LoopGroup> G;
    std::string key;
    int rank = 0;
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
    std::vector<unsigned char> host;
    std::string p2p(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) override {
        cudaEventRecord(ev_ready, s);
        G->sends[rank] = sends;
        G->ready[rank] = ev_ready;
        G->barrier();
        for (auto& rv : recvs) {
            if (!rv.bytes) continue;
            const Xfer* match = nullptr;
            for (auto& sx : G->sends[rv.peer])
                if (sx.peer == rank) { match = &sx; break; }
            if (!match || match->bytes != rv.bytes) return "loopback: unmatched receive";
            cudaStreamWaitEvent(s, G->ready[rv.peer], 0);
            cudaError_t e = cudaMemcpyAsync(rv.buf, match->buf, rv.bytes, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return cudaGetErrorString(e);
        }
        cudaEventRecord(ev_done, s);
        G->done[rank] = ev_done;
        G->barrier();
        for (auto& sx : sends)
            if (sx.bytes) cudaStreamWaitEvent(s, G->done[sx.peer], 0);
        G->barrier();
        return std::string();
    }
    std::string allreduce(void* d, size_t count, int kind, cudaStream_t s) override {
        size_t esz = kind == 3 ? 4 : 8;
        size_t bytes = count * esz;
        cudaStreamSynchronize(s);
        G->bufs[rank] = d;
        G->barrier();
        std::vector<unsigned char> acc(bytes), tmp(bytes);
        for (int q = 0; q < G->world; ++q) {
            if (d2h_sync(q == 0 ? acc.data() : tmp.data(), G->bufs[q], bytes, s) != cudaSuccess)
                return "loopback allreduce copy failed";
            if (q == 0) continue;
            for (size_t e = 0; e < count; ++e) {
                if (kind == 0) {
                    uint64_t a, b; std::memcpy(&a, &acc[e * 8], 8); std::memcpy(&b, &tmp[e * 8], 8);
                    a = std::max(a, b); std::memcpy(&acc[e * 8], &a, 8);
                } else if (kind == 1 || kind == 2) {
                    double a, b; std::memcpy(&a, &acc[e * 8], 8); std::memcpy(&b, &tmp[e * 8], 8);
                    a = kind == 1 ? (b > a ? b : a) : a + b; std::memcpy(&acc[e * 8], &a, 8);
                } else {
                    int32_t a, b; std::memcpy(&a, &acc[e * 4], 4); std::memcpy(&b, &tmp[e * 4], 4);
                    a = std::max(a, b); std::memcpy(&acc[e * 4], &a, 4);
                }
            }
        }
        G->barrier();   // everyone has read every buffer
        if (h2d_sync(d, acc.data(), bytes, s) != cudaSuccess) return "loopback allreduce write failed";
        G->barrier();
        return std::string();
    }
    std::string map_peers(void* base, size_t, std::vector<void*>& out, cudaStream_t, int tag = 0) override {
        (void)tag;
        G->bufs[rank] = base;   // virtual ranks share the process: their buffers are directly addressable
        G->barrier();
        for (int q = 0; q < G->world; ++q) out[q] = G->bufs[q];
        G->barrier();
        return std::string();
    }
    std::string fence(cudaStream_t s) override {   // CUDA events between the virtual ranks' streams (no spinning)
        cudaEventRecord(ev_ready, s);
        G->ready[rank] = ev_ready;
        G->barrier();
        for (int q = 0; q < G->world; ++q)
            if (q != rank) cudaStreamWaitEvent(s, G->ready[q], 0);
        G->barrier();
        return std::string();
    }
    ~LoopTransport() override {
        if (ev_ready) cudaEventDestroy(ev_ready);
        if (ev_done) cudaEventDestroy(ev_done);
        std::lock_guard<std::mutex> lk(g_loop_mu);
        if (G && --G->users == 0) g_loops.erase(key);
    }
};

// =====================================================================================  Comm
Comm::Comm() = default;
Comm::~Comm() = default;

amr_status Comm::init(amr_ctx* c) {
    n = c->n;
    world = c->cfg.world_size;
    rank = c->cfg.rank;
    halo_mode = c->cfg.halo_mode;
    subcycle = c->cfg.subcycle != 0;
    owner = partition_owners(c->tree, world);
    if (world == 1) return AMR_OK;
    if (c->cfg.comm_backend == 2) {
        if (!c->cfg.host_comm || !c->cfg.host_comm->allgather || !c->cfg.host_comm->barrier) {
            c->err = "comm_backend 2 needs host_comm with allgather and barrier";
            return AMR_E_CONFIG;
        }
        auto* T = new HostTransport();
        T->hc = c->cfg.host_comm;
        T->world = world;
        T->rank = rank;
        tr.reset(T);
        return AMR_OK;
    }
    if (c->cfg.comm_backend == 1) {
        auto* T = new LoopTransport();
        T->rank = rank;
        T->key.assign((const char*)c->cfg.nccl_unique_id, strnlen((const char*)c->cfg.nccl_unique_id, 128));
        {
            std::lock_guard<std::mutex> lk(g_loop_mu);
            auto& G = g_loops[T->key];
            if (!G) {
                G = std::make_shared<LoopGroup>();
                G->world = world;
                G->sends.resize(world);
                G->ready.resize(world);
                G->done.resize(world);
                G->bufs.resize(world);
            }
            if (G->world != world) { delete T; c->err = "loopback group size mismatch"; return AMR_E_CONFIG; }
            G->users++;
            T->G = G;
        }
        cudaEventCreateWithFlags(&T->ev_ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&T->ev_done, cudaEventDisableTiming);
        tr.reset(T);
        T->G->barrier();   // all virtual ranks created
        return AMR_OK;
    }
#ifdef AMR_HAVE_NCCL_H
    std::string e;
    if (!nccl_api().load(e)) { c->err = e; return AMR_E_COMM; }
    auto* T = new NcclTransport();
    ncclUniqueId id;
    std::memcpy(&id, c->cfg.nccl_unique_id, sizeof id);
    ncclResult_t r = nccl_api().CommInitRank(&T->comm, world, id, rank);
    if (r != ncclSuccess) {
        c->err = std::string("ncclCommInitRank: ") + nccl_api().GetErrorString(r);
        delete T;
        return AMR_E_COMM;
    }
    T->windows = c->cfg.peer_map == 1;
    tr.reset(T);
    return AMR_OK;
#else
    c->err = "library built without nccl.h";
    return AMR_E_COMM;
#endif
}

void Comm::finalize(amr_ctx*) {
    free_dev_lists();
    for (PullList* P : {&pull_halo, &pull_flux, &pull_halo_cf})
        if (P->slots) { cudaFree(P->slots); cudaFree(P->peers); P->slots = P->peers = nullptr; }
    if (d_pool_bases) cudaFree(d_pool_bases);
    if (d_freg_bases) cudaFree(d_freg_bases);
    d_pool_bases = d_freg_bases = nullptr;
    tr.reset();
}

void Comm::repartition(const PatchTree& t) { owner = partition_owners(t, world); }

void Comm::replan(const PatchTree& t) {
    if (world == 1) return;
    free_dev_lists();
    halo = plan_halo(t, owner, world, rank, n);
    flux = plan_flux(t, owner, world, rank);
    if (halo_mode == 2) halo_cf = plan_halo(t, owner, world, rank, n, false);
    if (subcycle) sub = plan_subcycle(t, owner, world, rank, n);
    ++lists_version;
}

void Comm::free_dev_lists() {
    for (auto& kv : dev_lists) {
        if (kv.second.send) cudaFree(kv.second.send);
        if (kv.second.recv) cudaFree(kv.second.recv);
    }
    dev_lists.clear();
}

amr_status Comm::exchange_lists(amr_ctx* c, const ExchangeLists& L, double* U, int per, const char* what,
                                bool persistent) {
    if (world == 1) return AMR_OK;
    NvtxRange nv(what);
    if (L.items) per = 16 * n;   // a band item: 4 variables x 4 n cells
    size_t ns = L.nsend(), nr = L.nrecv();
    cudaStream_t s = c->stream;
    auto bad = [&](amr_status st, const std::string& m) { c->err = std::string(what) + ": " + m; c->sticky = st; return st; };
    const int32_t *dsidx = nullptr, *dridx = nullptr;
    DevLists* dl = persistent ? &dev_lists[&L] : nullptr;
    if (dl && dl->version == lists_version) {   // index lists already on the device (this plan)
        dsidx = dl->send;
        dridx = dl->recv;
    } else {
        std::vector<int32_t> sidx, ridx;
        sidx.reserve(ns);
        ridx.reserve(nr);
        for (auto& v : L.send) sidx.insert(sidx.end(), v.begin(), v.end());
        for (auto& v : L.recv) ridx.insert(ridx.end(), v.begin(), v.end());
        if (dl) {
            if (dl->send) cudaFree(dl->send);
            if (dl->recv) cudaFree(dl->recv);
            dl->send = dl->recv = nullptr;
            if ((ns && cudaMalloc(&dl->send, ns * 4) != cudaSuccess) || (nr && cudaMalloc(&dl->recv, nr * 4) != cudaSuccess))
                return bad(AMR_E_CUDA, "index lists");
            if ((ns && h2d_sync(dl->send, sidx.data(), ns * 4, s) != cudaSuccess) ||
                (nr && h2d_sync(dl->recv, ridx.data(), nr * 4, s) != cudaSuccess))
                return bad(AMR_E_CUDA, "index lists upload");
            dl->version = lists_version;
            dsidx = dl->send;
            dridx = dl->recv;
        } else {
            if (c->x_sidx.upload(sidx, s) != cudaSuccess || c->x_ridx.upload(ridx, s) != cudaSuccess)
                return bad(AMR_E_CUDA, "exchange lists");
            dsidx = c->x_sidx.p;
            dridx = c->x_ridx.p;
        }
    }
    if (c->x_send.reserve(std::max<size_t>(1, ns * per)) != cudaSuccess ||
        c->x_recv.reserve(std::max<size_t>(1, nr * per)) != cudaSuccess)
        return bad(AMR_E_CUDA, "exchange buffers");
    if (ns) {
        cudaError_t e = L.items ? launch_band_gather(U, dsidx, (int)ns, c->x_send.p, n, s)
                                : launch_gather(U, dsidx, (int)ns, c->x_send.p, per, s);
        if (e != cudaSuccess) return bad(AMR_E_CUDA, "pack");
    }
    std::vector<Xfer> sends, recvs;
    size_t so = 0, ro = 0;
    for (int p = 0; p < world; ++p) {
        if (!L.send[p].empty()) sends.push_back({p, c->x_send.p + so * per, L.send[p].size() * per * sizeof(double)});
        if (!L.recv[p].empty()) recvs.push_back({p, c->x_recv.p + ro * per, L.recv[p].size() * per * sizeof(double)});
        so += L.send[p].size();
        ro += L.recv[p].size();
    }
    std::string e = tr->p2p(sends, recvs, s);
    if (!e.empty()) return bad(AMR_E_COMM, e);
    bytes_sent += (int64_t)(ns * per * sizeof(double));
    if (nr) {
        cudaError_t e2 = L.items ? launch_band_scatter(c->x_recv.p, dridx, (int)nr, U, n, s)
                                 : launch_scatter(c->x_recv.p, dridx, (int)nr, U, per, s);
        if (e2 != cudaSuccess) return bad(AMR_E_CUDA, "unpack");
    }
    c->st.launches += (ns ? 1 : 0) + (nr ? 1 : 0);
    return AMR_OK;
}

amr_status Comm::exchange_halos(amr_ctx* c, double* U) {
    if (world > 1 && halo_mode >= 1) return peer_pull(c, halo, pull_halo, U, false, "halo pull");
    return exchange_lists(c, halo, U, (int)c->PS, "halo exchange", true);
}

amr_status Comm::exchange_halos_stage(amr_ctx* c, double* U) {
    if (world > 1 && halo_mode == 2) return peer_pull(c, halo_cf, pull_halo_cf, U, false, "C/F source pull");
    return exchange_halos(c, U);
}

amr_status Comm::exchange_fluxes(amr_ctx* c) {
    if (world > 1 && halo_mode >= 1) return peer_pull(c, flux, pull_flux, c->freg.p, true, "flux-register pull");
    return exchange_lists(c, flux, c->freg.p, 16 * c->n, "flux-register exchange", true);
}

amr_status Comm::map_pool(amr_ctx* c, void* base, size_t bytes) {
    std::vector<void*> peers(world, nullptr);
    std::string e = tr->map_peers(base, bytes, peers, c->stream);
    if (!e.empty()) { c->err = "halo_mode 1: " + e; return AMR_E_COMM; }
    if (!d_pool_bases && cudaMalloc(&d_pool_bases, world * sizeof(double*)) != cudaSuccess) return AMR_E_CUDA;
    if (h2d_sync(d_pool_bases, peers.data(), world * sizeof(double*), c->stream) != cudaSuccess)
        return AMR_E_CUDA;
    pool_base = base;
    peer_pool.assign(world, nullptr);
    for (int q = 0; q < world; ++q) peer_pool[q] = (double*)peers[q];
    return AMR_OK;
}

// fence, then one pull kernel for every slot of L.recv (each from its owner's mapped buffer at the same offset);
// the slot lists go to the device once per plan.  Every rank calls this at the same points (collective fence).
amr_status Comm::peer_pull(amr_ctx* c, const ExchangeLists& L, PullList& P, double* dst, bool freg, const char* what) {
    NvtxRange nv(what);
    auto bad = [&](amr_status st, const std::string& m) { c->err = std::string(what) + ": " + m; c->sticky = st; return st; };
    if (freg && mapped_freg != c->freg.p) {   // (re)map the flux-register buffers (identical sizes on every rank)
        std::vector<void*> peers(world, nullptr);
        std::string e = tr->map_peers(c->freg.p, c->freg.cap * sizeof(double), peers, c->stream, 1);
        if (!e.empty()) return bad(AMR_E_COMM, e);
        if (!d_freg_bases && cudaMalloc(&d_freg_bases, world * sizeof(double*)) != cudaSuccess) return bad(AMR_E_CUDA, "alloc");
        if (h2d_sync(d_freg_bases, peers.data(), world * sizeof(double*), c->stream) != cudaSuccess)
            return bad(AMR_E_CUDA, "peer table");
        mapped_freg = c->freg.p;
    }
    if (P.version != lists_version) {
        std::vector<int32_t> sl, pe;
        for (int p = 0; p < world; ++p)
            for (int32_t id : L.recv[p]) { sl.push_back(id); pe.push_back(p); }
        if (P.slots) { cudaFree(P.slots); cudaFree(P.peers); P.slots = P.peers = nullptr; }
        P.n = (int)sl.size();
        if (P.n) {
            if (cudaMalloc(&P.slots, sl.size() * 4) != cudaSuccess || cudaMalloc(&P.peers, pe.size() * 4) != cudaSuccess)
                return bad(AMR_E_CUDA, "lists");
            if (h2d_sync(P.slots, sl.data(), sl.size() * 4, c->stream) != cudaSuccess ||
                h2d_sync(P.peers, pe.data(), pe.size() * 4, c->stream) != cudaSuccess)
                return bad(AMR_E_CUDA, "lists upload");
        }
        P.version = lists_version;
    }
    std::string e = tr->fence(c->stream);
    if (!e.empty()) return bad(AMR_E_COMM, e);
    const int per = L.items ? 16 * c->n : (freg ? 16 * c->n : (int)c->PS);
    const size_t off = freg ? 0 : (size_t)(dst - (double*)pool_base);
    if (P.n) {
        cudaError_t ce = L.items ? launch_band_pull(P.slots, P.peers, P.n, d_pool_bases, off, dst, c->n, c->stream)
                                 : launch_peer_pull(P.slots, P.peers, P.n, freg ? d_freg_bases : d_pool_bases, off, dst,
                                                    per, c->stream);
        if (ce != cudaSuccess) return bad(AMR_E_CUDA, "pull kernel");
        c->st.launches += 1;
        bytes_sent += (int64_t)P.n * per * (int64_t)sizeof(double);   // bytes moved into this rank
    }
    return AMR_OK;
}

amr_status Comm::allreduce_max_u64(amr_ctx* c, unsigned long long* d) {
    if (world == 1) return AMR_OK;
    std::string e = tr->allreduce(d, 1, 0, c->stream);
    if (!e.empty()) { c->err = e; c->sticky = AMR_E_COMM; return AMR_E_COMM; }
    return AMR_OK;
}

amr_status Comm::allreduce_max_i32(amr_ctx* c, int32_t* d, int n) {
    if (world == 1) return AMR_OK;
    std::string e = tr->allreduce(d, n, 3, c->stream);
    if (!e.empty()) { c->err = e; c->sticky = AMR_E_COMM; return AMR_E_COMM; }
    return AMR_OK;
}

amr_status Comm::allreduce_sum4(amr_ctx* c, double* h4) {
    if (world == 1) return AMR_OK;
    if (c->x_send.reserve(4) != cudaSuccess) { c->sticky = AMR_E_CUDA; return AMR_E_CUDA; }
    cudaMemcpyAsync(c->x_send.p, h4, 32, cudaMemcpyHostToDevice, c->stream);
    std::string e = tr->allreduce(c->x_send.p, 4, 2, c->stream);
    if (!e.empty()) { c->err = e; c->sticky = AMR_E_COMM; return AMR_E_COMM; }
    cudaMemcpyAsync(h4, c->x_send.p, 32, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    return AMR_OK;
}

amr_status Comm::allgather_flags(amr_ctx* c, std::vector<double>& eta, std::vector<uint8_t>& amb) {
    if (world == 1) return AMR_OK;
    size_t m = eta.size();
    std::vector<double> e2(m);
    std::vector<int32_t> a2(m);
    for (size_t k = 0; k < m; ++k) {
        e2[k] = (eta[k] >= 0.0) ? eta[k] : -1.0;   // non-owned (NaN) -> -1 loses every max
        a2[k] = amb[k];
    }
    if (c->x_send.reserve(std::max<size_t>(1, m)) != cudaSuccess ||
        c->x_recv.reserve(std::max<size_t>(1, (m + 1) / 2)) != cudaSuccess) {
        c->sticky = AMR_E_CUDA;
        return AMR_E_CUDA;
    }
    cudaMemcpyAsync(c->x_send.p, e2.data(), m * 8, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(c->x_recv.p, a2.data(), m * 4, cudaMemcpyHostToDevice, c->stream);
    std::string e = tr->allreduce(c->x_send.p, m, 1, c->stream);
    if (e.empty()) e = tr->allreduce(c->x_recv.p, m, 3, c->stream);
    if (!e.empty()) { c->err = e; c->sticky = AMR_E_COMM; return AMR_E_COMM; }
    cudaMemcpyAsync(e2.data(), c->x_send.p, m * 8, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(a2.data(), c->x_recv.p, m * 4, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    for (size_t k = 0; k < m; ++k) {
        eta[k] = e2[k] >= 0.0 ? e2[k] : std::nan("");
        amb[k] = (uint8_t)a2[k];
    }
    return AMR_OK;
}

amr_status Comm::allgather_requests(amr_ctx* c, std::vector<int32_t>& lst) {
    if (world == 1) return AMR_OK;
    auto bad = [&](amr_status st, const std::string& m) { c->err = "request exchange: " + m; c->sticky = st; return st; };
    const int32_t mine = (int32_t)lst.size();
    // device scratch: [world] counts out, [world] counts in, then the lists
    if (c->x_send.reserve((size_t)world + lst.size() / 2 + 2) != cudaSuccess) return bad(AMR_E_CUDA, "alloc");
    int32_t* dsend = reinterpret_cast<int32_t*>(c->x_send.p);
    std::vector<int32_t> cnt_out(world, mine), cnt_in(world, 0);
    if (c->x_recv.reserve((size_t)world) != cudaSuccess) return bad(AMR_E_CUDA, "alloc");
    int32_t* drecv = reinterpret_cast<int32_t*>(c->x_recv.p);
    if (h2d_sync(dsend, cnt_out.data(), world * 4, c->stream) != cudaSuccess) return bad(AMR_E_CUDA, "upload");
    std::vector<Xfer> sends, recvs;
    for (int p = 0; p < world; ++p)
        if (p != rank) { sends.push_back({p, dsend + p, 4}); recvs.push_back({p, drecv + p, 4}); }
    std::string e = tr->p2p(sends, recvs, c->stream);
    if (!e.empty()) return bad(AMR_E_COMM, e);
    if (d2h_sync(cnt_in.data(), drecv, world * 4, c->stream) != cudaSuccess) return bad(AMR_E_CUDA, "download");
    cnt_in[rank] = mine;
    size_t total = 0;
    for (int p = 0; p < world; ++p) {
        if (cnt_in[p] < 0 || cnt_in[p] % 2) return bad(AMR_E_COMM, "bad count");
        total += (size_t)cnt_in[p];
    }
    if (c->x_send.reserve(std::max<size_t>(1, (size_t)mine / 2 + 1)) != cudaSuccess ||
        c->x_recv.reserve(std::max<size_t>(1, total / 2 + 1)) != cudaSuccess)
        return bad(AMR_E_CUDA, "alloc");
    dsend = reinterpret_cast<int32_t*>(c->x_send.p);
    drecv = reinterpret_cast<int32_t*>(c->x_recv.p);
    if (mine && h2d_sync(dsend, lst.data(), (size_t)mine * 4, c->stream) != cudaSuccess) return bad(AMR_E_CUDA, "upload");
    sends.clear();
    recvs.clear();
    size_t off = 0;
    std::vector<size_t> at(world, 0);
    for (int p = 0; p < world; ++p) {
        at[p] = off;
        if (p != rank) {
            sends.push_back({p, dsend, (size_t)mine * 4});
            recvs.push_back({p, drecv + off, (size_t)cnt_in[p] * 4});
            off += (size_t)cnt_in[p];
        }
    }
    e = tr->p2p(sends, recvs, c->stream);
    if (!e.empty()) return bad(AMR_E_COMM, e);
    std::vector<int32_t> got(off);
    if (off && d2h_sync(got.data(), drecv, off * 4, c->stream) != cudaSuccess) return bad(AMR_E_CUDA, "download");
    lst.insert(lst.end(), got.begin(), got.end());
    bytes_sent += (int64_t)mine * 4 * (world - 1);
    return AMR_OK;
}

amr_status Comm::agree_error(amr_ctx*, int32_t*) { return AMR_OK; }

void* comm_nccl_mem_alloc(size_t bytes, std::string& err) {
#ifdef AMR_HAVE_NCCL_H
    if (!nccl_api().load(err)) return nullptr;
    if (!nccl_api().MemAlloc) { err = "NCCL without ncclMemAlloc (need >= 2.19)"; return nullptr; }
    void* p = nullptr;
    ncclResult_t r = nccl_api().MemAlloc(&p, bytes);
    if (r != ncclSuccess) { err = std::string("ncclMemAlloc: ") + nccl_api().GetErrorString(r); return nullptr; }
    return p;
#else
    (void)bytes;
    err = "library built without nccl.h";
    return nullptr;
#endif
}

void comm_nccl_mem_free(void* p) {
#ifdef AMR_HAVE_NCCL_H
    if (p && nccl_api().MemFree) nccl_api().MemFree(p);
#else
    (void)p;
#endif
}

}  // namespace amr

// ====================================================================================  C ABI pieces
extern "C" amr_status amr_nccl_unique_id(void* out128) {
    if (!out128) return AMR_E_ARG;
#ifdef AMR_HAVE_NCCL_H
    std::string e;
    if (!amr::nccl_api().load(e)) return AMR_E_COMM;
    ncclUniqueId id;
    if (amr::nccl_api().GetUniqueId(&id) != ncclSuccess) return AMR_E_COMM;
    std::memcpy(out128, &id, sizeof id);
    return AMR_OK;
#else
    return AMR_E_COMM;
#endif
}

// ====================================================================================  test-only: NCCL self-test
// Drives the NCCL transport of the data path (NcclTransport: grouped send/recv, the four allreduce kinds, the
// peer-mapping exchange and the stream-ordered fence) on a ONE-rank communicator -- the only communicator a one-GPU
// box can host -- so that every resolved NCCL entry point runs once: ncclCommInitRank, ncclCommUserRank,
// ncclGroupStart/End, ncclSend/Recv (to self), ncclAllReduce (max u64 / max f64 / sum f64 / max i32 / byte sum),
// ncclGetErrorString, ncclCommDestroy.  Results are checked: the received bytes equal the sent ones and a 1-rank
// reduction is the identity.
extern "C" amr_status amr_debug_nccl_selftest(const void* uid128, char* msg, int32_t msg_cap) {
    auto say = [&](const std::string& m) {
        if (msg && msg_cap > 0) {
            std::strncpy(msg, m.c_str(), (size_t)msg_cap - 1);
            msg[msg_cap - 1] = 0;
        }
    };
    if (!uid128) return AMR_E_ARG;
#ifdef AMR_HAVE_NCCL_H
    std::string e;
    if (!amr::nccl_api().load(e)) { say(e); return AMR_E_COMM; }
    amr::NcclApi& A = amr::nccl_api();
    auto T = std::make_unique<amr::NcclTransport>();
    ncclUniqueId id;
    std::memcpy(&id, uid128, sizeof id);
    ncclResult_t r = A.CommInitRank(&T->comm, 1, id, 0);
    if (r != ncclSuccess) { say(std::string("ncclCommInitRank: ") + A.GetErrorString(r)); return AMR_E_COMM; }
    say(std::string("ok: ") + A.GetErrorString(ncclSuccess));
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) { say("stream"); return AMR_E_CUDA; }
    const size_t n = 4096;
    std::vector<double> h(n), back(n);
    for (size_t i = 0; i < n; ++i) h[i] = std::ldexp((double)(i * 2654435761u % 1000003u), -7) - 3.0;
    double *src = nullptr, *dst = nullptr;
    amr_status st = AMR_OK;
    auto fail = [&](amr_status code, const std::string& m) { say(m); st = code; };
    if (cudaMalloc(&src, n * 8) != cudaSuccess || cudaMalloc(&dst, n * 8) != cudaSuccess) fail(AMR_E_CUDA, "malloc");
    if (st == AMR_OK) {
        amr::h2d_sync(src, h.data(), n * 8, s);
        cudaMemsetAsync(dst, 0, n * 8, s);
        // grouped send/recv to self, as exchange_lists issues them (one Xfer per peer)
        std::string x = T->p2p({{0, src, n * 8}}, {{0, dst, n * 8}}, s);
        if (!x.empty()) fail(AMR_E_COMM, x);
        else if (amr::d2h_sync(back.data(), dst, n * 8, s) != cudaSuccess) fail(AMR_E_CUDA, "d2h");
        else if (std::memcmp(back.data(), h.data(), n * 8) != 0) fail(AMR_E_COMM, "send/recv to self: data differ");
    }
    for (int kind = 0; kind < 4 && st == AMR_OK; ++kind) {   // 1-rank reductions: identity
        std::string x = T->allreduce(src, kind == 3 ? 2 * n : n, kind, s);
        if (!x.empty()) { fail(AMR_E_COMM, x); break; }
        if (amr::d2h_sync(back.data(), src, n * 8, s) != cudaSuccess) { fail(AMR_E_CUDA, "d2h"); break; }
        if (std::memcmp(back.data(), h.data(), n * 8) != 0) fail(AMR_E_COMM, "allreduce kind " + std::to_string(kind) + " changed data");
    }
    if (st == AMR_OK) {   // peer table (byte-sum allreduce of the IPC records) and the fence
        std::vector<void*> peers(1, nullptr);
        std::string x = T->map_peers(src, n * 8, peers, s);
        if (!x.empty()) fail(AMR_E_COMM, x);
        else if (peers[0] != (void*)src) fail(AMR_E_COMM, "map_peers: own base not returned");
        else if (!(x = T->fence(s)).empty()) fail(AMR_E_COMM, x);
        else if (cudaStreamSynchronize(s) != cudaSuccess) fail(AMR_E_CUDA, "sync");
    }
    std::string win_note = "windows not exercised";
    if (st == AMR_OK && A.MemAlloc && A.CommWindowRegister) {   // peer_map 1: ncclMemAlloc + symmetric window
        std::string e2;
        const size_t wb = 1 << 20;
        void* wbuf = amr::comm_nccl_mem_alloc(wb, e2);
        if (!wbuf) fail(AMR_E_COMM, e2);
        else {
            T->windows = true;
            std::vector<void*> peers(1, nullptr), alias;
            std::string x = T->map_peers_window(wbuf, wb, peers, s, 0, &alias);
            if (!x.empty()) fail(AMR_E_COMM, x);
            else if (peers[0] != wbuf || !alias[0]) fail(AMR_E_COMM, "window: own base / alias not returned");
            else {   // rank 0's window address aliases the buffer: write through the alias, read through the base
                std::vector<double> got(n);
                if (cudaMemcpyAsync(alias[0], h.data(), n * 8, cudaMemcpyHostToDevice, s) != cudaSuccess ||
                    amr::d2h_sync(got.data(), wbuf, n * 8, s) != cudaSuccess)
                    fail(AMR_E_CUDA, "window: copy");
                else if (std::memcmp(got.data(), h.data(), n * 8) != 0) fail(AMR_E_COMM, "window: alias does not map the buffer");
                else win_note = "window ok";
                // the peer_map 1 fence: an LSA barrier session in a kernel when the device communicator exists
                if (st == AMR_OK && T->lsa_fence) {
                    const long long f0 = T->lsa_fences;
                    for (int k = 0; k < 3 && st == AMR_OK; ++k)
                        if (!(x = T->fence(s)).empty()) fail(AMR_E_COMM, x);
                    if (st == AMR_OK && cudaStreamSynchronize(s) != cudaSuccess) fail(AMR_E_CUDA, "LSA fence: sync");
                    else if (st == AMR_OK && T->lsa_fences == f0 + 3) win_note += "; lsa barrier fence ok";
                } else if (st == AMR_OK) {
                    win_note += T->have_dc ? "; devcomm LSA team is not the world" : "; no ncclDevCommCreate";
                }
            }
            if (T->win[0]) { A.CommWindowDeregister(T->comm, T->win[0]); T->win[0] = nullptr; }
            amr::comm_nccl_mem_free(wbuf);
        }
    }
    if (st == AMR_OK) say(std::string("ok: ") + A.GetErrorString(ncclSuccess) + "; " + win_note);
    cudaFree(src);
    cudaFree(dst);
    T.reset();   // ncclCommDestroy
    cudaStreamDestroy(s);
    return st;
#else
    (void)msg_cap;
    say("library built without nccl.h");
    return AMR_E_COMM;
#endif
}
