// plan.cpp -- the host spin pool and the parallel plan phases (plan.h).
#include "plan.h"

#include <unistd.h>

#include <algorithm>
#include <cstdlib>

namespace amr {

namespace {
inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#elif defined(__aarch64__)
    asm volatile("yield" ::: "memory");
#endif
}
}  // namespace

HostPool& HostPool::get() {
    // leaked on purpose: workers asleep on the condition variable at process exit are never joined
    static HostPool* p = [] {
        // default: the hardware threads shared among the node's ranks (torchrun's LOCAL_WORLD_SIZE), at most 8 --
        // spinning workers must not oversubscribe the cores the ranks' own threads run on
        const char* e = std::getenv("AMR_HOST_THREADS");
        const char* lw = std::getenv("LOCAL_WORLD_SIZE");
        const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
        const int ranks = lw ? std::max(1, std::atoi(lw)) : 1;
        int total = e ? std::atoi(e) : std::max(1, std::min(8, hw / ranks));
        return new HostPool(std::max(0, std::min(total, 64) - 1));
    }();
    return *p;
}

HostPool::HostPool(int workers) : nworkers_(workers), pid_((int)getpid()) {
    for (int w = 0; w < nworkers_; ++w) th_.emplace_back([this] { worker(); });
}

void HostPool::arm() {
    if (nworkers_ == 0) return;
    std::lock_guard<std::mutex> lk(m_);
    armed_.fetch_add(1);
    cv_.notify_all();
}

void HostPool::disarm() {
    if (nworkers_ == 0) return;
    armed_.fetch_sub(1);
}

void HostPool::worker() {
    uint64_t last = 0;
    for (;;) {
        {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return armed_.load() > 0; });
        }
        while (armed_.load(std::memory_order_relaxed) > 0) {
            const uint64_t g = gen_.load(std::memory_order_acquire);
            if (g == last) {
                cpu_relax();
                continue;
            }
            // announce before touching the job: run_erased waits for busy_ == 0 after withdrawing it (seq_cst)
            busy_.fetch_add(1);
            Job* j = cur_.load();
            if (j) {
                for (int k; (k = j->next.fetch_add(1)) < j->parts;) {
                    j->fn(j->ctx, k);
                    j->done.fetch_add(1, std::memory_order_release);
                }
                last = j->id;
            } else {
                last = g;
            }
            busy_.fetch_sub(1);
        }
    }
}

void HostPool::run_erased(int parts, void (*fn)(void*, int), void* ctx) {
    if (parts <= 0) return;
    std::unique_lock<std::mutex> jl(job_m_, std::try_to_lock);
    if (parts == 1 || nworkers_ == 0 || serial_ || armed_.load() == 0 || !jl.owns_lock() || (int)getpid() != pid_) {
        for (int k = 0; k < parts; ++k) fn(ctx, k);
        return;
    }
    Job j;
    j.fn = fn;
    j.ctx = ctx;
    j.parts = parts;
    j.id = ++seq_;
    cur_.store(&j);
    gen_.store(j.id);
    for (int k; (k = j.next.fetch_add(1)) < parts;) {
        fn(ctx, k);
        j.done.fetch_add(1, std::memory_order_release);
    }
    while (j.done.load(std::memory_order_acquire) < parts) cpu_relax();
    cur_.store(nullptr);
    while (busy_.load() > 0) cpu_relax();   // no worker still holds &j (a stack object)
}

void plan_face_neighbours(const PatchTree& t, const std::vector<int32_t>& roots, std::vector<int32_t>& nb4) {
    if (nb4.size() != (size_t)4 * t.capacity) nb4.assign((size_t)4 * t.capacity, -1);
    HostPool& pool = HostPool::get();
    // ONE part: the subtrees' slots interleave in the slot space, so parts would write the same cache lines of nb4
    // (false sharing made 4 threads 1.4x slower than one on the shock-bubble tree); the parts API is kept
    const int parts = 1;
    static thread_local std::vector<std::vector<int32_t>> stacks;
    std::vector<std::vector<int32_t>>& S = stacks;   // the caller's scratch (parts run on the workers)
    if ((int)S.size() < parts) S.resize(parts);
    const size_t nr = roots.size();
    pool.run(parts, [&](int k) {
        const size_t r0 = nr * k / parts, r1 = nr * (k + 1) / parts;
        t.face_neighbours_span(roots.data() + r0, r1 - r0, nb4, S[k]);
    });
}

void update_face_neighbours(const PatchTree& t, const std::vector<int32_t>& created, const std::vector<int32_t>& deleted,
                            std::vector<int32_t>& nb4) {
    for (int d : deleted)
        for (int s = 0; s < 4; ++s) {
            const int q = nb4[(size_t)4 * d + s];   // (the deleted slot's entries are those of the previous tree)
            if (q >= 0 && t.alive[q] && nb4[(size_t)4 * q + (s ^ 1)] == d) nb4[(size_t)4 * q + (s ^ 1)] = -1;
        }
    for (int id : created) {
        t.face_neighbours_one(id, nb4);
        for (int s = 0; s < 4; ++s) {
            const int q = nb4[(size_t)4 * id + s];
            if (q >= 0) nb4[(size_t)4 * q + (s ^ 1)] = id;
        }
    }
}

namespace {
// The descriptors of leaf_ids[e0, e1): proxies and reflux tasks numbered from 0 within the part (the merge shifts
// them); the first inconsistency sets err and stops the part.
bool describe_part(const PatchTree& t, const std::vector<int32_t>& nb4, const std::vector<int32_t>& leaf_ids,
                   size_t e0, size_t e1, const Owners& owner, int world, int rank, int halo_mode, DescOut& o,
                   std::string& err) {
    o.leaves.clear();
    o.ptasks.clear();
    o.rtasks.clear();
    // a C/F parent's 3 x 3 neighbourhood: faces from nb4, corners through the N / S face neighbour (R2: all 8
    // exist inside the domain); -2 outside the domain
    auto nbr = [&](int id, int dx, int dy) -> int {
        if (dx == 0 && dy == 0) return id;
        const int32_t* n4 = &nb4[(size_t)4 * id];
        if (dy == 0) return n4[dx < 0 ? kW : kE];
        const int v = n4[dy < 0 ? kS : kN];
        if (dx == 0 || v < 0) return v;
        const int r = nb4[(size_t)4 * v + (dx < 0 ? kW : kE)];
        return r == -1 ? t.neighbour(id, dx, dy) : r;   // (-1: R2 violated; neighbour() decides as before)
    };
    int cpar = -1, cnb[9];   // the last C/F parent's 3 x 3 neighbourhood
    for (size_t e = e0; e < e1; ++e) {
        const int id = leaf_ids[e];
        LeafDesc d{};
        d.slot = id;
        d.level = t.lev[id];
        d.cf = 0;
        RefluxTask rt{};
        rt.leaf = (int)(e - e0);
        rt.slot = id;
        rt.level = t.lev[id];
        rt.mask = 0;
        for (int s = 0; s < 4; ++s) {
            const int nb = nb4[(size_t)4 * id + s];
            if (nb >= 0) {
                d.side[s] = nb;
                if (world > 1 && halo_mode == 2 && owner[nb] != rank)
                    d.pad |= (16 << s) | (owner[nb] << (8 + 3 * s));   // strip read from the owner's pool
                if (t.has_children(nb)) {
                    d.cf |= 1 << s;
                    rt.mask |= 1 << s;
                    // the two children of nb adjacent to the shared face, ordered along it
                    int cidx[2];
                    if (s == kW) { cidx[0] = 1; cidx[1] = 3; }
                    else if (s == kE) { cidx[0] = 0; cidx[1] = 2; }
                    else if (s == kS) { cidx[0] = 2; cidx[1] = 3; }
                    else { cidx[0] = 0; cidx[1] = 1; }
                    for (int h = 0; h < 2; ++h) {
                        const int ch = t.child[4 * nb + cidx[h]];
                        if (ch < 0 || !t.is_leaf(ch)) { err = "reflux: fine side is not a leaf"; return false; }
                        rt.fine[s][h] = ch;
                    }
                }
            } else {
                ProxyTask p{};
                p.proxy = (int)o.ptasks.size();
                p.slot = id;
                p.side = s;
                p.level = t.lev[id];
                p.P = t.pi[id];
                p.Q = t.pj[id];
                if (nb == -2) {
                    p.kind = 0;
                    for (int q = 0; q < 9; ++q) p.coarse[q] = -1;
                } else {
                    p.kind = 1;
                    d.cf |= 1 << (4 + s);
                    const int par = t.parent[id];
                    if (par < 0) { err = "missing same-level neighbour of a root"; return false; }
                    if (par != cpar) {   // siblings are consecutive in Morton order: one 3 x 3 lookup per parent
                        cpar = par;
                        for (int dy = -1; dy <= 1; ++dy)
                            for (int dx = -1; dx <= 1; ++dx) {
                                const int q = nbr(par, dx, dy);
                                if (q == -1) { err = "R2 violated: coarse neighbourhood incomplete"; return false; }
                                cnb[(dy + 1) * 3 + (dx + 1)] = q < 0 ? -1 : q;
                            }
                    }
                    for (int q = 0; q < 9; ++q) p.coarse[q] = cnb[q];
                }
                d.side[s] = -1 - p.proxy;
                o.ptasks.push_back(p);
            }
        }
        o.leaves.push_back(d);
        if (rt.mask) o.rtasks.push_back(rt);
    }
    return true;
}
}  // namespace

bool plan_descriptors(const PatchTree& t, const std::vector<int32_t>& nb4, const std::vector<int32_t>& leaf_ids,
                      const Owners& owner, int world, int rank, int halo_mode, DescOut& out, std::string& err) {
    HostPool& pool = HostPool::get();
    const size_t nl = leaf_ids.size();
    // parts of at least ~1k leaves (a part's fixed cost is a few vector clears and the merge offsets)
    const int parts = pool.active() ? (int)std::max<size_t>(1, std::min<size_t>(4 * (size_t)pool.threads(), nl / 1024)) : 1;
    if (parts == 1) return describe_part(t, nb4, leaf_ids, 0, nl, owner, world, rank, halo_mode, out, err);
    static thread_local std::vector<DescOut> part_out;
    static thread_local std::vector<std::string> part_err;
    static thread_local std::vector<uint8_t> part_ok;
    std::vector<DescOut>& PO = part_out;   // the caller's scratch (parts run on the workers)
    std::vector<std::string>& PE = part_err;
    std::vector<uint8_t>& OK = part_ok;
    if ((int)PO.size() < parts) PO.resize(parts);
    PE.assign(parts, std::string());
    OK.assign(parts, 0);
    pool.run(parts, [&](int k) {
        OK[k] = describe_part(t, nb4, leaf_ids, nl * k / parts, nl * (k + 1) / parts, owner, world, rank, halo_mode,
                              PO[k], PE[k]);
    });
    for (int k = 0; k < parts; ++k)   // the first failing leaf in leaf order, as the serial loop
        if (!OK[k]) { err = PE[k]; return false; }
    // merge in part order: leaf indices and proxy numbers shifted by the preceding parts' counts
    std::vector<size_t> loff(parts + 1, 0), poff(parts + 1, 0), roff(parts + 1, 0);
    for (int k = 0; k < parts; ++k) {
        loff[k + 1] = loff[k] + PO[k].leaves.size();
        poff[k + 1] = poff[k] + PO[k].ptasks.size();
        roff[k + 1] = roff[k] + PO[k].rtasks.size();
    }
    out.leaves.resize(loff[parts]);
    out.ptasks.resize(poff[parts]);
    out.rtasks.resize(roff[parts]);
    pool.run(parts, [&](int k) {
        const int lo = (int)loff[k], po = (int)poff[k];
        LeafDesc* L = out.leaves.data() + loff[k];
        for (const LeafDesc& d0 : PO[k].leaves) {
            LeafDesc d = d0;
            for (int s = 0; s < 4; ++s)
                if (d.side[s] < 0) d.side[s] -= po;   // -1 - (p + po)
            *L++ = d;
        }
        ProxyTask* P = out.ptasks.data() + poff[k];
        for (const ProxyTask& p0 : PO[k].ptasks) {
            *P = p0;
            P->proxy += po;
            ++P;
        }
        RefluxTask* R = out.rtasks.data() + roff[k];
        for (const RefluxTask& r0 : PO[k].rtasks) {
            *R = r0;
            R->leaf += lo;
            ++R;
        }
    });
    return true;
}

}  // namespace amr
