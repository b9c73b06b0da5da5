// comm.h -- multi-GPU plumbing of one node: ownership of patches and the data
// exchanges a rank needs each stage.  World size 1 makes every
// hook a no-op.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/amr.h"

struct amr_ctx;

namespace amr {

struct Comm {
    int world = 1, rank = 0;
    void* nccl = nullptr;              // ncclComm_t
    std::vector<int32_t> owner;        // per slot (patch id), -1 free
    amr_status init(amr_ctx* c);
    void finalize(amr_ctx* c);
    bool owns(const amr_ctx* c, int id) const { return world == 1 || owner[id] == rank; }
    int owner_of(const amr_ctx* c, int id) const { return world == 1 ? 0 : owner[id]; }
    amr_status exchange_halos(amr_ctx* c, double* U);         // remote data read by local leaves / proxies
    amr_status exchange_fluxes(amr_ctx* c);                   // remote fine flux registers for reflux
    amr_status exchange_coarse(amr_ctx* c, double* U, int l); // remote coarse patches for new-patch prolongation
    amr_status exchange_children(amr_ctx* c, double* U);      // remote children for restriction (none: root-tree ownership)
    amr_status allreduce_max_u64(amr_ctx* c, unsigned long long* d);
    amr_status allreduce_sum4(amr_ctx* c, double* h4);
    amr_status allgather_flags(amr_ctx* c, std::vector<double>& eta, std::vector<uint8_t>& amb);
    amr_status agree_error(amr_ctx* c, int32_t* h_err4);
};

}  // namespace amr
