// comm.cpp -- see comm.h.
#include "comm.h"

#include "ctx.h"

namespace amr {

amr_status Comm::init(amr_ctx* c) {
    world = c->cfg.world_size;
    rank = c->cfg.rank;
    if (world != 1) {
        c->err = "world_size > 1 is not built into this library yet";
        return AMR_E_CONFIG;
    }
    return AMR_OK;
}
void Comm::finalize(amr_ctx*) {}
amr_status Comm::exchange_halos(amr_ctx*, double*) { return AMR_OK; }
amr_status Comm::exchange_fluxes(amr_ctx*) { return AMR_OK; }
amr_status Comm::exchange_coarse(amr_ctx*, double*, int) { return AMR_OK; }
amr_status Comm::exchange_children(amr_ctx*, double*) { return AMR_OK; }
amr_status Comm::allreduce_max_u64(amr_ctx*, unsigned long long*) { return AMR_OK; }
amr_status Comm::allreduce_sum4(amr_ctx*, double*) { return AMR_OK; }
amr_status Comm::allgather_flags(amr_ctx*, std::vector<double>&, std::vector<uint8_t>&) { return AMR_OK; }
amr_status Comm::agree_error(amr_ctx*, int32_t*) { return AMR_OK; }

}  // namespace amr
