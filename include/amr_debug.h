/*
 * amr_debug.h -- TEST-ONLY entry points of libamr.so: host-only planning calls (no CUDA call is made) and
 * one self-test of the NCCL transport (the only call here that touches the GPU).
 *
 * They expose the multi-rank plan the library computes from the replicated patch tree
 * (SURVEY.md s8(e)): the root-tree Morton partition and the per-peer exchange lists, so the N > 1
 * host logic can be checked on CPU (world-size-2 gloo tests) without a GPU.
 * Indices are canonical tree indices ((level, j, i) order, as amr_get_patch_tree).
 */
#ifndef PAPER_2508_05020_AMR_DEBUG_H
#define PAPER_2508_05020_AMR_DEBUG_H
#include "amr.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct amr_plan amr_plan;

/* Root scaffold of cfg (validated as amr_create; the device fields are ignored). */
amr_status amr_plan_create(const amr_config* cfg, amr_plan** out);
void amr_plan_destroy(amr_plan* p);
/* Apply refine (bit 1) / coarsen (bit 2) requests exactly as amr_regrid_with_flags does to the tree. */
amr_status amr_plan_regrid(amr_plan* p, int32_t n, const int32_t* tree_index, const uint8_t* bits);
/* Patch metadata in canonical order (owner = rank under a world_size partition). */
amr_status amr_plan_tree(amr_plan* p, int32_t world_size, amr_patch_desc* out, int32_t cap, int32_t* count);
/* Exchange lists of `rank`: kind 0 halo (per stage), 1 flux registers; subcycling (plan_subcycle) for level l:
 * kind 2 + 3 l face halo of a level-l stage, 3 + 3 l coarse sources of its C/F ghosts, 4 + 3 l accumulated
 * registers of the fine leaves its reflux reads.  counts_*[world] per peer;
 * the index arrays hold the peers' lists back to back (capacity cap each).  The halo lists (kind 0 and the
 * subcycling face lists) move BAND ITEMS -- the 4-wide strip of a face neighbour facing the reader, whole patches
 * (all row bands) of coarse sources -- and are reported as the distinct tree indices they touch; kind + 1000 reports
 * the items themselves as tree_index * 32 + code (code < 16: row band 4 code .. 4 code + 3; 16: columns 0..3;
 * 17: columns n-4..n-1). */
amr_status amr_plan_exchange(amr_plan* p, int32_t world_size, int32_t rank, int32_t kind, int32_t* send_counts,
                             int32_t* send_index, int32_t* recv_counts, int32_t* recv_index, int32_t cap);

/* Host plan work of `rank` at a regrid (what every rank computes: partition, its own and boundary roots, leaf launch
 * order, face-neighbour table, halo and flux-register lists), averaged over reps runs on this CPU.  ms[7]: partition,
 * roots, leaf order, face neighbours, halo lists, flux lists, total (milliseconds); counts[4]: active patches,
 * rank's leaves, halo items received, halo items sent.  Host only. */
amr_status amr_plan_profile(amr_plan* p, int32_t world, int32_t rank, int32_t reps, double* ms, int64_t* counts);

/* The plan phases of a regrid's build_plan (leaf launch order, face-neighbour table, leaf descriptors with their proxy
 * strip and reflux tasks) of `rank` under a world_size partition, computed serially and in parts on the library's armed
 * host thread pool (AMR_HOST_THREADS), reps times each.  ms[6]: serial leaf order, neighbours, descriptors, then the
 * same pooled (milliseconds per run, this CPU); counts[4]: leaves, proxy tasks, reflux tasks, pool threads; *equal = 1
 * iff the two plans agree byte for byte.  AMR_E_MESH if the tree fails the descriptor checks.  Host only. */
amr_status amr_plan_build_check(amr_plan* p, int32_t world, int32_t rank, int32_t halo_mode, int32_t reps, double* ms,
                                int64_t* counts, int32_t* equal);

/* NCCL self-test (needs a GPU and torch's libnccl.so.2): a ONE-rank communicator from the 128-byte unique id
 * (amr_nccl_unique_id) drives the data path's NCCL transport -- grouped send/recv to self (the halo / flux /
 * migration exchange call pattern), the four allreduce kinds (Lambda max-u64, max-f64, sum-f64 totals, max-i32
 * errors), the peer-table byte-sum allreduce and the one-word fence -- and checks the results (bytes received =
 * bytes sent; 1-rank reductions are the identity); then the symmetric-window mapping of peer_map 1 (ncclMemAlloc,
 * ncclCommWindowRegister, the device-side ncclGetPeerPointer, whose address must alias the buffer; msg then holds
 * "window ok"), and with ncclDevCommCreate present three peer_map 1 fences as ncclLsaBarrierSession kernels ("lsa
 * barrier fence ok").  Returns AMR_OK, AMR_E_COMM (message in msg, NUL-terminated,
 * at most msg_cap bytes) or AMR_E_CUDA. */
amr_status amr_debug_nccl_selftest(const void* nccl_unique_id, char* msg, int32_t msg_cap);

#ifdef __cplusplus
}
#endif
#endif
