/*
 * amr.h -- C ABI of the B200-native AMR compressible-Euler hot path
 *          (arXiv 2508.05020, "Task-Based Programming for Adaptive Mesh Refinement
 *           in Compressible Flow Simulations").
 *
 * The library advances a 2D patch-based quadtree mesh of the compressible Euler
 * equations for a calorically perfect gas (PAPER.md s2.1, Eq. 1-7) with
 * Central4 (Eq. 8/9) or WENO5-JS + Rusanov (Eq. 11-12)
 * fluxes and SSP-RK3, on patches of one fixed size kept valid by
 * rules R1/R2 through Alg. 1 (refinement) and Alg. 2
 * (coarsening, prose P:L259).  Readings where the paper is silent
 * (ghost fill, prolongation, restriction, flux correction, the indicator) are
 * DESIGN.md s3.
 *
 * Conventions (all entry points):
 *  - Every function returns amr_status and never throws or aborts.
 *  - Host pointers are owned by the caller; the library copies during the call
 *    and keeps none.  The library owns amr_ctx and all device memory it
 *    allocates; a caller-provided device `pool` stays owned by the caller and
 *    must outlive the ctx.
 *  - Conserved state arrays are fp64, layout [patch][var][j][i] with var order
 *    (rho, rho u, rho v, rho e) (Eq. 10 vector U; Fig. 9 CVARS) and i
 *    the fastest (x) index, n = patch_cells.
 *  - `tree_index` is a position in the canonical patch order returned by
 *    amr_get_patch_tree: sorted by (level, j, i).  Slots are internal.
 *  - A ctx is not thread-safe: one ctx per rank / GPU.  amr_create, amr_set_state,
 *    amr_step, amr_regrid and amr_diagnostics are collective over the ranks.
 *  - AMR_E_CUDA and AMR_E_COMM are sticky: afterwards every call except
 *    amr_destroy / amr_last_error returns AMR_E_STATE.
 */
#ifndef PAPER_2508_05020_AMR_H
#define PAPER_2508_05020_AMR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMR_ABI_VERSION 5

typedef struct amr_ctx amr_ctx;   /* opaque */

typedef enum {
    AMR_OK = 0,
    AMR_E_ARG = 1,          /* bad argument (null pointer, index out of range)          */
    AMR_E_CONFIG = 2,       /* invalid configuration (mirrors SPEC exit code 2)         */
    AMR_E_NONPHYSICAL = 3,  /* rho <= 0, p <= 0 or non-finite (SPEC exit 3)     */
    AMR_E_MESH = 4,         /* mesh-validity violation R1/R2 (SPEC exit 4)              */
    AMR_E_CAPACITY = 5,     /* slot capacity exceeded; mesh unchanged          */
    AMR_E_CUDA = 6,         /* CUDA runtime error (sticky)                              */
    AMR_E_COMM = 7,         /* NCCL error (sticky)                                      */
    AMR_E_STATE = 8         /* ctx unusable after a sticky error, or wrong call order   */
} amr_status;

typedef enum { AMR_BC_PERIODIC = 0, AMR_BC_TRANSMISSIVE = 1, AMR_BC_REFLECTIVE = 2 } amr_bc;
typedef enum { AMR_CENTRAL4 = 0, AMR_WENO5_RUSANOV = 1 } amr_scheme;
typedef enum { AMR_COARSEN_R2_EXACT = 0, AMR_COARSEN_ALG2_LITERAL = 1 } amr_coarsen_rule;

/* comm_backend 2 (multi-process test transport): collectives supplied by the caller, e.g. over a torch gloo
 * group.  allgather: every rank contributes `bytes` from `send`; `recv` receives world_size x bytes in rank order.
 * barrier: returns once every rank has called it.  Both return 0 on success.  Lets several processes share ONE GPU
 * (NCCL refuses that) so that the CUDA-IPC peer mapping of halo_mode 1 / 2 is exercised without a second GPU. */
typedef struct {
    int32_t (*allgather)(const void* send, uint64_t bytes, void* recv, void* user);
    int32_t (*barrier)(void* user);
    void* user;
} amr_host_comm;

typedef struct {
    int32_t dim;                  /* 2, or 1 for the strip embedding of 1D problems (A23)   */
    double lo[2], hi[2];          /* domain [lo_x,hi_x] x [lo_y,hi_y]                        */
    int32_t base_cells[2];        /* level-0 cells per axis; multiples of patch_cells        */
    int32_t patch_cells;          /* n: 8, 16, 32 or 64 ("same grid size")           */
    int32_t num_levels;           /* total levels including the base (A22)                  */
    int32_t ratio;                /* refinement ratio; must be 2 (quadtree)         */
    double gamma;                 /* ratio of specific heats (1.4)                  */
    int32_t bc[4];                /* amr_bc for x-lo, x-hi, y-lo, y-hi; periodic on both or neither side */
    int32_t scheme;               /* amr_scheme                                              */
    int32_t weno_characteristic;  /* 1: characteristic variables, 0: component-wise */
    int32_t div_order;            /* 4: Eq. 9 flux form, 2: plain difference                 */
    double weno_eps;              /* WENO epsilon (A5: 1e-6)                                 */
    double refine_threshold;      /* theta: refine where eta = dx |grad rho| / rho > theta  */
    double coarsen_fraction;      /* coarsen where all children's eta < theta * fraction    */
    int32_t coarsen_rule;         /* amr_coarsen_rule (A16)                                  */
    int32_t max_patches;          /* slot capacity per rank (active patches incl. non-leaf) */
    void* pool;                   /* optional device buffer for the 3 RK state buffers; NULL -> library allocates */
    uint64_t pool_bytes;          /* size of `pool`; see amr_query_pool_bytes                */
    void* cuda_stream;            /* cudaStream_t to launch on (e.g. torch's current stream); NULL -> library stream */
    int32_t device;               /* CUDA device ordinal; -1 -> current device               */
    int32_t world_size, rank;     /* ranks of one node, one GPU each; 1 / 0 for single GPU   */
    const void* nccl_unique_id;   /* 128-byte ncclUniqueId broadcast by the caller (world_size > 1) */
    int32_t check_positivity;     /* 1: amr_step checks rho, p > 0 and finiteness (default)  */
    int32_t use_graphs;           /* 1: amr_step / amr_steps replay one step as a CUDA graph (captured per position
                                     of U^n in the RK buffer rotation, once a mesh plan has served 3 steps;
                                     re-captured after mesh changes); single rank with kernel timing off only */
    int32_t comm_backend;         /* world_size > 1: 0 NCCL (nccl_unique_id = ncclUniqueId); 1 in-process
                                     loopback of virtual ranks on one GPU, one host thread each
                                     (test-only; nccl_unique_id = 128-byte group key string); 2 one process
                                     per rank with caller-supplied host collectives (host_comm; test-only:
                                     data through host memory, peer pools through CUDA IPC)      */
    int32_t stage_kernel;         /* stage kernel organisation (NEXT #1 fusion study): 0 default (Central4 with
                                     n >= 32: persistent TMA-pipelined fused kernel, else 1); 1 fused, one CTA per
                                     tile with a cp.async halo gather; 2 unfused: four kernels per stage with the
                                     primitives and face fluxes through HBM; 3 one launch of kernel 1 per leaf */
    int32_t subcycle;             /* 1: Berger-Colella time subcycling (NEXT #4; DESIGN.md s3b S1-S6): level l takes
                                     2^l steps of dt_0 / 2^l per amr_step, C/F ghosts interpolated in time, fluxes
                                     refluxed with quadrature-weighted registers; dt / cfl of amr_step refer to
                                     level 0 and amr_diagnostics' lambda is normalised to level 0.  Any world_size
                                     (per-level face / coarse-source / register exchanges);
                                     a non-physical step is reported (AMR_E_NONPHYSICAL) but only level 0 rolls back */
    int32_t halo_mode;            /* world_size > 1, halo and flux-register exchanges (NEXT #3): 0 pack kernel +
                                     transport point-to-point (NCCL send/recv, or loopback copies) + unpack kernel;
                                     1 peer pull: at amr_create every rank maps every other rank's state pool (CUDA
                                     IPC handles exchanged over NCCL; directly for loopback virtual ranks), and each
                                     exchange is a stream-ordered cross-rank fence (a one-word NCCL allreduce, or
                                     CUDA events between loopback streams) followed by ONE kernel that loads the
                                     needed slots from the owners' pools over NVLink into the local pool;
                                     2 (stage_kernel 0 / 1; Central4 with patch_cells < 32 needs stage_kernel 1, the
                                     per-tile kernel; <= 8 ranks; else AMR_E_CONFIG) as 1, but the stage kernel itself
                                     loads the 4-wide face strips of remote neighbours from the owners' pools (TMA /
                                     cp.async over NVLink), so before a stage only the coarse sources of C/F ghosts
                                     are pulled (the halo transfer overlaps the compute).  The halo lists of modes
                                     0 / 1 move band items (the facing 4-wide strips), not whole patches.
                                     Regrid exchanges (coarse sources, migration, flags) use the transport in all
                                     modes */
    const amr_host_comm* host_comm;   /* comm_backend 2: the caller's collectives (kept alive until destroy) */
    int32_t peer_map;             /* halo_mode 1 / 2 over NCCL (comm_backend 0): how every rank's state pool and
                                     flux-register buffer are mapped into this process.  0 CUDA IPC handles exchanged
                                     by an NCCL byte-sum allreduce; 1 NCCL symmetric memory windows: both buffers are
                                     allocated by the library with ncclMemAlloc (cfg.pool must be NULL), registered
                                     with ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC), and every peer's address
                                     is taken on the device from the window with ncclGetPeerPointer (NCCL's
                                     load/store-accessible device API, nccl_device.h); with NCCL's device
                                     communicator (ncclDevCommCreate, one LSA barrier) and every rank in one LSA
                                     team, the stage fence is an ncclLsaBarrierSession kernel instead of the
                                     one-word allreduce (ncclDevCommCreate failing -> AMR_E_COMM at amr_create);
                                     ABI 5 */
} amr_config;

/* Patch metadata as in Fig. 2; links are tree indices, -1 = none
 * (nbr order N, E, S, W, NE, SE, SW, NW; -1 also for a physical boundary). */
typedef struct {
    int32_t level, i, j;
    int32_t parent;
    int32_t child[4];             /* child index a + 2b: SW, SE, NW, NE                      */
    int32_t nbr[8];
    int32_t owner;                /* rank that holds the patch data                          */
    uint8_t leaf, refine_req, coarsen_req, ambiguous;
} amr_patch_desc;

typedef struct {
    int64_t launches;             /* kernels launched by this ctx since the last reset       */
    int64_t stage_launches;       /* launches of the fused stage kernel                      */
    double  stage_ms;             /* sum of CUDA-event durations of the timed stage launches */
    int64_t stage_timed;          /* number of stage launches with a duration in stage_ms    */
    int64_t stage_cells;          /* leaf cell-updates done by those timed launches          */
    double  stage_bytes;          /* algorithmic HBM bytes of those launches  */
    int64_t steps;                /* committed steps                                         */
    int64_t leaf_cells;           /* current leaf cells owned by this rank                   */
    int64_t leaves, patches;      /* current leaf / active patch counts (whole mesh)         */
    int64_t proxies;              /* ghost strips filled per stage (C/F or physical BC sides) */
    double  sim_time;             /* simulated time advanced by committed steps since the last reset
                                     (summed on the device; reading it synchronises the stream) */
} amr_stats;

/* Library / ABI version; never fails. */
int32_t amr_abi_version(void);

/* Fill *cfg with defaults (2D, gamma 1.4, periodic, Central4, div 4, eps 1e-6,
 * theta 0.1, fraction 0.25, R2-exact, max_patches 4096, checks on).  AMR_E_ARG on NULL. */
amr_status amr_default_config(amr_config* cfg);

/* Bytes needed in `pool` for cfg (3 RK buffers x max_patches x 4 x n^2 x 8). */
amr_status amr_query_pool_bytes(const amr_config* cfg, uint64_t* bytes);

/* Create the mesh: level-0 scaffold of roots (R1), all values zero.
 * AMR_E_CONFIG: base not divisible by n, ratio != 2, n < 8, levels < 1, periodic on
 * one side only, bad scheme / div order.  AMR_E_CAPACITY: roots exceed max_patches. */
amr_status amr_create(const amr_config* cfg, amr_ctx** out);
void amr_destroy(amr_ctx* ctx);

/* Set the conserved state of `npatch` active patches (tree_index[k], data
 * U + k * 4 n^2), then restrict (fine -> coarse averaging, O9) so
 * covered cells equal their children's mean.  Patches owned by other ranks are
 * ignored.  AMR_E_ARG: bad index. */
amr_status amr_set_state(amr_ctx* ctx, int32_t npatch, const int32_t* tree_index, const double* U);

/* Initial-condition callback: fill U [4][ncell] (conserved, var-major) at the ncell points (x[c], y[c]). */
typedef void (*amr_ic_fn)(int32_t ncell, const double* x, const double* y, double* U, void* user);

/* Sample every locally owned active patch (leaves and covered patches) at its cell centres through `fn`
 * (one call per patch, ncell = n^2 points in [j][i] order), then restrict as amr_set_state does (A33 point
 * values).  `user` is passed through.  AMR_E_ARG: fn is NULL. */
amr_status amr_set_state_fn(amr_ctx* ctx, amr_ic_fn fn, void* user);

/* As amr_set_state, with U a DEVICE pointer (e.g. a torch CUDA tensor) on the ctx's device. */
amr_status amr_set_state_device(amr_ctx* ctx, int32_t npatch, const int32_t* tree_index, const double* dU);

/* As amr_get_state, into a DEVICE buffer dU_out (npatch x 4 n^2 doubles). */
amr_status amr_get_state_device(amr_ctx* ctx, int32_t npatch, const int32_t* tree_index, double* dU_out);

/* Copy the conserved state of `npatch` patches to host U_out (same layout).
 * Patches owned by other ranks are left untouched. */
amr_status amr_get_state(amr_ctx* ctx, int32_t npatch, const int32_t* tree_index, double* U_out);

/* One SSP-RK3 step (O11) of the whole composite mesh with one
 * global dt: dt > 0 is used as given, else dt = cfl / Lambda with Lambda the max over
 * leaf cells of (|u|+c)/dx + (|v|+c)/dy (O13).  Each stage: ghost fill (O7/O8),
 * fused reconstruction + Riemann flux + divergence + RK update over all leaves,
 * flux correction at coarse/fine faces (O12), restriction (O9).
 * dt_used may be NULL: then (and with check_positivity = 0) the call does not
 * synchronise with the device.  AMR_E_NONPHYSICAL: the step is NOT committed
 * (U^n unchanged); amr_last_error names level, patch and stage. */
amr_status amr_step(amr_ctx* ctx, double dt, double cfl, double* dt_used);

/* nsteps steps queued without host synchronisation in between: each step is amr_step's arithmetic, but errors are
 * reported LATE and nothing is rolled back.  A non-physical state (check_positivity) or a non-finite dt detected on
 * the device in any of the queued steps is returned as AMR_E_NONPHYSICAL by the next amr_sync (or by the next amr_step,
 * which then does not commit its own step either); the mesh then holds the state advanced by all nsteps steps (the steps
 * queued after the failing one ran on its non-physical data) -- unlike amr_step, which keeps U^n on failure.  Use
 * amr_step where a failed step must leave U^n intact. */
amr_status amr_steps(amr_ctx* ctx, int32_t nsteps, double dt, double cfl);

/* Wait for all queued work; returns a deferred AMR_E_NONPHYSICAL (of amr_steps) if any, without rollback. */
amr_status amr_sync(amr_ctx* ctx);

/* Evaluate the refinement indicator (BJ configs[0]: eta = dx |grad rho| / rho,
 * DESIGN.md O6) on the ghost-filled state and write, per active patch in canonical
 * order, its max eta (leaves; NaN for patches whose children are not all leaves,
 * the children's max otherwise) and bits: 1 refine_req, 2 coarsen_req, 4 ambiguous
 * (|eta - threshold| <= 1e-9 relative).  cap >= number of active patches. */
amr_status amr_get_flags(amr_ctx* ctx, int32_t cap, double* maxeta, uint8_t* bits);

/* Regrid: flags (evaluated and compacted on the device into a (slot, refine|coarsen) request list; on N > 1
 * ranks the lists are exchanged, so the host handles O(requests), not O(patches)), refinement pass (Alg. 1 with
 * recursion), coarsening pass (Alg. 2 / prose rule, finest level first), R1/R2 validation, prolongation of new
 * patches, restriction, repartition and migration on N > 1.  The requests equal amr_get_flags' bits 1 and 2.
 * *n_refined / *n_coarsened (may be NULL) receive the numbers of patches created / deleted.
 * AMR_E_CAPACITY leaves the mesh unchanged. */
amr_status amr_regrid(amr_ctx* ctx, int32_t* n_refined, int32_t* n_coarsened);

/* Regrid with externally given requests (bits as in amr_get_flags, indexed by
 * tree_index of the current tree); used by the lockstep parity protocol (A32). */
amr_status amr_regrid_with_flags(amr_ctx* ctx, int32_t n, const int32_t* tree_index, const uint8_t* bits,
                                 int32_t* n_refined, int32_t* n_coarsened);

/* The active patches in canonical order; *count = number of patches.  cap may be
 * smaller than the count (then only *count is meaningful and AMR_E_ARG returned). */
amr_status amr_get_patch_tree(amr_ctx* ctx, amr_patch_desc* out, int32_t cap, int32_t* count);

/* Totals sum over leaf cells of U_k dx dy (O18; per-patch sums on the device,
 * combined on the host in canonical order in long double) and the current Lambda. */
amr_status amr_diagnostics(amr_ctx* ctx, double totals[4], double* lambda_max);

/* Kernel-level statistics; timing of the fused stage kernel with CUDA events on
 * the launch stream is on while amr_set_kernel_timing(ctx, 1). */
amr_status amr_set_kernel_timing(amr_ctx* ctx, int32_t enable);
amr_status amr_get_stats(amr_ctx* ctx, amr_stats* out);
amr_status amr_reset_stats(amr_ctx* ctx);

/* Fill out128 with a fresh ncclUniqueId (rank 0; the caller broadcasts it, e.g. through a torch
 * process group).  Loads torch's libnccl.so.2 (or $AMR_NCCL_LIB) at run time.  AMR_E_COMM if NCCL is
 * unavailable. */
amr_status amr_nccl_unique_id(void* out128);

/* Message of the last failing call on ctx (valid until the next call); ctx may be NULL. */
const char* amr_last_error(const amr_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
