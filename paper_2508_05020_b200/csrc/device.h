// device.h -- plain-old-data descriptors shared by the host planner (api.cpp) and
// the sm_100a kernels (kernels.cu), plus the kernel launchers.
//
// HBM layout: three RK state buffers U[buf][slot][var][j][i] (fp64 SoA,
// 4 n^2 doubles per slot, var = rho, rho u, rho v, rho e); a proxy buffer of
// patch-shaped ghost strips P[proxy][var][j][i] for leaf sides that have no
// same-level neighbour (coarse/fine or physical boundary); flux registers
// F[slot][side][var][n] holding F-hat on coarse/fine sides.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace amr {

constexpr int kMaxLevels = 16;

enum Side { kW = 0, kE = 1, kS = 2, kN = 3 };

// One leaf patch in launch order.  side[s] >= 0: slot of the same-level
// neighbour (read from the stage input buffer); side[s] < 0: proxy -1-side[s].
struct LeafDesc {
    int32_t slot;
    int32_t level;
    int32_t side[4];
    int32_t cf;        // bits 0-3: side is the COARSE side of a C/F face; bits 4-7: FINE side
    int32_t pad;       // bit 0 covered patch (subcycling); bit 1 group member slots consecutive; halo_mode 2:
                       // bits 4-7 side neighbour owned by another rank, bits 8 + 3 s .. 10 + 3 s its rank
};

// Fill one proxy strip (the g columns / rows of a virtual neighbour that touch the leaf).
struct ProxyTask {
    int32_t proxy;     // proxy index
    int32_t slot;      // the leaf's own slot (physical BC source)
    int32_t side;      // Side of the leaf the strip lies on
    int32_t kind;      // 0 physical boundary, 1 coarse/fine prolongation
    int32_t level;     // leaf level l
    int32_t P, Q;      // leaf patch position at level l
    int32_t coarse[9]; // slots of the parent's 3x3 level-(l-1) neighbourhood [(dy+1)*3+(dx+1)], -1 outside
};

// Flux correction of one coarse leaf (O12): for each C/F side the two fine leaves
// across it (leaf indices into the flux registers), ordered along the side.
struct RefluxTask {
    int32_t leaf;      // index of the coarse leaf in the leaf list
    int32_t slot;      // its slot (flux registers are indexed by slot)
    int32_t level;
    int32_t mask;      // sides that are coarse sides of a C/F face
    int32_t fine[4][2];   // slots of the two fine leaves across each C/F side
};

// Restriction parent <- 4 children (O9); child c = a + 2b.
struct RestrictTask {
    int32_t parent;
    int32_t child[4];
};

// New patch initialised from its parent by prolongation (O8).
struct ProlongTask {
    int32_t slot;
    int32_t level;     // level of the new patch
    int32_t P, Q;
    int32_t coarse[9]; // parent's 3x3 neighbourhood at level-1 (centre = parent)
};

struct Geometry {
    int32_t n;                     // patch cells
    int32_t nc[2][kMaxLevels];     // cells per axis per level
    int32_t bc[4];                 // x-lo, x-hi, y-lo, y-hi
    double inv_dx[kMaxLevels], inv_dy[kMaxLevels];
    double dx[kMaxLevels], dy[kMaxLevels];
};

struct StageArgs {
    const LeafDesc* leaves;
    int32_t nleaves;
    int32_t tiles;             // tiles per side of a patch (n / T)
    const double* Uin;         // stage input U^(s-1)
    const double* Un;          // U^n
    double* Uout;              // U^(s)
    const double* proxy;
    double* freg;              // flux registers
    const double* dt;          // device scalar
    double a, b;               // U^(s) = a U^n + b (U^(s-1) + dt L)
    int32_t stage;             // 1, 2, 3
    int32_t div_order;
    int32_t characteristic;
    int32_t check;             // positivity check
    int32_t want_lambda;       // accumulate Lambda (stage 3)
    double gamma, eps;
    unsigned long long* lambda_bits;
    int32_t* err;              // [0] flag, [1] slot, [2] stage, [3] cell
    int32_t nslots;            // slots in each RK buffer (TMA tensor-map extent)
    int32_t nproxy;            // proxy patches allocated (TMA tensor-map extent)
    int32_t variant;           // amr_config.stage_kernel: 0 best, 1 per-tile fused, 2 unfused, 3 per-patch launches
    double* scratch;           // variant 2: intermediate fields (unfused_scratch_doubles)
    const LeafDesc* gleaves;   // n = 8, 16 Central4: members of 32 x 32 blocks [ngroups][(32/n)^2] (Morton order);
    int32_t ngroups;           //   leaves / nleaves then list only the leaves outside complete blocks
    int32_t prof;              // phase timing of the TMA kernel (AMR_PHASE_PROF, debug)
    int32_t lam0;              // subcycling: Lambda normalised to level 0 (S6); LeafDesc.pad bit 0 = covered patch;
                               // group tiles: pad bit 1 of member 0 = members in consecutive slots
    int32_t npeers;            // halo_mode 2: ranks whose pools are mapped (0 otherwise)
    const double* peer_in[8];  //   rank q's U^(s-1) as mapped here (host-side: tensor-map bases of the strip loads)
    Geometry geo;
};

// Subcycling (S3): one C/F side of a leaf whose F-hat is accumulated over a step; kind 1 coarse side, 2 fine side.
struct AccTask {
    int32_t slot, side, kind;
};

struct AuxArgs {
    const double* U;           // state read (ghost source / restriction source ...)
    const double* Uc;          // ghost kernel: coarse-level source of C/F prolongation (= U without subcycling)
    const double* Uold;        // subcycling: coarse level at the start of its step (nullptr: no time interpolation)
    double tfrac;              //   fraction of that step at the stage time (S2)
    int32_t lam0;              // subcycling: Lambda normalised to level 0 (S6)
    double* Uw;                // state written
    double* proxy;
    const double* freg;
    const double* dt;
    double b;                  // RK weight of the stage for the reflux
    int32_t stage;
    int32_t check;
    int32_t want_lambda;
    double gamma;
    double theta, coarsen_fraction;
    unsigned long long* lambda_bits;
    int32_t* err;
    Geometry geo;
};

// The work between two stage kernels (post_stage_kernel, one cooperative launch): reflux, restriction of every
// level (finest first), then -- np > 0 -- the ghost strips of the next stage's input (= this stage's output).
struct PostArgs {
    AuxArgs a;                           // U = Uw = the stage output; b, stage, want_lambda of the stage
    const RefluxTask* rtasks;
    int32_t nr;
    int32_t levels;
    const RestrictTask* rl[kMaxLevels];  // rl[l]: level l restricted into level l - 1
    int32_t nrl[kMaxLevels];
    const ProxyTask* ptasks;
    int32_t np;
    int32_t g;
};

// launchers (kernels.cu); each returns the CUDA error of the launch
cudaError_t launch_post_stage(const PostArgs& p, cudaStream_t s);
// peer_map 1: every world rank's address of offset 0 of an NCCL symmetric window (win: an ncclWindow_t), read on the
// device with ncclGetPeerPointer, into d_out[0 .. world)
cudaError_t launch_window_peer_ptrs(const void* win, int world, void** d_out, cudaStream_t s);
// peer_map 1: the stream-ordered cross-rank fence as an NCCL LSA barrier session in one CTA (devcomm: the host copy of
// an ncclDevComm made by ncclDevCommCreate with lsaBarrierCount >= 1; passed to the kernel by value)
cudaError_t launch_lsa_fence(const void* devcomm, cudaStream_t s);
cudaError_t launch_stage(int scheme, const StageArgs& a, cudaStream_t s);
cudaError_t launch_ghost(const ProxyTask* tasks, int ntasks, int g, const AuxArgs& a, cudaStream_t s);
cudaError_t launch_reflux(const RefluxTask* tasks, int ntasks, const AuxArgs& a, cudaStream_t s);
cudaError_t launch_restrict(const RestrictTask* tasks, int ntasks, const AuxArgs& a, cudaStream_t s);
cudaError_t launch_prolong(const ProlongTask* tasks, int ntasks, const AuxArgs& a, cudaStream_t s);
cudaError_t launch_lambda(const LeafDesc* leaves, int nleaves, const AuxArgs& a, cudaStream_t s);
cudaError_t launch_dt(double* dt, unsigned long long* lambda_bits, int32_t* err, double dt_fixed, double cfl,
                      cudaStream_t s);
cudaError_t launch_dt_dev(double* dt, unsigned long long* lambda_bits, int32_t* err, const double* params,
                          cudaStream_t s);
cudaError_t launch_set2(double* p, double a, double b, cudaStream_t s);
cudaError_t launch_dt_levels(double* dt, int levels, cudaStream_t s);
cudaError_t launch_accumulate(const AccTask* tasks, int ntasks, int n, const double* freg, double* acc, double w_coarse,
                              double w_fine, int assign_coarse, int assign_fine, cudaStream_t s);
cudaError_t launch_flags(const LeafDesc* leaves, int nleaves, const AuxArgs& a, double* maxeta, int32_t* amb,
                         cudaStream_t s);
// compact (slot, bits) list of the refine (bit 0) / coarsen (bit 1) requests; count is reset on the stream first
cudaError_t launch_flags_compact(const LeafDesc* leaves, int nleaves, const int32_t* sib, int nsib,
                                 const double* maxeta, double th, double tc, int top, int32_t* list, int32_t* count,
                                 cudaStream_t s);
cudaError_t launch_totals(const LeafDesc* leaves, int nleaves, const AuxArgs& a, double* partial, cudaStream_t s);

// slot-granular copies between a packed [npatch][per] buffer and per-slot arrays (state: per = 4 n^2;
// flux registers: per = 16 n)
cudaError_t launch_scatter(const double* packed, const int32_t* slots, int npatch, double* U, int per, cudaStream_t s);
cudaError_t launch_gather(const double* U, const int32_t* slots, int npatch, double* packed, int per, cudaStream_t s);
// slots[k] of the local buffer dst <- the same slot of peer peers[k]'s buffer (bases[peer] + off), `per` doubles each
cudaError_t launch_peer_pull(const int32_t* slots, const int32_t* peers, int n, const double* const* bases,
                             size_t off, double* dst, int per, cudaStream_t s);

// band items of the halo exchange (item = slot * 32 + code, comm.h): pack / unpack 16 n doubles per item between a
// buffer of the pool (U) and a packed array; pull the same bands of the same buffer (offset off in every pool) from
// each item's owner
cudaError_t launch_band_scatter(const double* packed, const int32_t* items, int nitem, double* U, int n, cudaStream_t s);
cudaError_t launch_band_gather(const double* U, const int32_t* items, int nitem, double* packed, int n, cudaStream_t s);
cudaError_t launch_band_pull(const int32_t* items, const int32_t* peers, int nitem, const double* const* bases,
                             size_t off, double* dst, int n, cudaStream_t s);

// unfused stage (variant 2): scratch doubles for nleaves patches; kernel launches per stage of a variant
size_t unfused_scratch_doubles(int n, int nleaves);
int stage_launches_per_stage(int variant, int nleaves);

// bytes of dynamic shared memory the stage kernel needs (for occupancy queries)
size_t stage_smem_bytes(int scheme, int n);

}  // namespace amr
