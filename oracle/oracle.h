/*
 * oracle.h -- C API of the CPU ORACLE for the AMR compressible-Euler hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_2508_05020_b200/csrc, include/amr.h); neither includes the other.
 *
 * Definitions follow PAPER.md (arXiv 2508.05020) and SURVEY.md s8(c) O1-O18
 * (the readings A1-A42 are listed in DESIGN.md).  Every value is fp64; the
 * library is built with -O2 -ffp-contract=off and no fast-math.
 *
 * Return codes: 0 ok, 1 bad argument, 2 bad config, 3 non-physical state,
 * 4 mesh-validity violation.  orc_error() gives the message of the last error.
 */
#ifndef PAPER_ORACLE_H
#define PAPER_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double lo[2], hi[2];   /* domain [lo_x,hi_x] x [lo_y,hi_y]                 */
    int base[2];           /* level-0 cells per axis (multiple of n)           */
    int n;                 /* patch cells per side                              */
    int levels;            /* total levels including the base (A22)            */
    double gamma;          /* ratio of specific heats (1.4)            */
    int bc[4];             /* x-lo, x-hi, y-lo, y-hi: 0 periodic, 1 transmissive, 2 reflective */
    int scheme;            /* 0 Central4 (Eq. 8/9), 1 WENO5-JS + Rusanov (Eq. 11-12) */
    int characteristic;    /* WENO only: 1 characteristic (O10), 0 component-wise */
    int div_order;         /* 4: Eq. 9 flux form, 2: plain difference          */
    double weno_eps;       /* 1e-6 (A5)                                         */
    double theta;          /* refinement threshold (BJ configs[0]: 0.1)        */
    double coarsen_frac;   /* coarsen when eta < theta*coarsen_frac (A20: 0.25) */
    int coarsen_rule;      /* 0 R2-exact prose rule, 1 Alg. 2 literal  */
    int check_positivity;  /* 1: a non-physical leaf state after a stage is an error; 0: not checked
                              (the white-noise sweep is a throughput config, not physics) */
    int reflux;            /* 1: O12 flux correction at coarse/fine faces (default); 0: TEST-ONLY control that
                              omits it (the pins show conservation then fails) */
} orc_config;

void*       orc_create(const orc_config* cfg);
void        orc_destroy(void* h);
const char* orc_error(void* h);

/* tree (O3), canonical order (level, Q, P) */
int orc_num_patches(void* h);
int orc_get_tree(void* h, int cap, int* level, int* P, int* Q, int* leaf, int* nchild_leaf);
int orc_validate(void* h);

/* fields: U[4][n][n] conserved, row-major in (j, i) */
int orc_set_patch(void* h, int l, int P, int Q, const double* U);
int orc_get_patch(void* h, int l, int P, int Q, double* U);
int orc_restrict_all(void* h);                         /* O9 */
int orc_lambda(void* h, double* lam);                  /* O13; NaN if any leaf cell gives NaN */
int orc_lambda_subcycled(void* h, double* lam);        /* S6: per-leaf value divided by 2^l */
int orc_totals(void* h, double* out4);                 /* O18 */
int orc_step(void* h, double dt, double cfl, double* dt_used);   /* O11 */
/* O11 stage 1 alone (U <- U + dt L(U), reflux with b_1 = 1, restriction): the unit the reflux-placement pin
 * takes apart */
int orc_stage1(void* h, double dt);
/* OpenMP over patches: results are independent of the thread count */
void orc_set_num_threads(int n);
int  orc_get_max_threads(void);
/* NEXT #4: one level-0 step of Berger-Colella time subcycling (dt_l = dt0 / 2^l, readings S1-S6 in oracle.cpp
 * and DESIGN.md s3b); dt0 <= 0: dt0 = cfl / max over leaves of the level-0-normalised wave speed */
int orc_step_subcycled(void* h, double dt0, double cfl, double* dt_used);

/* flags (O6) for every active patch, canonical order */
int orc_flags(void* h, int cap, double* maxeta, unsigned char* refine,
              unsigned char* coarsen, unsigned char* ambiguous);
/* regrid (O4, O5, O8, O9) with given requests keyed by (l,P,Q) */
int orc_regrid_with_requests(void* h, int m, const int* l, const int* P, const int* Q,
                             const unsigned char* refine, const unsigned char* coarsen,
                             int* n_refined, int* n_coarsened);
int orc_regrid(void* h, int* n_refined, int* n_coarsened);

/* unit-level access for pins */
int orc_ghost_tile(void* h, int l, int P, int Q, int g, double* tile /* [4][n+2g][n+2g] */);
int orc_rhs(void* h, int l, int P, int Q, double* Lout /* [4][n][n] */);
void orc_cons2prim(double gamma, const double* U, double* W);
void orc_prim2cons(double gamma, const double* W, double* U);
void orc_euler_flux_x(double gamma, const double* U, double* F);
void orc_rusanov_x(double gamma, const double* UL, const double* UR, double* F);
double orc_weno5(const double* v /* 5 */, double eps);
void orc_eigen_x(double gamma, const double* WL, const double* WR, double* Lm /*16*/, double* Rm /*16*/);
void orc_face_flux_x(const orc_config* cfg, const double* cells /* [6][4] cells i-2..i+3 */, double* F);
double orc_mc(double a, double b);

#ifdef __cplusplus
}
#endif
#endif
