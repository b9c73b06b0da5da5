// kernels.cu -- sm_100a kernels of the AMR compressible-Euler hot path.
//
// The fused stage kernel is the GPU analogue of the paper's task fusion:
// one launch over the leaf-patch list does, per patch tile, the halo gather
// (same-level neighbours read in place, proxies for C/F and physical sides),
// cons->prim (Eq. 4-7), reconstruction (Eq. 8 Central4 or WENO5-JS),
// the face flux (central, or Rusanov Eq. 11-12), the flux divergence (Eq. 9 in
// flux form), the SSP-RK3 combination (Fig. 9 ssprk3Stage), the positivity
// check, flux registers for the coarse/fine correction and, at stage 3, the
// per-patch max wave speed (warp shuffles + one atomic per warp).
// Auxiliary kernels: ghost/proxy fill (O7/O8), reflux (O12), restriction (O9),
// prolongation of new patches (O8), flags (O6), Lambda, totals (O18).
// Readings and rewrites (A41: single-division WENO weights, reciprocal dx,
// FMA contraction) are listed in DESIGN.md.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cuda.h>
#include <cooperative_groups.h>

#include <algorithm>

#include "device.h"
#ifdef AMR_HAVE_NCCL_H
#include <nccl.h>
#include <nccl_device.h>   // ncclGetPeerPointer (symmetric memory windows, peer_map 1)
#endif

namespace amr {
namespace cg = cooperative_groups;
namespace {

constexpr int kBcPeriodic = 0, kBcTransmissive = 1, kBcReflective = 2;

// ---------------------------------------------------------------- fast fp64 reciprocal / square root (A41)
// Branch-free replacements for IEEE division and sqrt on the hot path (no slow-path calls): MUFU seed + Newton
// steps, <= 1 ulp for the positive normal arguments the scheme produces (rho, c^2, p, WENO weight sums); a
// non-physical argument (<= 0, NaN) yields NaN or inf, which the positivity check reports.
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    // r (1 + e + e^2) with e = 1 - x r: relative error e^3 (the seed's e ~ 2^-23), below half an ulp before the
    // final rounding -- three DFMA instead of two Newton steps' four
    double e = fma(-x, r, 1.0);
    e = fma(e, e, e);
    return fma(r, e, r);
}
// 1/sqrt(x): seed y, t = x y^2 - 1, y (1 - t/2 + 3 t^2/8) (relative error O(t^3) below half an ulp, then rounding)
__device__ __forceinline__ double fast_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double t = fma(x * y, y, -1.0);
    return fma(y, t * fma(0.375, t, -0.5), y);
}
// sqrt(x) = x / sqrt(x) (A41: <= 2 ulp for positive normal x, scripts/rcp_check.cu; 0, negative and NaN give NaN)
__device__ __forceinline__ double fast_sqrt(double x) { return x * fast_rsqrt(x); }

__device__ __forceinline__ double wave_speed(double r, double m, double w, double E, double g, double idx,
                                             double idy) {
    double ir = fast_rcp(r);
    double u = m * ir, v = w * ir;
    double p = (g - 1.0) * (E - 0.5 * (m * u + w * v));
    double c = fast_sqrt(g * p * ir);
    return (fabs(u) + c) * idx + (fabs(v) + c) * idy;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

__device__ __forceinline__ void report_error(int32_t* err, int slot, int stage, int cell) {
    if (atomicCAS(err, 0, 1) == 0) {
        err[1] = slot;
        err[2] = stage;
        err[3] = cell;
    }
}

// S5 positivity check and, at the last stage, the O13 wave speed of a new leaf state from ONE reciprocal of rho
// (A41: the check's velocities use the <= 1 ulp reciprocal of cons->prim instead of two IEEE divisions with their
// slow-path calls; the speed is wave_speed()'s arithmetic)
__device__ __forceinline__ void leaf_check(double r, double m, double w, double E, double g, double idx, double idy,
                                           bool check, bool want_lambda, int lam_shift, int32_t* err, int slot,
                                           int stage, int cell, unsigned long long& lam) {
    const double ir = fast_rcp(r);
    const double u = m * ir, v = w * ir;
    const double p = (g - 1.0) * (E - 0.5 * (m * u + w * v));
    if (check && !(r > 0.0 && p > 0.0 && isfinite(r) && isfinite(m) && isfinite(w) && isfinite(E) && isfinite(u) &&
                   isfinite(v) && isfinite(p)))
        report_error(err, slot, stage, cell);
    if (want_lambda) {
        const double c = fast_sqrt(g * p * ir);
        double sp = (fabs(u) + c) * idx + (fabs(v) + c) * idy;
        if (lam_shift) sp = ldexp(sp, -lam_shift);   // subcycling: level-0-normalised (S6)
        const unsigned long long b = (unsigned long long)__double_as_longlong(sp);
        lam = b > lam ? b : lam;
    }
}

// ---------------------------------------------------------------- reconstruction + flux
// Both WENO5-JS interpolations at one face from the 6 stencil values w0..w5 (cells i-2 .. i+3): the left-biased
// value from (w0..w4) and the right-biased one from (w5..w1) (A2), rewritten exactly in real arithmetic (A41):
// - everything from the first differences d_ij = w_i - w_j: the second differences T of the smoothness indicators
//   (shared by the two sides), their one-sided u terms, and the candidate stencils as corrections to the
//   face-adjacent cell (w2 left, w3 right) -- the result is w2 + sum_k omega_k (q_k - w2), since sum omega_k = 1;
// - the linear weights (1, 10, 5)/16 folded into the corrections and the normalisation (the 1/16 cancels);
// - every indicator evaluated scaled by 4: S = (4 eps + 13/3 T^2 + u^2)^2 = 16 (eps + beta)^2, a common factor of all
//   weights that cancels in the normalisation (the 13/3 on the four shared T terms), and one weight product per candidate
//   (omega_k ~ d_k prod_{j != k} S_j, one reciprocal per side).
__device__ __forceinline__ void weno5_pair(double w0, double w1, double w2, double w3, double w4, double w5,
                                           double eps4, double& left, double& right) {
    const double d01 = w0 - w1, d12 = w1 - w2, d23 = w2 - w3, d34 = w3 - w4, d45 = w4 - w5;
    // corrections q_k - w2 (left) / r_k - w3 (right) times the linear weights 1, 10, 5 (x 16):
    // left (3 d01 - 7 d12)/8, -10 (d12 + 3 d23)/8, 5 (d34 - 5 d23)/8; right (7 d34 - 3 d45)/8, 10 (3 d23 + d34)/8,
    // 5 (5 d23 - d12)/8
    const double q0 = fma(0.375, d01, -0.875 * d12), q1 = fma(-1.25, d12, -3.75 * d23);
    const double q2 = fma(0.625, d34, -3.125 * d23);
    const double r0 = fma(0.875, d34, -0.375 * d45), r1 = fma(3.75, d23, 1.25 * d34);
    const double r2 = fma(3.125, d23, -0.625 * d12);
    // second differences (shared) and one-sided terms: T_a = w0 - 2 w1 + w2 ... T_d = w3 - 2 w4 + w5
    const double Ta = d01 - d12, Tb = d12 - d23, Tc = d23 - d34, Td = d34 - d45;
    constexpr double c13 = 13.0 / 3.0;   // (13/3) T^2 on the four shared terms, u^2 unscaled on the six one-sided ones
    const double Aa = fma(c13 * Ta, Ta, eps4), Ab = fma(c13 * Tb, Tb, eps4);
    const double Ac = fma(c13 * Tc, Tc, eps4), Ad = fma(c13 * Td, Td, eps4);
    const double u0 = fma(-2.0, d12, Ta), u1 = d12 + d23, u2 = fma(2.0, d23, Tc);   // w0-4w1+3w2, w1-w3, 3w2-4w3+w4
    const double v0 = fma(2.0, d34, Td), v1 = d23 + d34, v2 = fma(-2.0, d23, Tb);   // 3w3-4w4+w5, w2-w4, w1-4w2+3w3
    double s0 = fma(u0, u0, Aa), s1 = fma(u1, u1, Ab), s2 = fma(u2, u2, Ac);
    double z0 = fma(v0, v0, Ad), z1 = fma(v1, v1, Ac), z2 = fma(v2, v2, Ab);
    s0 *= s0; s1 *= s1; s2 *= s2;
    z0 *= z0; z1 *= z1; z2 *= z2;
    {
        const double a0 = s1 * s2, a1 = s0 * s2, a2 = s0 * s1;
        left = fma(fma(a0, q0, fma(a1, q1, a2 * q2)), fast_rcp(fma(10.0, a1, fma(5.0, a2, a0))), w2);
    }
    {
        const double a0 = z1 * z2, a1 = z0 * z2, a2 = z0 * z1;
        right = fma(fma(a0, r0, fma(a1, r1, a2 * r2)), fast_rcp(fma(10.0, a1, fma(5.0, a2, a0))), w3);
    }
}

// WENO5 + Rusanov flux at one face in the face-normal frame (O10).
// q points at component 0 of cell i-2 (the first of the 6 stencil cells) in shared memory;
// cs = cell stride along the face normal, plane = component stride, kn / kt = components of
// the normal / tangential momentum.  Each characteristic field re-reads its 6 x 4 stencil from
// shared memory (keeps the live register set small; shared-memory bandwidth is not the limit).
template <bool CHAR>
__device__ __forceinline__ void weno_rusanov(const double* __restrict__ q, int cs, int plane, int kn, int kt, double g,
                                             double eps, double F[4]) {
    const double gm1 = g - 1.0;
    const double eps4 = 4.0 * eps;
#define QV(s, k) q[(k) * plane + (s) * cs]
    double wl[4], wr[4];
    double u = 0.0, v = 0.0, c = 0.0, qk = 0.0, H = 0.0;
    if (CHAR) {
        // eigen-system at the arithmetic-mean primitive state of cells i, i+1 (A4)
        double rL = QV(2, 0), rR = QV(3, 0);
        double iL = fast_rcp(rL), iR = fast_rcp(rR);
        double uL = QV(2, kn) * iL, vL = QV(2, kt) * iL;
        double uR = QV(3, kn) * iR, vR = QV(3, kt) * iR;
        // internal energies per volume e = E - (m u + w v)/2 (p = (g-1) e); at the mean state
        // c^2 = g p / rho = g (g-1) (e_L + e_R) / (rho_L + rho_R)
        const double eL = QV(2, 3) - 0.5 * (QV(2, kn) * uL + QV(2, kt) * vL);
        const double eR = QV(3, 3) - 0.5 * (QV(3, kn) * uR + QV(3, kt) * vR);
        u = 0.5 * (uL + uR);
        v = 0.5 * (vL + vR);
        const double c2 = (g * gm1) * (eL + eR) * fast_rcp(rL + rR);
        const double ic = fast_rsqrt(c2);   // 1/c, and c = c2 / c (A41: <= 3 / 2 ulp, scripts/rcp_check.cu)
        c = c2 * ic;
        qk = 0.5 * (u * u + v * v);
        H = c2 * (1.0 / gm1) + qk;   // (1 / gm1: one division per thread, hoisted by the compiler)
        // rows of L (O10): l1 = 1/2 (b2 + u/c, -b1 u - 1/c, -b1 v, b1), l2 = (1 - b2, b1 u, b1 v, -b1),
        // l3 = (-v, 0, 1, 0), l4 = 1/2 (b2 - u/c, -b1 u + 1/c, -b1 v, b1), b1 = (g-1)/c^2, b2 = b1 q -- applied
        // factorised (A41): with X = u Qn + v Qt - Q3, hA = (b2 Q0 - b1 X)/2 and hB = (u Q0 - Qn)/(2c),
        // l1 Q = hA + hB, l4 Q = hA - hB, l2 Q = Q0 - 2 hA, l3 Q = Qt - v Q0
        const double hb1 = 0.5 * (gm1 * (ic * ic)), hb2 = hb1 * qk, hic = 0.5 * ic;
        double hA[6], hB[6], w[6];
#pragma unroll
        for (int s = 0; s < 6; ++s) {
            const double q0 = QV(s, 0), qn = QV(s, kn);
            const double X = fma(u, qn, fma(v, QV(s, kt), -QV(s, 3)));
            hA[s] = fma(hb2, q0, -hb1 * X);
            hB[s] = fma(u, q0, -qn) * hic;
        }
#pragma unroll
        for (int s = 0; s < 6; ++s) w[s] = hA[s] + hB[s];
        weno5_pair(w[0], w[1], w[2], w[3], w[4], w[5], eps4, wl[0], wr[0]);
#pragma unroll
        for (int s = 0; s < 6; ++s) w[s] = hA[s] - hB[s];
        weno5_pair(w[0], w[1], w[2], w[3], w[4], w[5], eps4, wl[3], wr[3]);
#pragma unroll
        for (int s = 0; s < 6; ++s) w[s] = fma(-2.0, hA[s], QV(s, 0));
        weno5_pair(w[0], w[1], w[2], w[3], w[4], w[5], eps4, wl[1], wr[1]);
#pragma unroll
        for (int s = 0; s < 6; ++s) w[s] = fma(-v, QV(s, 0), QV(s, kt));
        weno5_pair(w[0], w[1], w[2], w[3], w[4], w[5], eps4, wl[2], wr[2]);
    } else {
        const int kk[4] = {0, kn, kt, 3};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            weno5_pair(QV(0, kk[k]), QV(1, kk[k]), QV(2, kk[k]), QV(3, kk[k]), QV(4, kk[k]), QV(5, kk[k]), eps4,
                       wl[k], wr[k]);
        }
    }
#undef QV
    double UL[4], UR[4];
    if (CHAR) {
        // U = R w, columns r1 = (1, u-c, v, H-uc), r2 = (1, u, v, q), r3 = (0,0,1,v), r4 = (1, u+c, v, H+uc), as
        // U0 = w1 + w2 + w4, U1 = u U0 + c (w4 - w1), U2 = v U0 + w3, U3 = H (w1 + w4) + uc (w4 - w1) + q w2 + v w3
        const double uc = u * c;
        auto back = [&](const double (&wk)[4], double (&U)[4]) {
            const double S03 = wk[0] + wk[3], D = wk[3] - wk[0];
            U[0] = S03 + wk[1];
            U[1] = fma(u, U[0], c * D);
            U[2] = fma(v, U[0], wk[2]);
            U[3] = fma(H, S03, fma(uc, D, fma(qk, wk[1], v * wk[2])));
        };
        back(wl, UL);
        back(wr, UR);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) { UL[k] = wl[k]; UR[k] = wr[k]; }
    }
    // Rusanov (Eq. 11) with S = max(c^R + |u^R|, c^L + |u^L|) (Eq. 12)
    double irL = fast_rcp(UL[0]), irR = fast_rcp(UR[0]);
    double unL = UL[1] * irL, utL = UL[2] * irL;
    double unR = UR[1] * irR, utR = UR[2] * irR;
    double pL = gm1 * (UL[3] - 0.5 * (UL[1] * unL + UL[2] * utL));
    double pR = gm1 * (UR[3] - 0.5 * (UR[1] * unR + UR[2] * utR));
    double sL = fast_sqrt(g * pL * irL) + fabs(unL);
    double sR = fast_sqrt(g * pR * irR) + fabs(unR);
    double S = sR > sL ? sR : sL;   // as the oracle (O10): a NaN wave speed propagates instead of being dropped
    // returned as 2 F (the 1/2 of Eq. 11 goes into the caller's divergence / flux-register scale, kWenoFluxScale)
    F[0] = (UR[1] + UL[1]) - S * (UR[0] - UL[0]);
    F[1] = (fma(UR[1], unR, pR) + fma(UL[1], unL, pL)) - S * (UR[1] - UL[1]);
    F[2] = fma(UR[2], unR, UL[2] * unL) - S * (UR[2] - UL[2]);
    F[3] = fma(UR[3] + pR, unR, (UL[3] + pL) * unL) - S * (UR[3] - UL[3]);
}
// weno_rusanov returns 2 F
constexpr double kWenoFluxScale = 0.5;

// Central4 edge flux: Eq. 8 weights (9/16, -1/16) applied edge-from-node (A7)
// to (p, T = p/rho, u_n, u_t) of cells i-1..i+2; rho_e = p_e / T_e (A6).
// q points at component 0 (p) of cell i-1 in shared memory (components p, T, u, v).
__device__ __forceinline__ void central4_flux(const double* __restrict__ q, int cs, int plane, int kn, int kt,
                                              double inv_gm1, double F[4]) {
#define QV(s, k) q[(k) * plane + (s) * cs]
    double pe = 0.5625 * (QV(1, 0) + QV(2, 0)) - 0.0625 * (QV(0, 0) + QV(3, 0));
    double Te = 0.5625 * (QV(1, 1) + QV(2, 1)) - 0.0625 * (QV(0, 1) + QV(3, 1));
    double un = 0.5625 * (QV(1, kn) + QV(2, kn)) - 0.0625 * (QV(0, kn) + QV(3, kn));
    double ut = 0.5625 * (QV(1, kt) + QV(2, kt)) - 0.0625 * (QV(0, kt) + QV(3, kt));
#undef QV
    double re = pe / Te;
    double Ee = pe * inv_gm1 + 0.5 * re * (un * un + ut * ut);
    double mn = re * un;
    F[0] = mn;
    F[1] = mn * un + pe;
    F[2] = mn * ut;
    F[3] = (Ee + pe) * un;
}

// ---------------------------------------------------------------- the fused stage kernel
constexpr int kGL = 4;   // ghost width loaded into shared memory (16-byte aligned strips, A8)

template <int T>
struct Block;
template <>
struct Block<8> { static constexpr int NT = 64; static constexpr int MINB = 8; };
template <>
struct Block<16> { static constexpr int NT = 128; static constexpr int MINB = 4; };
template <>
struct Block<32> { static constexpr int NT = 256; static constexpr int MINB = 2; };

// T <= 16: x and y face fluxes in separate planes, computed in ONE loop over both directions (at T = 16 the
// 16 x 19 faces per direction fill 128 threads to 79 % per pass, 2 x 304 faces in one pass fill 95 %)
template <int T>
constexpr bool kCombFaces = T <= 16;

// WENO tiles of T <= 16 also stage U^n of the tile in shared memory (cp.async issued with the halo gather, waited
// for before the divergence), instead of a dependent global load in the update
template <int SCHEME, int T>
constexpr bool kUnSmem = SCHEME == 1 && T <= 16;   // (component-wise WENO runs 5 CTAs/SM at T = 16: no room)
template <int SCHEME, int T>
constexpr size_t stage_smem() {
    return sizeof(double) * (4 * (T + 2 * kGL) * (T + 2 * kGL) + (kCombFaces<T> ? 2 : 1) * 4 * T * (T + 3) +
                             (kUnSmem<SCHEME, T> ? 4 * T * T : 0));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// The stage-input buffer a same-level side neighbour is read from: the local one, or -- halo_mode 2, neighbour owned
// by another rank (LeafDesc.pad bits 4 + s, owner in bits 8 + 3 s) -- that rank's pool mapped over NVLink, so the
// face strip is loaded by this kernel from the owner's memory (no halo exchange before the stage)
__device__ __forceinline__ const double* side_source(const StageArgs& a, const LeafDesc& d, int side) {
    if (!(d.pad & (16 << side))) return a.Uin;
    return a.peer_in[(d.pad >> (8 + 3 * side)) & 7];
}

// SCHEME 0: Central4; 1: WENO5 characteristic; 2: WENO5 component-wise.
// One CTA per T x T tile of a leaf patch (T = n, or 32 for n = 64).
// CTAs per SM the stage kernel is compiled for: component-wise WENO5 at T = 16 fits 96 registers without spills at
// 5 (shared memory admits 5 x 38 KB), 1.22 -> 1.16 ms on the 4096^2 sweep; the characteristic kernel was 1.2 % slower
// there (1.51 -> 1.53 ms) and keeps 4
template <int SCHEME, int T>
struct StageMinB { static constexpr int v = (SCHEME == 2 && T == 16) ? 5 : Block<T>::MINB; };

template <int SCHEME, int T>
__global__ void __launch_bounds__(Block<T>::NT, StageMinB<SCHEME, T>::v) stage_kernel(const StageArgs a) {
    constexpr int G = kGL;
    constexpr int NT = Block<T>::NT;
    constexpr int W = T + 2 * G;       // tile row width in shared memory (doubles)
    constexpr int PL = W * W;          // one component plane
    constexpr int NF = T + 3;          // faces per row: m = -1 .. T+1 (face m = left of cell m)
    constexpr int CPT = (T * T + NT - 1) / NT;
    extern __shared__ __align__(16) double smem[];
    double* sQ = smem;                 // [4][W][W]: conserved (WENO) / (p, T, u, v) (Central4)
    double* sF = smem + 4 * PL;        // [4][T][NF] x-fluxes, then [4][NF][T] y-fluxes
    double* const sUn = sF + (kCombFaces<T> ? 2 : 1) * 4 * T * (T + 3);   // [4][T][T] U^n (kUnSmem)

    const int tid = threadIdx.x;
    const int tiles2 = a.tiles * a.tiles;
    const int leaf = blockIdx.x / tiles2;
    const int tt = blockIdx.x - leaf * tiles2;
    const int tx = tt % a.tiles, ty = tt / a.tiles;
    const LeafDesc d = a.leaves[leaf];
    const int n = a.geo.n;
    const size_t nn = (size_t)n * n;
    const size_t PS = 4 * nn;
    const double* own = a.Uin + (size_t)d.slot * PS;

    // ---- halo gather (a1): plus-shaped tile, 16-byte cp.async (corners are never read, A26)
    {
        constexpr int CR = W / 2, CB = T * CR, CS = G * T / 2, CV = CB + 2 * CS;
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sQ);
        // 16-byte chunk f of one component plane -> (shared offset, source address of component 0)
        auto chunk = [&](int f, uint32_t& dst, const double*& src) {
            int i, j;
            if (f < CB) { j = f / CR; i = 2 * (f - j * CR) - G; }
            else if (f < CB + CS) { int h = f - CB; j = h / (T / 2) - G; i = 2 * (h - (j + G) * (T / 2)); }
            else { int h = f - CB - CS; j = h / (T / 2); i = 2 * (h - j * (T / 2)); j += T; }
            int pi = tx * T + i, pj = ty * T + j;
            int s = 0, sd = -1;
            bool halo = true;
            if (pi < 0) { sd = kW; pi += n; }
            else if (pi >= n) { sd = kE; pi -= n; }
            else if (pj < 0) { sd = kS; pj += n; }
            else if (pj >= n) { sd = kN; pj -= n; }
            else halo = false;
            if (halo) s = d.side[sd];
            const double* base = !halo ? own : (s >= 0 ? side_source(a, d, sd) + (size_t)s * PS : a.proxy + (size_t)(-1 - s) * PS);
            dst = sb + (uint32_t)(((j + G) * W + (i + G)) * 8);
            src = base + (size_t)pj * n + pi;
        };
        if (CV % NT == 0) {   // a thread's chunks are the same CV / NT positions in each of the 4 planes: map once
#pragma unroll
            for (int r = 0; r < CV / NT; ++r) {
                uint32_t dst;
                const double* src;
                chunk(tid + r * NT, dst, src);
#pragma unroll
                for (int k = 0; k < 4; ++k) cp_async16(dst + (uint32_t)(k * PL * 8), src + k * nn);
            }
        } else {
            for (int e = tid; e < 4 * CV; e += NT) {
                const int k = e / CV;
                uint32_t dst;
                const double* src;
                chunk(e - k * CV, dst, src);
                cp_async16(dst + (uint32_t)(k * PL * 8), src + k * nn);
            }
        }
        if (kUnSmem<SCHEME, T> && a.stage > 1) {   // U^n of the tile: a second group, waited for before the divergence
            cp_async_commit();
            const uint32_t su = (uint32_t)__cvta_generic_to_shared(sUn);
            const double* pn0 = a.Un + (size_t)d.slot * PS;
            constexpr int CH = T * T / 2;   // 16-byte chunks per component
            for (int e = tid; e < 4 * CH; e += NT) {
                const int k = e / CH, r = e - k * CH, jj = r / (T / 2), ii = 2 * (r - jj * (T / 2));
                cp_async16(su + (uint32_t)((k * T * T + jj * T + ii) * 8), pn0 + k * nn + (size_t)(ty * T + jj) * n + tx * T + ii);
            }
            cp_async_commit();
            cp_async_wait1();
        } else {
            cp_async_wait_all();
        }
    }
    __syncthreads();

    const double g = a.gamma;
    const double inv_gm1 = 1.0 / (g - 1.0);
    if (SCHEME == 0) {
        // cons -> (p, T, u, v) in place (Eq. 4-6) over the plus-shaped tile
        constexpr int EB = T * W, ES = G * T, ET = EB + 2 * ES;
        for (int e = tid; e < ET; e += NT) {
            int i, j;
            if (e < EB) { j = e / W; i = e - j * W - G; }
            else if (e < EB + ES) { int f = e - EB; j = f / T - G; i = f - (j + G) * T; }
            else { int f = e - EB - ES; j = f / T; i = f - j * T; j += T; }
            int o = (j + G) * W + (i + G);
            double r = sQ[o], m = sQ[PL + o], w = sQ[2 * PL + o], E = sQ[3 * PL + o];
            double ir = 1.0 / r;
            double u = m * ir, v = w * ir;
            double p = (g - 1.0) * (E - 0.5 * (m * u + w * v));
            sQ[o] = p;
            sQ[PL + o] = p * ir;
            sQ[2 * PL + o] = u;
            sQ[3 * PL + o] = v;
        }
        __syncthreads();
    }

    const int lvl = d.level;
    const double idx = a.geo.inv_dx[lvl], idy = a.geo.inv_dy[lvl];
    const bool div4 = a.div_order == 4;
    // Eq. 9 as 24 F-hat = 26 f - (f- + f+): the 1/24 goes into the divergence and the flux registers
    const double fsc = (SCHEME == 0 ? 1.0 : kWenoFluxScale) * (div4 ? 1.0 / 24.0 : 1.0), idx24 = fsc * idx, idy24 = fsc * idy;
    const int x_lo = tx == 0, x_hi = tx == a.tiles - 1, y_lo = ty == 0, y_hi = ty == a.tiles - 1;
    const int store_mask = (d.cf | (d.cf >> 4)) & 15;

    constexpr bool COMB = kCombFaces<T>;
    double* const sFy = COMB ? sF + 4 * T * NF : sF;   // y-face fluxes [4][NF][T]
    auto x_face = [&](int e) {   // face m (left of cell m), row j
        int j = e / NF, m = e - j * NF - 1;
        int o = (j + G) * W + (m + G);
        double f[4];
        if (SCHEME == 0) central4_flux(sQ + o - 2, 1, PL, 2, 3, inv_gm1, f);
        else weno_rusanov<SCHEME == 1>(sQ + o - 3, 1, PL, 1, 2, g, a.eps, f);
#pragma unroll
        for (int k = 0; k < 4; ++k) sF[(k * T + j) * NF + m + 1] = f[k];
    };
    auto y_flux = [&](int e, double (&f)[4]) {   // face m (below cell m), column i; normal momentum is component 2
        int m = e / T - 1, i = e - (m + 1) * T;
        int o = (m + G) * W + (i + G);
        if (SCHEME == 0) central4_flux(sQ + o - 2 * W, W, PL, 3, 2, inv_gm1, f);
        else weno_rusanov<SCHEME == 1>(sQ + o - 3 * W, W, PL, 2, 1, g, a.eps, f);
    };
    auto y_store = [&](int e, const double (&f)[4]) {
        int m = e / T - 1, i = e - (m + 1) * T;
        sFy[(0 * NF + m + 1) * T + i] = f[0];
        sFy[(1 * NF + m + 1) * T + i] = f[2];
        sFy[(2 * NF + m + 1) * T + i] = f[1];
        sFy[(3 * NF + m + 1) * T + i] = f[3];
    };
    auto y_face = [&](int e) {
        double f[4];
        y_flux(e, f);
        y_store(e, f);
    };
    // one plane (T > 16): the threads left idle by the last x-face pass compute their first y face then and keep
    // it in registers until the x divergence has read the plane (T = 32: 9 face passes instead of 10)
    constexpr int NXF = T * NF, KX = (NXF + NT - 1) / NT;
    int yh_e = -1;
    double yh[4];
    // ---- faces (a4-a6)
    if (COMB) {   // both directions in one pass; the x range padded to whole warps (no warp straddles x / y)
        constexpr int NX = T * NF, NXP = (NX + 31) / 32 * 32;
        for (int e = tid; e < NXP + NX; e += NT) {
            if (e < NXP) {
                if (e < NX) x_face(e);
            } else {
                y_face(e - NXP);
            }
        }
    } else {
#pragma unroll 1
        for (int k = 0; k < KX; ++k) {
            const int e = tid + k * NT;
            if (e < NXF) x_face(e);
            else if (e - NXF < NXF) { yh_e = e - NXF; y_flux(yh_e, yh); }
        }
    }
    if (kUnSmem<SCHEME, T> && a.stage > 1) cp_async_wait0();   // this thread's U^n chunks; the barrier shows all
    __syncthreads();
    // ---- x divergence (a7, Eq. 9 flux form) into registers
    double acc[CPT][4];
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
        int c = tid + r * NT;
        if (c < T * T) {
            int i = c % T, j = c / T;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double* fr = sF + (k * T + j) * NF + i + 1;   // fr[0] = f at face i
                double fl = fr[0], fh = fr[1];
                double Fl = div4 ? fma(26.0, fl, -(fr[-1] + fh)) : fl;   // 24 F-hat
                double Fh = div4 ? fma(26.0, fh, -(fl + fr[2])) : fh;
                acc[r][k] = -(Fh - Fl) * idx24;
                if (i == 0 && x_lo && (store_mask & 1))
                    a.freg[(((size_t)d.slot * 4 + kW) * 4 + k) * n + ty * T + j] = fsc * Fl;
                if (i == T - 1 && x_hi && (store_mask & 2))
                    a.freg[(((size_t)d.slot * 4 + kE) * 4 + k) * n + ty * T + j] = fsc * Fh;
            }
        }
    }
    if (!COMB) {   // y faces into the same plane once the x divergence has read it
        __syncthreads();
        if (yh_e >= 0) y_store(yh_e, yh);
        for (int e = tid + KX * NT - NXF; e < NXF; e += NT) y_face(e);
        __syncthreads();
    }

    // ---- y divergence, SSP-RK3 combination (a8), checks, Lambda (a9)
    const double dt = *a.dt;
    const int coarse_mask = d.cf & 15;
    const double* pin = a.Uin + (size_t)d.slot * PS;
    const double* pn = a.Un + (size_t)d.slot * PS;
    double* po = a.Uout + (size_t)d.slot * PS;
    unsigned long long lam = 0ull;
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
        int c = tid + r * NT;
        if (c < T * T) {
            int i = c % T, j = c / T;
            size_t off = (size_t)(ty * T + j) * n + tx * T + i;
            double o4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double* fr = sFy + (k * NF + j + 1) * T + i;   // fr[0] = f at face j
                double fl = fr[0], fh = fr[T];
                double Fl = div4 ? fma(26.0, fl, -(fr[-T] + fh)) : fl;   // 24 F-hat
                double Fh = div4 ? fma(26.0, fh, -(fl + fr[2 * T])) : fh;
                double L = acc[r][k] - (Fh - Fl) * idy24;
                if (j == 0 && y_lo && (store_mask & 4))
                    a.freg[(((size_t)d.slot * 4 + kS) * 4 + k) * n + tx * T + i] = fsc * Fl;
                if (j == T - 1 && y_hi && (store_mask & 8))
                    a.freg[(((size_t)d.slot * 4 + kN) * 4 + k) * n + tx * T + i] = fsc * Fh;
                // U^(s-1): the WENO tile holds it in shared memory (Central4 converted its tile to primitives)
                double v = (SCHEME != 0 ? sQ[k * PL + (j + G) * W + (i + G)] : __ldg(pin + k * nn + off)) + dt * L;
                if (a.stage > 1) v = a.a * (kUnSmem<SCHEME, T> ? sUn[(k * T + j) * T + i] : __ldg(pn + k * nn + off)) + a.b * v;
                o4[k] = v;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) po[k * nn + off] = o4[k];
            // cells on an edge that is the coarse side of a C/F face are finished by the reflux kernel
            bool edge_cf = ((coarse_mask & 1) && x_lo && i == 0) || ((coarse_mask & 2) && x_hi && i == T - 1) ||
                           ((coarse_mask & 4) && y_lo && j == 0) || ((coarse_mask & 8) && y_hi && j == T - 1);
            if (!edge_cf && !(d.pad & 1)) {   // covered patches (subcycling) are not leaves
                if (a.check || a.want_lambda)
                    leaf_check(o4[0], o4[1], o4[2], o4[3], g, idx, idy, a.check, a.want_lambda, a.lam0 ? d.level : 0,
                               a.err, d.slot, a.stage, (int)off, lam);
            }
        }
    }
    if (a.want_lambda) {
        lam = warp_max_u64(lam);
        if ((tid & 31) == 0 && lam) atomicMax(a.lambda_bits, lam);
    }
}

template <int SCHEME, int T>
cudaError_t launch_stage_t(const StageArgs& a, cudaStream_t s) {
    constexpr size_t smem = stage_smem<SCHEME, T>();
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(stage_kernel<SCHEME, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    unsigned blocks = (unsigned)a.nleaves * a.tiles * a.tiles;
    if (blocks == 0) return cudaSuccess;
    stage_kernel<SCHEME, T><<<blocks, Block<T>::NT, smem, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Central4 fused stage kernel
// Specialised for the HBM-bound shock-free scheme (Eq. 8/9): warp-per-row 16-byte cp.async gather,
// in-place cons->prim, sliding-window face fluxes (each thread computes R consecutive faces of one
// row / column with a rolling 4-cell register window) and sliding-window divergences (each thread owns
// CPT cells of one column), so that every cell is loaded from shared memory a handful of times.

template <int T>
struct C4Cfg;
template <>
struct C4Cfg<32> { static constexpr int NT = 256, SEG = 7, R = 5, MINB = 2; };
template <>
struct C4Cfg<16> { static constexpr int NT = 128, SEG = 8, R = 3, MINB = 4; };
template <>
struct C4Cfg<8> { static constexpr int NT = 64, SEG = 8, R = 2, MINB = 8; };

// Central4 edge flux from a rolling window c[0..3] = cells i-1..i+2 of (p, T, un, ut).
__device__ __forceinline__ void c4_face(const double (&p)[4], const double (&Tt)[4], const double (&un)[4],
                                        const double (&ut)[4], double inv_gm1, double F[4]) {
    double pe = 0.5625 * (p[1] + p[2]) - 0.0625 * (p[0] + p[3]);
    double Te = 0.5625 * (Tt[1] + Tt[2]) - 0.0625 * (Tt[0] + Tt[3]);
    double ue = 0.5625 * (un[1] + un[2]) - 0.0625 * (un[0] + un[3]);
    double ve = 0.5625 * (ut[1] + ut[2]) - 0.0625 * (ut[0] + ut[3]);
    double re = pe * fast_rcp(Te);
    double Ee = pe * inv_gm1 + 0.5 * re * (ue * ue + ve * ve);
    double mn = re * ue;
    F[0] = mn;
    F[1] = mn * ue + pe;
    F[2] = mn * ve;
    F[3] = (Ee + pe) * ue;
}

// The same edge flux scaled by 16 (F16 = 16 F, bit-exactly: every rescaling below is by a power of two): the
// Eq. 8 weights (9/16, -1/16) become fma(9, inner pair, -outer pair), one operation fewer per variable; the
// ratio p/T is scale-free, and the caller folds 1/16 into the divergence (idx / 16).
__device__ __forceinline__ void c4_face16(const double (&p)[4], const double (&Tt)[4], const double (&un)[4],
                                          const double (&ut)[4], double g_gm1, double F16[4]) {
    const double pe = fma(9.0, p[1] + p[2], -(p[0] + p[3]));      // 16 p_e
    const double Te = fma(9.0, Tt[1] + Tt[2], -(Tt[0] + Tt[3]));  // 16 T_e
    const double U16 = fma(9.0, un[1] + un[2], -(un[0] + un[3]));   // 16 u_e
    const double ue = 0.0625 * U16;
    const double ve = 0.0625 * fma(9.0, ut[1] + ut[2], -(ut[0] + ut[3]));
    const double re = pe * fast_rcp(Te);                          // rho_e (scale-free)
    // 16 (E_e + p_e) = 16 p_e g/(g-1) + 8 rho_e (u_e^2 + v_e^2) (one operation fewer than E_e, then + p_e)
    const double He = fma(pe, g_gm1, (8.0 * re) * fma(ve, ve, ue * ue));
    const double mn16 = re * U16;                                 // = 16 (re ue) exactly
    F16[0] = mn16;
    F16[1] = fma(mn16, ue, pe);
    F16[2] = mn16 * ve;
    F16[3] = He * ue;
}

template <int N>
__global__ void __launch_bounds__(C4Cfg<(N > 32 ? 32 : N)>::NT, C4Cfg<(N > 32 ? 32 : N)>::MINB)
    stage_c4_kernel(const StageArgs a) {
    constexpr int T = N > 32 ? 32 : N;       // tile edge
    constexpr int TILES = N / T;             // tiles per patch edge
    constexpr int G = kGL;
    constexpr int NT = C4Cfg<T>::NT, SEG = C4Cfg<T>::SEG, R = C4Cfg<T>::R;
    constexpr int NW = NT / 32;
    constexpr int W = T + 2 * G;
    constexpr int PL = W * W;
    constexpr int NF = T + 3;                // faces m = -1 .. T+1
    constexpr int CPT = T * T / NT;          // cells per thread (one column strip)
    constexpr int NN = N * N;
    constexpr int PS = 4 * NN;
    constexpr bool EXACT = SEG * R == NF;    // no face-segment guard needed
    static_assert(SEG * R >= NF, "face segments must cover the row");
    static_assert(T * SEG <= NT, "one thread per face segment");
    extern __shared__ __align__(16) double smem[];
    double* sQ = smem;                       // [4][W][W] conserved, then (p, T, u, v)
    double* sF = smem + 4 * PL;              // [4][T][NF] x-fluxes, then [4][NF][T] y-fluxes

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int leaf = TILES == 1 ? blockIdx.x : blockIdx.x / (TILES * TILES);
    const int tt = TILES == 1 ? 0 : blockIdx.x - leaf * (TILES * TILES);
    const int tx = tt % TILES, ty = tt / TILES;
    const LeafDesc d = a.leaves[leaf];
    const double* own = a.Uin + (size_t)d.slot * PS;
    const double* src[4];
#pragma unroll
    for (int s = 0; s < 4; ++s)
        src[s] = d.side[s] >= 0 ? side_source(a, d, s) + (size_t)d.side[s] * PS   // halo_mode 2: maybe a peer's pool
                                : a.proxy + (size_t)(-1 - d.side[s]) * PS;

    // ---- (a1) halo gather: one warp per (component, row); lanes move 16-byte chunks
    {
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sQ);
        constexpr int CR = W / 2;            // chunks per band row
        for (int task = warp; task < 4 * T; task += NW) {
            const int k = task / T, j = task - k * T;
            const int pj = ty * T + j;
            if (lane < CR) {
                int pi = tx * T + 2 * lane - G;
                const double* b = own;
                if (pi < 0) { b = src[kW]; pi += N; }
                else if (pi >= N) { b = src[kE]; pi -= N; }
                cp_async16(sb + (uint32_t)((k * PL + (j + G) * W + 2 * lane) * 8), b + k * NN + pj * N + pi);
            }
        }
        for (int task = warp; task < 4 * 2 * G; task += NW) {
            const int k = task / (2 * G), r = task - k * (2 * G);
            const int j = r < G ? r - G : T + (r - G);
            int pj = ty * T + j;
            const double* b = own;
            if (pj < 0) { b = src[kS]; pj += N; }
            else if (pj >= N) { b = src[kN]; pj -= N; }
            if (lane < T / 2)
                cp_async16(sb + (uint32_t)((k * PL + (j + G) * W + G + 2 * lane) * 8), b + k * NN + pj * N + tx * T + 2 * lane);
        }
        cp_async_wait_all();
    }
    __syncthreads();

    const double g = a.gamma, gm1 = g - 1.0;
    const double inv_gm1 = 1.0 / gm1;
    // ---- (a3) cons -> (p, T, u, v) in place: band rows then strip rows, lanes along the row
    for (int task = warp; task < T + 2 * G; task += NW) {
        const int j = task < T ? task : (task - T < G ? task - T - G : task - G);
        const int i0 = task < T ? -G : 0, len = task < T ? W : T;
        double* q = sQ + (j + G) * W + i0 + G;
        for (int c = lane; c < len; c += 32) {
            double r = q[c], m = q[PL + c], w = q[2 * PL + c], E = q[3 * PL + c];
            double ir = fast_rcp(r);
            double u = m * ir, v = w * ir;
            double p = gm1 * (E - 0.5 * (m * u + w * v));
            q[c] = p;
            q[PL + c] = p * ir;
            q[2 * PL + c] = u;
            q[3 * PL + c] = v;
        }
    }
    __syncthreads();

    const int lvl = d.level;
    const double idx = a.geo.inv_dx[lvl], idy = a.geo.inv_dy[lvl];
    const bool div4 = a.div_order == 4;
    const bool x_lo = tx == 0, x_hi = tx == TILES - 1, y_lo = ty == 0, y_hi = ty == TILES - 1;
    const int store_mask = (d.cf | (d.cf >> 4)) & 15;
    const double c13 = 13.0 / 12.0, c24 = 1.0 / 24.0;

    // ---- (a4-a6) x faces: thread (row j, segment s) computes faces m0 .. m0+R-1
    if (tid < T * SEG && (EXACT || (tid % SEG) * R - 1 <= T + 1)) {
        const int j = tid / SEG, s = tid - j * SEG;
        const int m0 = s * R - 1;
        const double* q = sQ + (j + G) * W + G + m0;   // q[c] = cell m0 + c of row j
        double* fo = sF + j * NF + m0 + 1;              // fo[k*T*NF + f] = flux at face m0 + f
        double p[4], Tt[4], un[4], ut[4];
#pragma unroll
        for (int c = 0; c < 3; ++c) { p[c + 1] = q[c - 2]; Tt[c + 1] = q[PL + c - 2]; un[c + 1] = q[2 * PL + c - 2]; ut[c + 1] = q[3 * PL + c - 2]; }
#pragma unroll
        for (int f = 0; f < R; ++f) {
#pragma unroll
            for (int c = 0; c < 3; ++c) { p[c] = p[c + 1]; Tt[c] = Tt[c + 1]; un[c] = un[c + 1]; ut[c] = ut[c + 1]; }
            if (EXACT || m0 + f <= T + 1) {
                p[3] = q[f + 1]; Tt[3] = q[PL + f + 1]; un[3] = q[2 * PL + f + 1]; ut[3] = q[3 * PL + f + 1];
                double F[4];
                c4_face(p, Tt, un, ut, inv_gm1, F);
#pragma unroll
                for (int k = 0; k < 4; ++k) fo[k * T * NF + f] = F[k];
            }
        }
    }
    __syncthreads();

    // ---- (a7) x divergence (Eq. 9 flux form): thread owns column ci, rows cj0 .. cj0+CPT-1
    const int ci = tid % T, cj0 = (tid / T) * CPT;
    double acc[CPT][4];
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double* fr = sF + (k * T + cj0 + r) * NF + ci + 1;   // fr[0] = f at face ci
            double fl = fr[0], fh = fr[1];
            double Fl = div4 ? c13 * fl - c24 * (fr[-1] + fh) : fl;
            double Fh = div4 ? c13 * fh - c24 * (fl + fr[2]) : fh;
            acc[r][k] = -(Fh - Fl) * idx;
            if (store_mask) {
                if (ci == 0 && x_lo && (store_mask & 1)) a.freg[(((size_t)d.slot * 4 + kW) * 4 + k) * N + ty * T + cj0 + r] = Fl;
                if (ci == T - 1 && x_hi && (store_mask & 2)) a.freg[(((size_t)d.slot * 4 + kE) * 4 + k) * N + ty * T + cj0 + r] = Fh;
            }
        }
    }
    __syncthreads();

    // ---- y faces: thread (column i, segment s), rolling window along j; normal velocity = v
    if (tid < T * SEG && (EXACT || (tid / T) * R - 1 <= T + 1)) {
        const int i = tid % T, s = tid / T;
        const int m0 = s * R - 1;
        const double* q = sQ + (m0 + G) * W + (i + G);   // q[c*W] = cell (i, m0 + c)
        double* fo = sF + (m0 + 1) * T + i;               // fo[k*NF*T + f*T] = flux at face m0 + f
        double p[4], Tt[4], un[4], ut[4];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int o = (c - 2) * W;
            p[c + 1] = q[o]; Tt[c + 1] = q[PL + o]; un[c + 1] = q[3 * PL + o]; ut[c + 1] = q[2 * PL + o];
        }
#pragma unroll
        for (int f = 0; f < R; ++f) {
#pragma unroll
            for (int c = 0; c < 3; ++c) { p[c] = p[c + 1]; Tt[c] = Tt[c + 1]; un[c] = un[c + 1]; ut[c] = ut[c + 1]; }
            if (EXACT || m0 + f <= T + 1) {
                const int o = (f + 1) * W;
                p[3] = q[o]; Tt[3] = q[PL + o]; un[3] = q[3 * PL + o]; ut[3] = q[2 * PL + o];
                double F[4];
                c4_face(p, Tt, un, ut, inv_gm1, F);
                fo[0 * NF * T + f * T] = F[0];
                fo[1 * NF * T + f * T] = F[2];
                fo[2 * NF * T + f * T] = F[1];
                fo[3 * NF * T + f * T] = F[3];
            }
        }
    }
    __syncthreads();

    // ---- y divergence (sliding along the owned column), SSP-RK3 (a8), checks, Lambda (a9)
    const double dt = *a.dt;
    const int coarse_mask = d.cf & 15;
    const int base_off = (ty * T + cj0) * N + tx * T + ci;
    const double* pin = a.Uin + (size_t)d.slot * PS + base_off;
    const double* pn = a.Un + (size_t)d.slot * PS + base_off;
    double* po = a.Uout + (size_t)d.slot * PS + base_off;
    const bool rk_un = a.stage > 1;
    const double ca = a.a, cb = a.b;
    double out[CPT][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double* fc = sF + (k * NF + cj0 + 1) * T + ci;   // fc[r*T] = f at face cj0 + r
        double fm1 = fc[-T], f0 = fc[0], f1 = fc[T];
        double Flo = div4 ? c13 * f0 - c24 * (fm1 + f1) : f0;
        if (store_mask && cj0 == 0 && y_lo && (store_mask & 4))
            a.freg[(((size_t)d.slot * 4 + kS) * 4 + k) * N + tx * T + ci] = Flo;
#pragma unroll
        for (int r = 0; r < CPT; ++r) {
            double f2 = fc[(r + 2) * T];
            double Fhi = div4 ? c13 * f1 - c24 * (f0 + f2) : f1;
            double L = acc[r][k] - (Fhi - Flo) * idy;
            double v = __ldg(pin + k * NN + r * N) + dt * L;
            if (rk_un) v = ca * __ldg(pn + k * NN + r * N) + cb * v;
            out[r][k] = v;
            if (store_mask && r == CPT - 1 && cj0 + r == T - 1 && y_hi && (store_mask & 8))
                a.freg[(((size_t)d.slot * 4 + kN) * 4 + k) * N + tx * T + ci] = Fhi;
            Flo = Fhi;
            f0 = f1;
            f1 = f2;
        }
    }
    unsigned long long lam = 0ull;
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
        const int j = cj0 + r;
#pragma unroll
        for (int k = 0; k < 4; ++k) po[k * NN + r * N] = out[r][k];
        bool edge_cf = coarse_mask && (((coarse_mask & 1) && x_lo && ci == 0) || ((coarse_mask & 2) && x_hi && ci == T - 1) ||
                                       ((coarse_mask & 4) && y_lo && j == 0) || ((coarse_mask & 8) && y_hi && j == T - 1));
        if (!edge_cf && !(d.pad & 1)) {   // covered patches (subcycling) are not leaves
            if (a.check || a.want_lambda)
                leaf_check(out[r][0], out[r][1], out[r][2], out[r][3], g, idx, idy, a.check, a.want_lambda,
                           a.lam0 ? d.level : 0, a.err, d.slot, a.stage, (ty * T + j) * N + tx * T + ci, lam);
        }
    }
    if (a.want_lambda) {
        lam = warp_max_u64(lam);
        if (lane == 0 && lam) atomicMax(a.lambda_bits, lam);
    }
}

template <int N>
cudaError_t launch_c4_t(const StageArgs& a, cudaStream_t s) {
    constexpr int T = N > 32 ? 32 : N;
    constexpr size_t smem = stage_smem<0, T>();
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(stage_c4_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    unsigned blocks = (unsigned)a.nleaves * (N / T) * (N / T);
    if (blocks == 0) return cudaSuccess;
    stage_c4_kernel<N><<<blocks, C4Cfg<T>::NT, smem, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Central4 persistent TMA-pipelined stage kernel
// One CTA of 512 threads per SM walks the 32 x 32 tiles of the leaf list (tile t, t + grid, ...).  Each tile's
// conserved values -- the interior box and the four 4-wide side strips of the plus-shaped halo (corners are never
// read, A26) -- arrive by five 3D TMA box loads (cp.async.bulk.tensor, pool viewed as [slot*4 + var][j][i]) into
// one of two landing buffers, completing on an mbarrier; the loads of tile t + grid are issued as soon as tile t's
// landing data has been converted, so HBM streams while the CTA computes.  U^n of the tile's epilogue cells is
// loaded into registers at the top of the tile.  Per tile:
//   (a3) cons -> (p, T, u, v) into padded planes (row stride 44); the interior cell's U^(s-1) stays in registers;
//   (a4-a6) x faces (warps 0-7) and y faces (warps 8-15) concurrently: a lane owns a 5-face segment of one line
//   (lane = line + 4 * segment), slides a 4-cell register window along it, evaluates the Central4 edge flux
//   (Eq. 8, A6/A7) and the Eq. 9 face flux F-hat with the outer neighbours f(m0-1), f(m0+5) shuffled in from
//   the adjacent segments (lanes -4 / +4), and stores F-hat;
//   (a7, a8) per cell (lane = column, warp = row pair): the divergence of F-hat, SSP-RK3, checks, streaming
//   stores; Lambda (a9) reduced once per CTA.
// The strides (prim 44, F-hat 36) give every half-warp's 8-byte shared accesses 16 distinct bank pairs: ncu
// reports zero load conflicts (profiles/).
struct C4Maps {
    CUtensorMap in_int;   // stage input, box {32, 32, 4}
    CUtensorMap in_we;    // stage input, box {4, 32, 4}
    CUtensorMap in_sn;    // stage input, box {32, 4, 4}
    CUtensorMap px_we;    // proxy buffer, box {4, 32, 4}
    CUtensorMap px_sn;    // proxy buffer, box {32, 4, 4}
    CUtensorMap un_int;   // U^n, box {32, 32, 4}
    CUtensorMap out_int;  // U^(s), box {32, 32, 4} (TMA store)
    CUtensorMap peer_we[8];   // halo_mode 2: rank q's U^(s-1) mapped over NVLink, W/E strip boxes
    CUtensorMap peer_sn[8];   //   S/N strip boxes
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_prefetch3(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];"
                 ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, int c0, int c1, int c2, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                 ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(src) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// LeafDesc load the compiler may not sink towards its use (issued one tile ahead on purpose)
__device__ __forceinline__ LeafDesc load_desc_early(const LeafDesc* p) {
    static_assert(sizeof(LeafDesc) == 32, "LeafDesc is two 16-byte words");
    int4 a, b;
    asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p));
    asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(reinterpret_cast<const char*>(p) + 16));
    LeafDesc d;
    d.slot = a.x; d.level = a.y; d.side[0] = a.z; d.side[1] = a.w;
    d.side[2] = b.x; d.side[3] = b.y; d.cf = b.z; d.pad = b.w;
    return d;
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint32_t mb, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(mb), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t mb) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mb)
        : "memory");
}

// 1D bulk copies (cp.async.bulk, no tensor map) for boxes that are one contiguous run of the pool: the whole
// [4][n][n] patch of a 32^2 patch, or K consecutive slots of a group
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mb) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_prefetch(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// U^(s) of the Central4 TMA kernels by direct coalesced stores from registers (default: 1.3 % faster than
// writing it into shared memory for one TMA / bulk store, and one barrier less per tile); -DAMR_C4_TMA_STORE
// selects the store through shared memory
#ifdef AMR_C4_TMA_STORE
constexpr bool kC4Stg = false;
#else
constexpr bool kC4Stg = true;
#endif
// Interior conversion and epilogue of the Central4 TMA kernel on adjacent cell pairs (16-byte shared and global
// accesses: half the shared-memory instructions, whose queue throttled the kernel; 0.384 -> 0.377 ms);
// -DAMR_C4_SCALAR selects one column cell per row pair
#ifdef AMR_C4_SCALAR
constexpr bool kC4Vec2 = false;
#else
constexpr bool kC4Vec2 = true;
#endif
#ifdef AMR_GHOST_PER_CELL   // A/B: the per-cell ghost kernel (every coarse value re-read by each fine cell)
constexpr bool kGhostTile = false;
#else
constexpr bool kGhostTile = true;
#endif
#ifdef AMR_NO_BULK1D
constexpr bool kBulk1D = false;
#else
constexpr bool kBulk1D = true;
#endif
// the per-tile kernel keeps 3D tensor boxes for the 32 KB interior, U^n and prefetch (0.6 % faster than one 1D bulk
// copy at n = 32, A/B on one box); the group kernel's K-member bulk copies replace K boxes (n = 8: -16 %)
constexpr bool kBulk1DTile = false;

constexpr int kTmaThreads = 512;
// optional phase timing (build with AMR_NVCC_FLAGS=-DAMR_PHASE_PROF, run with AMR_PHASE_PROF=1): per-warp
// cycle counts of the kernel phases, printed per launch by the launcher
#ifdef AMR_PHASE_PROF
__device__ unsigned long long g_phase[16][8];
#define PH_MARK(slot) do { if (prof) { long long _c = clock64(); ph_acc[slot] += _c - ph_t; ph_t = _c; } } while (0)
#else
#define PH_MARK(slot) do { } while (0)
#endif
constexpr int kTmaT = 32;                                  // tile edge
constexpr int kTmaWP = 44;                                 // prim plane row stride
constexpr int kTmaPL = (kTmaT + 2 * kGL) * kTmaWP;         // prim plane (40 rows: j = -4 .. 35)
constexpr int kTmaNH = kTmaT + 1;                          // F-hat faces per line: 0 .. T
constexpr int kTmaFXS = 36, kTmaFYS = 36;                  // row strides of the Lx / Ly planes (equal)
constexpr int kLandI = 0, kLandW = 4 * kTmaT * kTmaT, kLandE = kLandW + 4 * kTmaT * kGL,
              kLandS = kLandE + 4 * kTmaT * kGL, kLandN = kLandS + 4 * kGL * kTmaT,
              kLandSz = kLandN + 4 * kGL * kTmaT;
constexpr size_t kTmaSmem =
    sizeof(double) * (2 * kLandSz + 4 * kTmaPL + 4 * kTmaT * kTmaFXS + 4 * kTmaT * kTmaFYS) + 32 + 96 + 128;
constexpr size_t kTmaGroupSmem = kTmaSmem - 96 + 3 * 16 * 32;   // member descriptors [3][<=16]

// One 5-face segment (faces m0 .. m0+4 of a row or column; 7 segments cover faces -1 .. T+1): sliding 4-cell
// window of (p, T, u_n, u_t) over the prim planes (q = cell m0, cs = cell stride along the line, kn / kt = planes
// of the normal / tangential velocity), Central4 edge fluxes, and Eq. 9 F-hat at the 5 faces with f(m0-1) and
// f(m0+5) from the neighbouring segments' lanes, plus F-hat(m0+5) from the next segment (s unused: the values
// shuffled in across the line ends are garbage and never used).
// scale of the F-hat values c4_segment returns: 16 (c4_face16) x 24 (Eq. 9 as 26 f - (f- + f+)) with DIV4, else 16
template <bool DIV4>
__host__ __device__ constexpr double c4_fh_scale() { return DIV4 ? 1.0 / 384.0 : 0.0625; }

template <bool DIV4>
__device__ __forceinline__ void c4_segment(const double* __restrict__ q, int cs, int kn, int kt, double g_gm1,
                                           int s, double (&Fh)[6][4]) {
    constexpr int PL = kTmaPL;
    double p[4], Tt[4], un[4], ut[4];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int o = (c - 2) * cs;
        p[c + 1] = q[o]; Tt[c + 1] = q[PL + o]; un[c + 1] = q[kn * PL + o]; ut[c + 1] = q[kt * PL + o];
    }
    double f[5][4];
#pragma unroll
    for (int e = 0; e < 5; ++e) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { p[c] = p[c + 1]; Tt[c] = Tt[c + 1]; un[c] = un[c + 1]; ut[c] = ut[c + 1]; }
        const int o = (e + 1) * cs;
        p[3] = q[o]; Tt[3] = q[PL + o]; un[3] = q[kn * PL + o]; ut[3] = q[kt * PL + o];
        c4_face16(p, Tt, un, ut, g_gm1, f[e]);   // 16 f
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double lo = __shfl_up_sync(0xffffffffu, f[4][k], 4);
        const double hi = __shfl_down_sync(0xffffffffu, f[0][k], 4);
        (void)s;
        if (DIV4) {   // 24 F-hat = 26 f - (f- + f+): two operations per component instead of three
            Fh[0][k] = fma(26.0, f[0][k], -(lo + f[1][k]));
#pragma unroll
            for (int e = 1; e < 4; ++e) Fh[e][k] = fma(26.0, f[e][k], -(f[e - 1][k] + f[e + 1][k]));
            Fh[4][k] = fma(26.0, f[4][k], -(f[3][k] + hi));
        } else {
#pragma unroll
            for (int e = 0; e < 5; ++e) Fh[e][k] = f[e][k];
        }
        Fh[5][k] = __shfl_down_sync(0xffffffffu, Fh[0][k], 4);   // F-hat(m0+5): the next segment's first face
    }
}

template <int N, bool DIV4>
__global__ void __launch_bounds__(kTmaThreads, 1)
    stage_c4_tma_kernel(const StageArgs a, const __grid_constant__ C4Maps maps, const int ntiles) {
    constexpr int T = kTmaT, G = kGL, TILES = N / T, TT = TILES * TILES;
    constexpr int NN = N * N, PS = 4 * NN;
    constexpr int WP = kTmaWP, PL = kTmaPL, NH = kTmaNH, FXS = kTmaFXS, FYS = kTmaFYS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* const land = reinterpret_cast<double*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
    double* const prim = land + 2 * kLandSz;
    double* const dUx = prim + 4 * PL;           // [4][T][FXS] Lx = -dF-hat_x/dx of cell (i, j) at j*FXS + i
    double* const dUy = dUx + 4 * T * FXS;       // [4][T][FYS] Ly = -dF-hat_y/dy (components in U order)
    uint64_t* const mbar = reinterpret_cast<uint64_t*>(dUy + 4 * T * FYS);   // [4]
    // [3] descriptor ring: tile k in slot k % 3, k+1 fetched into (k+1) % 3 while warps may still be finishing
    // the epilogue of tile k-1 (there is no barrier after the epilogue)
    LeafDesc* const sDesc = reinterpret_cast<LeafDesc*>(mbar + 4);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double g = a.gamma, gm1 = g - 1.0, g_gm1 = g / gm1;   // g/(g-1): c4_face16
    const bool rk_un = a.stage > 1;
    const double ca = a.a, cb = a.b;
    const double dt = *a.dt;
#ifdef AMR_PHASE_PROF
    const bool prof = a.prof;
    long long ph_t = clock64();
    long long ph_acc[8] = {};
#endif

    auto issue = [&](int t, int b, const LeafDesc& d) {
        const int leaf = TILES == 1 ? t : t / TT;
        const int tt = TILES == 1 ? 0 : t - leaf * TT;
        const int tx = tt % TILES, ty = tt / TILES;
        const uint32_t mb = smem_u32(&mbar[b]);
        const uint32_t dst = smem_u32(land + b * kLandSz);
        mbar_expect_tx(mb, (kLandSz - 2 * 4 * T) * 8);   // S / N strips: 3 rows (row -4 / T+3 is never read)
        if (kBulk1DTile && TILES == 1) bulk_load(dst + kLandI * 8, a.Uin + (size_t)d.slot * 4 * N * N, 4 * N * N * 8, mb);
        else tma_load3(dst + kLandI * 8, &maps.in_int, tx * T, ty * T, 4 * d.slot, mb);
        const CUtensorMap* mw = &maps.in_we;
        int i0 = tx * T - G, z = 4 * d.slot;
        // a patch-edge strip comes from the neighbour's slot -- in another rank's pool over NVLink when the
        // neighbour is remote (halo_mode 2, LeafDesc.pad) -- or from the proxy of a C/F side
        auto peer = [&](int side) { return (d.pad >> (8 + 3 * side)) & 7; };
        if (tx == 0) {
            i0 = N - G; const int s = d.side[kW];
            if (s >= 0) { z = 4 * s; if (d.pad & (16 << kW)) mw = &maps.peer_we[peer(kW)]; }
            else { z = 4 * (-1 - s); mw = &maps.px_we; }
        }
        tma_load3(dst + kLandW * 8, mw, i0, ty * T, z, mb);
        mw = &maps.in_we; i0 = tx * T + T; z = 4 * d.slot;
        if (tx == TILES - 1) {
            i0 = 0; const int s = d.side[kE];
            if (s >= 0) { z = 4 * s; if (d.pad & (16 << kE)) mw = &maps.peer_we[peer(kE)]; }
            else { z = 4 * (-1 - s); mw = &maps.px_we; }
        }
        tma_load3(dst + kLandE * 8, mw, i0, ty * T, z, mb);
        const CUtensorMap* ms = &maps.in_sn;
        int j0 = ty * T - (G - 1); z = 4 * d.slot;
        if (ty == 0) {
            j0 = N - (G - 1); const int s = d.side[kS];
            if (s >= 0) { z = 4 * s; if (d.pad & (16 << kS)) ms = &maps.peer_sn[peer(kS)]; }
            else { z = 4 * (-1 - s); ms = &maps.px_sn; }
        }
        tma_load3(dst + kLandS * 8, ms, tx * T, j0, z, mb);
        ms = &maps.in_sn; j0 = ty * T + T; z = 4 * d.slot;
        if (ty == TILES - 1) {
            j0 = 0; const int s = d.side[kN];
            if (s >= 0) { z = 4 * s; if (d.pad & (16 << kN)) ms = &maps.peer_sn[peer(kN)]; }
            else { z = 4 * (-1 - s); ms = &maps.px_sn; }
        }
        tma_load3(dst + kLandN * 8, ms, tx * T, j0, z, mb);
    };

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.in_int)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.in_we)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.in_sn)) : "memory");
        for (int q = 0; q < 4; ++q) mbar_init(smem_u32(&mbar[q]), 1);   // [0,1] landing, [2,3] U^n
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // tile descriptors travel global -> shared by cp.async one tile ahead (no register round trip: a warp-uniform
    // load would otherwise be waited for at once to fill uniform registers)
    auto desc_ptr = [&](int t) { return a.leaves + (TILES == 1 ? t : t / TT); };
    LeafDesc dn{};
    if ((int)blockIdx.x < ntiles) {
        dn = *desc_ptr(blockIdx.x);
        if (tid == 0) {
            issue(blockIdx.x, 0, dn);
            if (rk_un) {                     // (tile offsets added below for N = 64)
                if (kBulk1DTile && TILES == 1) bulk_prefetch(a.Un + (size_t)dn.slot * 4 * N * N, 4 * N * N * 8);
                else tma_prefetch3(&maps.un_int, 0, 0, 4 * dn.slot);
            }
        }
    }

    // interior / epilogue cells of a thread: kC4Vec2 -- the adjacent pair (cr, cc), (cr, cc+1) of row
    // cr = 2 warp + lane/16 (16-byte shared / global accesses); else column ci = lane of rows 2 warp, 2 warp + 1
    const int ci = lane, cj0 = 2 * warp;
    const int cr = 2 * warp + (lane >> 4), cc = 2 * (lane & 15);
    const int seg_line = lane & 3, seg = lane < 28 ? lane >> 2 : 6;
    const bool seg_store = lane < 28;
    unsigned long long lam = 0ull;
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int b = k & 1;
        const int leaf = TILES == 1 ? t : t / TT;
        const int tt = TILES == 1 ? 0 : t - leaf * TT;
        const int tx = tt % TILES, ty = tt / TILES;
        const int ds = k % 3, dsn = ds == 2 ? 0 : ds + 1;
        const LeafDesc d = k == 0 ? dn : sDesc[ds];
        if (tid == 32 && t + (int)gridDim.x < ntiles) {
            const uint32_t dst = smem_u32(&sDesc[dsn]);
            const LeafDesc* src = desc_ptr(t + gridDim.x);
            cp_async16(dst, src);
            cp_async16(dst + 16, reinterpret_cast<const char*>(src) + 16);
        }
        const int base_off = (ty * T + cj0) * N + tx * T + ci;
        const double* L = land + b * kLandSz;
        PH_MARK(0);
        mbar_wait(smem_u32(&mbar[b]), (uint32_t)((k >> 1) & 1));
        PH_MARK(1);
        auto c2p = [&](double r, double m, double w, double E, int o) {
            const double ir = fast_rcp(r);
            const double u = m * ir, v = w * ir;
            const double p = gm1 * (E - 0.5 * (m * u + w * v));
            prim[o] = p;
            prim[PL + o] = p * ir;
            prim[2 * PL + o] = u;
            prim[3 * PL + o] = v;
        };
        double uc[2][4];
        if (kC4Vec2) {
            const double* s = L + kLandI + cr * T + cc;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double2 v = *reinterpret_cast<const double2*>(s + q * T * T);
                uc[0][q] = v.x;
                uc[1][q] = v.y;
            }
            double pr[4][2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double ir = fast_rcp(uc[e][0]);
                const double u = uc[e][1] * ir, v = uc[e][2] * ir;
                const double p = gm1 * (uc[e][3] - 0.5 * (uc[e][1] * u + uc[e][2] * v));
                pr[0][e] = p; pr[1][e] = p * ir; pr[2][e] = u; pr[3][e] = v;
            }
            const int o = (cr + G) * WP + cc + G;
#pragma unroll
            for (int q = 0; q < 4; ++q) *reinterpret_cast<double2*>(prim + q * PL + o) = make_double2(pr[q][0], pr[q][1]);
        } else {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const double* s = L + kLandI + (cj0 + r) * T + ci;
#pragma unroll
                for (int q = 0; q < 4; ++q) uc[r][q] = s[q * T * T];
                c2p(uc[r][0], uc[r][1], uc[r][2], uc[r][3], (cj0 + r + G) * WP + ci + G);
            }
        }
        static_assert(kC4Vec2, "the per-tile kernel converts interior cells in pairs");
        {   // strips: the 3 W / E columns and 3 S / N rows the faces read (cells -3..-1 and T..T+2; the TMA boxes
            // land 4 columns, the outermost is never read), one cell per thread of warps 0-11
            if (tid < 384) {
                int off, i, j, ps;
                if (tid < 192) {
                    const int wg = tid >= 96, e = tid - 96 * wg, jj = e / 3, c = e - 3 * jj + (wg == 0 ? 1 : 0);
                    off = (wg == 0 ? kLandW : kLandE) + jj * G + c; i = wg == 0 ? c - G : T + c; j = jj; ps = G * T;
                } else {
                    const int h = tid - 192, wg = h >= 96, e = h - 96 * wg, rr = e >> 5;
                    i = e & 31;
                    off = (wg == 0 ? kLandS : kLandN) + rr * T + i; j = wg == 0 ? rr - (G - 1) : T + rr; ps = (G - 1) * T;
                }
                c2p(L[off], L[off + ps], L[off + 2 * ps], L[off + 3 * ps], (j + G) * WP + i + G);
            }
        }
        if (tid == 32) cp_async_wait_all();      // descriptor of tile k+1 in sDesc[dsn] before (A)
        PH_MARK(2);
        __syncthreads();
        PH_MARK(3);
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_wait_read0();                   // the store of tile k-1 has read landing[b^1]
            if (t + (int)gridDim.x < ntiles) {
                const LeafDesc dn = sDesc[dsn];
                issue(t + gridDim.x, b ^ 1, dn);
                if (rk_un) {                     // U^n of tile k+1 towards L2
                    const int t2 = t + gridDim.x, tt2 = TILES == 1 ? 0 : t2 % TT;
                    if (kBulk1DTile && TILES == 1) bulk_prefetch(a.Un + (size_t)dn.slot * 4 * N * N, 4 * N * N * 8);
                    else tma_prefetch3(&maps.un_int, (tt2 % TILES) * T, (tt2 / TILES) * T, 4 * dn.slot);
                }
            }
            if (rk_un) {                         // U^n of tile k into the converted landing[b] interior
                const uint32_t mb = smem_u32(&mbar[2 + b]);
                mbar_expect_tx(mb, 4 * T * T * 8);
                if (kBulk1DTile && TILES == 1) bulk_load(smem_u32(land + b * kLandSz + kLandI), a.Un + (size_t)d.slot * 4 * N * N, 4 * N * N * 8, mb);
                else tma_load3(smem_u32(land + b * kLandSz + kLandI), &maps.un_int, tx * T, ty * T, 4 * d.slot, mb);
            }
        }
        PH_MARK(4);
        {
            // faces, Eq. 9 F-hat and the divergence of the segment's own cells m0 .. m0+4 (within [0, T))
            const int m0 = seg * 5 - 1;
            const int lvl = d.level;
            double Fh[6][4];
            if (warp < 8) {
                const int j = 4 * warp + seg_line;
                const double idx = c4_fh_scale<DIV4>() * a.geo.inv_dx[lvl];   // F-hat arrive scaled (c4_segment)
                c4_segment<DIV4>(prim + (j + G) * WP + G + m0, 1, 2, 3, g_gm1, seg, Fh);
                if (seg_store) {
#pragma unroll
                    for (int e = 0; e < 5; ++e)
                        if (m0 + e >= 0 && m0 + e < T)
#pragma unroll
                            for (int q = 0; q < 4; ++q) dUx[(q * T + j) * FXS + m0 + e] = -(Fh[e + 1][q] - Fh[e][q]) * idx;
                    const int sm = (d.cf | (d.cf >> 4)) & 15;
                    if (sm & 3) {   // flux registers of coarse/fine x sides: F-hat at faces 0 and T
#pragma unroll
                        for (int e = 0; e < 5; ++e)
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                if (m0 + e == 0 && tx == 0 && (sm & 1)) a.freg[(((size_t)d.slot * 4 + kW) * 4 + q) * N + ty * T + j] = c4_fh_scale<DIV4>() * Fh[e][q];
                                if (m0 + e == T && tx == TILES - 1 && (sm & 2)) a.freg[(((size_t)d.slot * 4 + kE) * 4 + q) * N + ty * T + j] = c4_fh_scale<DIV4>() * Fh[e][q];
                            }
                    }
                }
            } else {
                const int i = 4 * (warp - 8) + seg_line;
                const double idy = c4_fh_scale<DIV4>() * a.geo.inv_dy[lvl];
                c4_segment<DIV4>(prim + (m0 + G) * WP + G + i, WP, 3, 2, g_gm1, seg, Fh);
                if (seg_store) {
#pragma unroll
                    for (int e = 0; e < 5; ++e)
                        if (m0 + e >= 0 && m0 + e < T) {
                            double* o = dUy + (m0 + e) * FYS + i;
                            o[0 * T * FYS] = -(Fh[e + 1][0] - Fh[e][0]) * idy;
                            o[1 * T * FYS] = -(Fh[e + 1][2] - Fh[e][2]) * idy;
                            o[2 * T * FYS] = -(Fh[e + 1][1] - Fh[e][1]) * idy;
                            o[3 * T * FYS] = -(Fh[e + 1][3] - Fh[e][3]) * idy;
                        }
                    const int sm = (d.cf | (d.cf >> 4)) & 15;
                    if (sm & 12) {
#pragma unroll
                        for (int e = 0; e < 5; ++e) {
                            constexpr double fs = c4_fh_scale<DIV4>();
                            const double Fu[4] = {fs * Fh[e][0], fs * Fh[e][2], fs * Fh[e][1], fs * Fh[e][3]};
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                if (m0 + e == 0 && ty == 0 && (sm & 4)) a.freg[(((size_t)d.slot * 4 + kS) * 4 + q) * N + tx * T + i] = Fu[q];
                                if (m0 + e == T && ty == TILES - 1 && (sm & 8)) a.freg[(((size_t)d.slot * 4 + kN) * 4 + q) * N + tx * T + i] = Fu[q];
                            }
                        }
                    }
                }
            }
        }
        PH_MARK(5);
        __syncthreads();
        PH_MARK(6);
        const int lvl = d.level;
        const double idx = a.geo.inv_dx[lvl], idy = a.geo.inv_dy[lvl];
        const bool x_lo = tx == 0, x_hi = tx == TILES - 1, y_lo = ty == 0, y_hi = ty == TILES - 1;
        const int coarse_mask = d.cf & 15;
        // U^n (TMA, landed in landing[b]) in, U^(s) out through the same slots, then one TMA store per tile
        double* const sU = land + b * kLandSz + kLandI;
        if (rk_un) mbar_wait(smem_u32(&mbar[2 + b]), (uint32_t)((k >> 1) & 1));
        double out[2][4];
        if (kC4Vec2) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int o = (q * T + cr) * FXS + cc;   // FXS == FYS
                const double2 lx = *reinterpret_cast<const double2*>(dUx + o);
                const double2 ly = *reinterpret_cast<const double2*>(dUy + o);
                double v0 = uc[0][q] + dt * (lx.x + ly.x), v1 = uc[1][q] + dt * (lx.y + ly.y);
                double2* su = reinterpret_cast<double2*>(sU + (q * T + cr) * T + cc);
                if (rk_un) {
                    const double2 un = *su;
                    v0 = ca * un.x + cb * v0;
                    v1 = ca * un.y + cb * v1;
                }
                out[0][q] = v0;
                out[1][q] = v1;
                if (kC4Stg)
                    *reinterpret_cast<double2*>(a.Uout + (size_t)d.slot * PS + ((size_t)q * N + ty * T + cr) * N + tx * T + cc) =
                        make_double2(v0, v1);
                else *su = make_double2(v0, v1);
            }
        } else
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int o = (q * T + cj0 + r) * FXS + ci;   // FXS == FYS
                const double L = dUx[o] + dUy[o];
                double v = uc[r][q] + dt * L;
                double* su = sU + (q * T + cj0 + r) * T + ci;
                if (rk_un) v = ca * *su + cb * v;
                out[r][q] = v;
                if (kC4Stg) a.Uout[(size_t)d.slot * PS + ((size_t)q * N + ty * T + cj0 + r) * N + tx * T + ci] = v;
                else *su = v;
            }
        }
        if (!kC4Stg) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int j = kC4Vec2 ? cr : cj0 + r, i = kC4Vec2 ? cc + r : ci;
            const bool edge_cf = coarse_mask && (((coarse_mask & 1) && x_lo && i == 0) || ((coarse_mask & 2) && x_hi && i == T - 1) ||
                                                 ((coarse_mask & 4) && y_lo && j == 0) || ((coarse_mask & 8) && y_hi && j == T - 1));
            if (!edge_cf && !(d.pad & 1)) {   // covered patches (subcycling) are not leaves
                if (a.check || a.want_lambda)
                    leaf_check(out[r][0], out[r][1], out[r][2], out[r][3], g, idx, idy, a.check, a.want_lambda,
                               a.lam0 ? d.level : 0, a.err, d.slot, a.stage, (ty * T + j) * N + tx * T + i, lam);
            }
        }
        if (!kC4Stg) {   // (with direct stores, barrier (A) of the next tile orders the Lx / Ly reuse)
            __syncthreads();   // (C) U^(s) of the tile complete in shared memory
            if (tid == 0) {
                if (kBulk1DTile && TILES == 1) bulk_store(a.Uout + (size_t)d.slot * 4 * N * N, smem_u32(sU), 4 * N * N * 8);
                else tma_store3(&maps.out_int, tx * T, ty * T, 4 * d.slot, smem_u32(sU));
            }
        }
        PH_MARK(7);
    }
    if (tid == 0) bulk_wait0();
    if (a.want_lambda) {
        lam = warp_max_u64(lam);
        if (lane == 0 && lam) atomicMax(a.lambda_bits, lam);
    }
#ifdef AMR_PHASE_PROF
    if (prof && lane == 0)
        for (int p = 0; p < 8; ++p) atomicAdd(&g_phase[warp][p], (unsigned long long)ph_acc[p]);
#endif
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 3D view [z = slot*4 + var][j][i] of a pool of `npatch` n x n patches
bool encode_pool_map(CUtensorMap* m, const double* base, int n, int npatch, int bx, int by) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn || !base || npatch < 1) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)npatch * 4};
    const cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)n * n * 8};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 4};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n < 1) n = 1;
    }
    return n;
}

template <int N, bool DIV4>
cudaError_t launch_c4_tma_t(const StageArgs& a, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(stage_c4_tma_kernel<N, DIV4>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int ntiles = a.nleaves * (N / kTmaT) * (N / kTmaT);
    if (ntiles == 0) return cudaSuccess;
    C4Maps m;
    const double* px = a.proxy ? a.proxy : a.Uin;   // no proxies: never dereferenced, any valid map will do
    const int npx = a.proxy && a.nproxy > 0 ? a.nproxy : a.nslots;
    if (!encode_pool_map(&m.in_int, a.Uin, N, a.nslots, kTmaT, kTmaT) ||
        !encode_pool_map(&m.in_we, a.Uin, N, a.nslots, kGL, kTmaT) ||
        !encode_pool_map(&m.in_sn, a.Uin, N, a.nslots, kTmaT, kGL - 1) ||
        !encode_pool_map(&m.px_we, px, N, npx, kGL, kTmaT) ||
        !encode_pool_map(&m.px_sn, px, N, npx, kTmaT, kGL - 1) ||
        !encode_pool_map(&m.un_int, a.Un, N, a.nslots, kTmaT, kTmaT) ||
        !encode_pool_map(&m.out_int, a.Uout, N, a.nslots, kTmaT, kTmaT))
        return cudaErrorInvalidValue;
    for (int q = 0; q < a.npeers && q < 8; ++q)   // halo_mode 2: every rank's U^(s-1) as mapped in this process
        if (!encode_pool_map(&m.peer_we[q], a.peer_in[q], N, a.nslots, kGL, kTmaT) ||
            !encode_pool_map(&m.peer_sn[q], a.peer_in[q], N, a.nslots, kTmaT, kGL - 1))
            return cudaErrorInvalidValue;
    const int grid = ntiles < sm_count() ? ntiles : sm_count();
#ifdef AMR_PHASE_PROF
    static const bool prof = getenv("AMR_PHASE_PROF") != nullptr;
    StageArgs ap = a;
    ap.prof = prof ? 1 : 0;
    if (prof) {
        static unsigned long long zero[16][8] = {};
        cudaMemcpyToSymbolAsync(g_phase, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s);
    }
    stage_c4_tma_kernel<N, DIV4><<<grid, kTmaThreads, kTmaSmem, s>>>(ap, m, ntiles);
    if (prof) {
        unsigned long long h[16][8];
        cudaMemcpyFromSymbolAsync(h, g_phase, sizeof(h), 0, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const double per = (double)grid * ((ntiles + grid - 1) / grid);
        fprintf(stderr, "stage %d phase cycles per tile [top, mbar, c2p, waitA, issue, faces, waitB, epi]:\n", a.stage);
        for (int w = 0; w < 16; w += 5) {
            fprintf(stderr, "  w%02d", w);
            for (int p = 0; p < 8; ++p) fprintf(stderr, " %6.0f", h[w][p] / per);
            fprintf(stderr, "\n");
        }
    }
#else
    stage_c4_tma_kernel<N, DIV4><<<grid, kTmaThreads, kTmaSmem, s>>>(a, m, ntiles);
#endif
    return cudaGetLastError();
}


// ---------------------------------------------------------------- unfused stage (NEXT #1 fusion study)
// The GPU analogue of the paper's unfused task graph (Fig. 9 ssprk3Stage as its own task): four
// kernels per stage over the leaf list, with the intermediate fields round-tripping through HBM:
//   unf_prim:  halo gather + cons->prim (Central4: p, T, u, v; WENO: conserved copy) into padded tiles
//   unf_xflux / unf_yflux: face fluxes (the fused kernel's reconstruction + Riemann flux) into face arrays
//   unf_rk:    Eq. 9 F-hat, divergence, SSP-RK3, checks, Lambda, flux registers (ssprk3Stage)
// Same device functions and arithmetic as the fused kernels; scratch layout per leaf: W [4][n+8][n+8],
// fx [4][n][n+3], fy [4][n+3][n] (face m at m+1).
constexpr int kUnfG = kGL;

__global__ void unf_prim_kernel(const StageArgs a, int scheme) {
    const int n = a.geo.n, Wd = n + 2 * kUnfG;
    const long long per = (long long)Wd * Wd;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)a.nleaves * per) return;
    const int leaf = (int)(t / per), e = (int)(t - (long long)leaf * per);
    const int jj = e / Wd, ii = e - jj * Wd;
    int i = ii - kUnfG, j = jj - kUnfG;
    const bool xin = i >= 0 && i < n, yin = j >= 0 && j < n;
    if (!xin && !yin) return;                       // corner blocks are never read (A26)
    const LeafDesc d = a.leaves[leaf];
    const size_t nn = (size_t)n * n, PS = 4 * nn;
    int s = d.slot;
    bool own = true;
    if (i < 0) { s = d.side[kW]; i += n; own = false; }
    else if (i >= n) { s = d.side[kE]; i -= n; own = false; }
    else if (j < 0) { s = d.side[kS]; j += n; own = false; }
    else if (j >= n) { s = d.side[kN]; j -= n; own = false; }
    const double* b = (own || s >= 0) ? a.Uin + (size_t)s * PS : a.proxy + (size_t)(-1 - s) * PS;
    const size_t o = (size_t)j * n + i;
    const double r = b[o], m = b[nn + o], w = b[2 * nn + o], E = b[3 * nn + o];
    double* W = a.scratch + (size_t)leaf * 4 * per + e;
    if (scheme == 0) {
        const double ir = fast_rcp(r);
        const double u = m * ir, v = w * ir;
        const double p = (a.gamma - 1.0) * (E - 0.5 * (m * u + w * v));
        W[0] = p; W[per] = p * ir; W[2 * per] = u; W[3 * per] = v;
    } else {
        W[0] = r; W[per] = m; W[2 * per] = w; W[3 * per] = E;
    }
}

template <int SCHEME, int DIR>
__global__ void unf_flux_kernel(const StageArgs a) {
    const int n = a.geo.n, Wd = n + 2 * kUnfG, NF = n + 3;
    const long long per = (long long)Wd * Wd, fper = 4LL * n * NF;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)a.nleaves * n * NF) return;
    const int leaf = (int)(t / ((long long)n * NF)), e = (int)(t - (long long)leaf * n * NF);
    const double* W = a.scratch + (size_t)leaf * 4 * per;
    double* f = a.scratch + (size_t)a.nleaves * 4 * per + (size_t)(2 * leaf + DIR) * fper;
    double F[4];
    const double g = a.gamma, inv_gm1 = 1.0 / (g - 1.0);
    if (DIR == 0) {   // x faces: row j, face m = -1 .. n+1 (left of cell m)
        const int j = e / NF, m = e - j * NF - 1;
        const int o = (j + kUnfG) * Wd + m + kUnfG;
        if (SCHEME == 0) central4_flux(W + o - 2, 1, (int)per, 2, 3, inv_gm1, F);
        else {
            weno_rusanov<SCHEME == 1>(W + o - 3, 1, (int)per, 1, 2, g, a.eps, F);
            for (int k = 0; k < 4; ++k) F[k] *= kWenoFluxScale;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) f[((size_t)k * n + j) * NF + m + 1] = F[k];
    } else {          // y faces: column i, face m (below cell m); components stored in U order
        const int m = e / n - 1, i = e - (m + 1) * n;
        const int o = (m + kUnfG) * Wd + i + kUnfG;
        if (SCHEME == 0) central4_flux(W + o - 2 * Wd, Wd, (int)per, 3, 2, inv_gm1, F);
        else {
            weno_rusanov<SCHEME == 1>(W + o - 3 * Wd, Wd, (int)per, 2, 1, g, a.eps, F);
            for (int k = 0; k < 4; ++k) F[k] *= kWenoFluxScale;
        }
        f[((size_t)0 * NF + m + 1) * n + i] = F[0];
        f[((size_t)1 * NF + m + 1) * n + i] = F[2];
        f[((size_t)2 * NF + m + 1) * n + i] = F[1];
        f[((size_t)3 * NF + m + 1) * n + i] = F[3];
    }
}

__global__ void unf_rk_kernel(const StageArgs a) {
    const int n = a.geo.n, Wd = n + 2 * kUnfG, NF = n + 3;
    const long long per = (long long)Wd * Wd, fper = 4LL * n * NF;
    const size_t nn = (size_t)n * n, PS = 4 * nn;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)a.nleaves * (long long)nn) return;
    const int leaf = (int)(t / (long long)nn), c = (int)(t - (long long)leaf * nn);
    const int i = c % n, j = c / n;
    const LeafDesc d = a.leaves[leaf];
    const double* fx = a.scratch + (size_t)a.nleaves * 4 * per + (size_t)(2 * leaf) * fper;
    const double* fy = fx + fper;
    const double idx = a.geo.inv_dx[d.level], idy = a.geo.inv_dy[d.level];
    const bool div4 = a.div_order == 4;
    const int store_mask = (d.cf | (d.cf >> 4)) & 15, coarse_mask = d.cf & 15;
    const double c13 = 13.0 / 12.0, c24 = 1.0 / 24.0;
    const double dt = *a.dt;
    double o4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double* fr = fx + ((size_t)k * n + j) * NF + i + 1;   // fr[0] = f at face i
        const double fl = fr[0], fh = fr[1];
        const double Fl = div4 ? c13 * fl - c24 * (fr[-1] + fh) : fl;
        const double Fh = div4 ? c13 * fh - c24 * (fl + fr[2]) : fh;
        const double* fc = fy + ((size_t)k * NF + j + 1) * n + i;   // fc[0] = f at face j
        const double gl = fc[0], gh = fc[n];
        const double Gl = div4 ? c13 * gl - c24 * (fc[-n] + gh) : gl;
        const double Gh = div4 ? c13 * gh - c24 * (gl + fc[2 * n]) : gh;
        if (store_mask) {
            if (i == 0 && (store_mask & 1)) a.freg[(((size_t)d.slot * 4 + kW) * 4 + k) * n + j] = Fl;
            if (i == n - 1 && (store_mask & 2)) a.freg[(((size_t)d.slot * 4 + kE) * 4 + k) * n + j] = Fh;
            if (j == 0 && (store_mask & 4)) a.freg[(((size_t)d.slot * 4 + kS) * 4 + k) * n + i] = Gl;
            if (j == n - 1 && (store_mask & 8)) a.freg[(((size_t)d.slot * 4 + kN) * 4 + k) * n + i] = Gh;
        }
        const double L = -(Fh - Fl) * idx - (Gh - Gl) * idy;
        double v = a.Uin[(size_t)d.slot * PS + k * nn + c] + dt * L;
        if (a.stage > 1) v = a.a * a.Un[(size_t)d.slot * PS + k * nn + c] + a.b * v;
        o4[k] = v;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) a.Uout[(size_t)d.slot * PS + k * nn + c] = o4[k];
    const bool edge_cf = ((coarse_mask & 1) && i == 0) || ((coarse_mask & 2) && i == n - 1) ||
                         ((coarse_mask & 4) && j == 0) || ((coarse_mask & 8) && j == n - 1);
    unsigned long long lam = 0ull;
    if (!edge_cf && !(d.pad & 1)) {   // covered patches (subcycling) are not leaves
        if (a.check || a.want_lambda)
            leaf_check(o4[0], o4[1], o4[2], o4[3], a.gamma, idx, idy, a.check, a.want_lambda, a.lam0 ? d.level : 0,
                       a.err, d.slot, a.stage, c, lam);
    }
    if (a.want_lambda) {
        lam = warp_max_u64(lam);
        if ((threadIdx.x & 31) == 0 && lam) atomicMax(a.lambda_bits, lam);
    }
}

template <int SCHEME>
cudaError_t launch_unfused(const StageArgs& a, cudaStream_t s) {
    if (a.nleaves == 0) return cudaSuccess;
    if (!a.scratch) return cudaErrorInvalidValue;
    const int n = a.geo.n, Wd = n + 2 * kUnfG;
    const long long w = (long long)a.nleaves * Wd * Wd, f = (long long)a.nleaves * n * (n + 3),
                    c = (long long)a.nleaves * n * n;
    unf_prim_kernel<<<(unsigned)((w + 255) / 256), 256, 0, s>>>(a, SCHEME);
    unf_flux_kernel<SCHEME, 0><<<(unsigned)((f + 127) / 128), 128, 0, s>>>(a);
    unf_flux_kernel<SCHEME, 1><<<(unsigned)((f + 127) / 128), 128, 0, s>>>(a);
    unf_rk_kernel<<<(unsigned)((c + 255) / 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Central4 TMA kernel for small patches (groups)
// For patch sizes N = 8, 16 a 32 x 32 tile is a B x B block (B = 32/N) of same-level leaves formed on the host
// (consecutive leaves in level-Morton order: K = B^2 members, member m at block position demorton(m)); leaves
// that do not complete a block go to the one-CTA-per-tile kernel.  The tile is then processed exactly like a
// 32 x 32 patch tile of stage_c4_tma_kernel: the halo strips come from the members on the block edge, the
// interior from K boxes; the TMA issue is spread over the lanes of warp 0 (K + 4B <= 32 boxes); U^n in and
// U^(s) out by one box per member.  Landing layout: interior [K][4][N][N], W/E strips [B][4][N][4], S/N
// strips [B][4][4][N].
__device__ __forceinline__ int gm_x(int m) { return (m & 1) | ((m >> 1) & 2); }          // demorton, B <= 4
__device__ __forceinline__ int gm_y(int m) { return ((m >> 1) & 1) | ((m >> 2) & 2); }
__device__ __forceinline__ int gm_of(int x, int y) { return (x & 1) | ((y & 1) << 1) | ((x & 2) << 1) | ((y & 2) << 2); }

template <int N, bool DIV4>
__global__ void __launch_bounds__(kTmaThreads, 1)
    stage_c4_group_kernel(const StageArgs a, const __grid_constant__ C4Maps maps, const int ntiles) {
    constexpr int T = kTmaT, G = kGL, B = T / N, K = B * B;
    constexpr int NN = N * N;
    constexpr int WP = kTmaWP, PL = kTmaPL, FXS = kTmaFXS, FYS = kTmaFYS;
    static_assert(K + 4 * B <= 32, "one TMA box per lane of warp 0");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* const land = reinterpret_cast<double*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
    double* const prim = land + 2 * kLandSz;
    double* const dUx = prim + 4 * PL;
    double* const dUy = dUx + 4 * T * FXS;
    uint64_t* const mbar = reinterpret_cast<uint64_t*>(dUy + 4 * T * FYS);   // [4]
    LeafDesc* const sDesc = reinterpret_cast<LeafDesc*>(mbar + 4);          // [3][K] member descriptor ring

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double g = a.gamma, gm1 = g - 1.0, g_gm1 = g / gm1;   // g/(g-1): c4_face16
    const bool rk_un = a.stage > 1;
    const double ca = a.a, cb = a.b;
    const double dt = *a.dt;
    const int stride = gridDim.x;
#ifdef AMR_PHASE_PROF
    const bool prof = a.prof;
    long long ph_t = clock64();
    long long ph_acc[8] = {};
#endif

    // warp 0: arm the landing barrier, then one box per lane (interior of member `lane`, or one edge strip)
    // landing of a tile, split so that several warps can issue it: the arrival with the byte count and the member
    // interiors (lanes < K), and the 4B block-edge strips (strip e = 0 .. 4B-1 per lane); the strips may complete
    // before the count is armed (the mbarrier's tx-count goes transiently negative)
    auto issue_interior = [&](int b, const LeafDesc* D) {
        const uint32_t mb = smem_u32(&mbar[b]);
        const uint32_t dst = smem_u32(land + b * kLandSz);
        if (lane == 0) mbar_expect_tx(mb, kLandSz * 8);
        __syncwarp();
        if (lane < K) {
            if (kBulk1D && (D[0].pad & 2)) {   // consecutive member slots: the K interiors are one pool run
                if (lane == 0) bulk_load(dst + kLandI * 8, a.Uin + (size_t)D[0].slot * 4 * NN, K * 4 * NN * 8, mb);
            } else {
                tma_load3(dst + (kLandI + lane * 4 * NN) * 8, &maps.in_int, 0, 0, 4 * D[lane].slot, mb);
            }
        }
    };
    auto issue_strip = [&](int b, const LeafDesc* D, int e) {
        const uint32_t mb = smem_u32(&mbar[b]);
        const uint32_t dst = smem_u32(land + b * kLandSz);
        {
            const int side = e / B, r = e - side * B;
            const int m = side == kW ? gm_of(0, r) : side == kE ? gm_of(B - 1, r) : side == kS ? gm_of(r, 0) : gm_of(r, B - 1);
            const int s = D[m].side[side];
            const int z = s >= 0 ? 4 * s : 4 * (-1 - s);
            if (side < 2) {
                const CUtensorMap* mp = s >= 0 ? &maps.in_we : &maps.px_we;
                tma_load3(dst + ((side == kW ? kLandW : kLandE) + r * 16 * N) * 8, mp, side == kW ? N - G : 0, 0, z, mb);
            } else {
                const CUtensorMap* mp = s >= 0 ? &maps.in_sn : &maps.px_sn;
                tma_load3(dst + ((side == kS ? kLandS : kLandN) + r * 16 * N) * 8, mp, 0, side == kS ? N - G : 0, z, mb);
            }
        }
    };
    auto issue = [&](int b, const LeafDesc* D) {   // the whole landing from warp 0 (first tile)
        issue_interior(b, D);
        if (lane >= K && lane < K + 4 * B) issue_strip(b, D, lane - K);
    };
    auto fetch_desc = [&](int t, int slotbuf) {   // warp 1: member descriptors of tile t -> sDesc[slotbuf]
        // the compiler predicates this copy in every warp; lanes that copy nothing keep one common address (ncu
        // counted ~32 shared wavefronts per predicated-off warp instruction with lane-varying addresses; no time)
        const int m = lane < K ? lane : 0;
        const uint32_t dst = smem_u32(&sDesc[slotbuf * K + m]);
        const LeafDesc* src = a.leaves + (size_t)t * K + m;
        if (lane < K) {
            cp_async16(dst, src);
            cp_async16(dst + 16, reinterpret_cast<const char*>(src) + 16);
        }
    };

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.in_int)) : "memory");
        for (int q = 0; q < 4; ++q) mbar_init(smem_u32(&mbar[q]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1 && (int)blockIdx.x < ntiles) { fetch_desc(blockIdx.x, 0); cp_async_wait_all(); }
    __syncthreads();
    if (warp == 0 && (int)blockIdx.x < ntiles) issue(0, sDesc);

    const int seg_line = lane & 3, seg = lane < 28 ? lane >> 2 : 6;
    const bool seg_store = lane < 28;
    // N = 8: the L_x / L_y planes are column-swizzled (odd tile rows: column ^ 8), see the cell mapping below
    constexpr int SWZ = N == 8 ? 8 : 0;
    // interior / epilogue cells c = tid + 512 r: member m, in-member index w, tile position (ci[r], cj[r])
    int cm[2], cw[2], ci[2], cj[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int c = tid + 512 * r;
        if (N == 8) {
            // a half-warp (16 cells, 8-byte accesses) takes four 4-cell chunks of two x-neighbour members P, Q at rows
            // r0, r0 + 1 (r0 even): P r0 [0,4), P r0 [4,8), P r0+1 [0,4), Q r0+1 [4,8) -- the other half-warp of the
            // warp the same with P, Q swapped -- so that its accesses hit 16 distinct bank pairs on the member-major
            // landing (member stride = 0 mod 16 doubles: 8 row + col), on the prim planes (stride 44: 12 row + 8 X
            // + col) and on the swizzled L planes (stride 36: 4 row + 8 X + col, + 8 on odd rows); the member-major
            // mapping (two rows of one member) had 2-way conflicts on the latter two
            const int H = c >> 4, l = c & 15, unit = H >> 1, second = H & 1;
            const int pr = unit >> 2, r0 = 2 * (unit & 3);
            const int XA = 2 * (pr & 1), Y = pr >> 1;
            const int XP = XA + second, XQ = XA + 1 - second;
            const int ch = l >> 2, e = l & 3;
            const int X = ch == 3 ? XQ : XP, row = r0 + (ch >> 1), col = (ch == 1 || ch == 3 ? 4 : 0) + e;
            cm[r] = gm_of(X, Y);
            cw[r] = row * N + col;
            ci[r] = X * N + col;
            cj[r] = Y * N + row;
        } else {
            cm[r] = c / NN;
            cw[r] = c - cm[r] * NN;
            ci[r] = gm_x(cm[r]) * N + cw[r] % N;
            cj[r] = gm_y(cm[r]) * N + cw[r] / N;
        }
    }
    unsigned long long lam = 0ull;
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += stride, ++k) {
        const int b = k & 1;
        const int ds = k % 3, dsn = ds == 2 ? 0 : ds + 1;
        const LeafDesc* D = sDesc + ds * K;
        if (warp == 1 && t + stride < ntiles) fetch_desc(t + stride, dsn);
        const double* L = land + b * kLandSz;
        PH_MARK(0);
        mbar_wait(smem_u32(&mbar[b]), (uint32_t)((k >> 1) & 1));
        PH_MARK(1);
        auto c2p = [&](double r, double m, double w, double E, int o) {
            const double ir = fast_rcp(r);
            const double u = m * ir, v = w * ir;
            const double p = gm1 * (E - 0.5 * (m * u + w * v));
            prim[o] = p;
            prim[PL + o] = p * ir;
            prim[2 * PL + o] = u;
            prim[3 * PL + o] = v;
        };
        double uc[2][4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const double* s = L + kLandI + cm[r] * 4 * NN + cw[r];
#pragma unroll
            for (int q = 0; q < 4; ++q) uc[r][q] = s[q * NN];
            c2p(uc[r][0], uc[r][1], uc[r][2], uc[r][3], (cj[r] + G) * WP + ci[r] + G);
        }
        if (tid < 384) {   // strips: the 3 columns / rows the faces read (cells -3..-1, T..T+2), warps 0-11
            int off, i, j;
            if (tid < 192) {
                const int wg = tid >= 96, e = tid - 96 * wg;   // 0 W, 1 E
                j = e / 3;
                const int c = e - 3 * j + (wg == 0 ? 1 : 0), r = j / N;
                off = (wg == 0 ? kLandW : kLandE) + r * 16 * N + (j - r * N) * 4 + c;
                i = wg == 0 ? c - G : T + c;
            } else {
                const int h = tid - 192, wg = h >= 96, e = h - 96 * wg;   // 0 S, 1 N
                const int rr = (e >> 5) + (wg == 0 ? 1 : 0);
                i = e & 31;
                const int r = i / N;
                off = (wg == 0 ? kLandS : kLandN) + r * 16 * N + rr * N + (i - r * N);
                j = wg == 0 ? rr - G : T + rr;
            }
            const double* s = L + off;
            c2p(s[0], s[4 * N], s[8 * N], s[12 * N], (j + G) * WP + i + G);   // strip plane = 4 N doubles
        }
        if (warp == 1) cp_async_wait_all();      // member descriptors of tile k+1 before (A)
        PH_MARK(2);
        __syncthreads();   // (A)
        PH_MARK(3);
        // the TMA work of this point spread over three warps (on warp 0 alone it delayed that warp's face pass, and
        // every other warp waited for it at barrier (B))
        const bool more = t + stride < ntiles;
        const LeafDesc* Dn = sDesc + dsn * K;
        if (warp == 0) {                         // tile k+1: the arrival and the member interiors
            if (lane < K) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk_wait_read0();               // this lane's store of tile k-1 has read landing[b^1]
            }
            __syncwarp();
            if (more) issue_interior(b ^ 1, Dn);
        } else if (warp == kTmaThreads / 32 - 1) {   // tile k+1: the block-edge strips
            if (more && lane < 4 * B) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_strip(b ^ 1, Dn, lane);
            }
        } else if (warp == kTmaThreads / 64 - 1) {   // U^n of tile k into the converted landing[b]; tile k+1's to L2
            if (rk_un) {
                if (lane < K) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint32_t mb = smem_u32(&mbar[2 + b]);
                if (lane == 0) mbar_expect_tx(mb, 4 * T * T * 8);
                __syncwarp();
                if (kBulk1D && (D[0].pad & 2)) {
                    if (lane == 0) bulk_load(smem_u32(land + b * kLandSz + kLandI), a.Un + (size_t)D[0].slot * 4 * NN, K * 4 * NN * 8, mb);
                } else if (lane < K) {
                    tma_load3(smem_u32(land + b * kLandSz + kLandI + lane * 4 * NN), &maps.un_int, 0, 0, 4 * D[lane].slot, mb);
                }
                if (more && lane < K) {
                    if (kBulk1D && (Dn[0].pad & 2)) { if (lane == 0) bulk_prefetch(a.Un + (size_t)Dn[0].slot * 4 * NN, K * 4 * NN * 8); }
                    else tma_prefetch3(&maps.un_int, 0, 0, 4 * Dn[lane].slot);
                }
            }
        }
        PH_MARK(4);
        {
            const int m0 = seg * 5 - 1;
            const int lvl = D[0].level;
            double Fh[6][4];
            if (warp < 8) {
                const int j = 4 * warp + seg_line;
                const double idx = c4_fh_scale<DIV4>() * a.geo.inv_dx[lvl];
                c4_segment<DIV4>(prim + (j + G) * WP + G + m0, 1, 2, 3, g_gm1, seg, Fh);
                if (seg_store) {
#pragma unroll
                    for (int e = 0; e < 5; ++e)
                        if (m0 + e >= 0 && m0 + e < T)
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                dUx[(q * T + j) * FXS + ((m0 + e) ^ ((j & 1) * SWZ))] = -(Fh[e + 1][q] - Fh[e][q]) * idx;
                    const int r = j / N;
                    const LeafDesc& dw = D[gm_of(0, r)];
                    const LeafDesc& de = D[gm_of(B - 1, r)];
                    const int smw = (dw.cf | (dw.cf >> 4)) & 1, sme = (de.cf | (de.cf >> 4)) & 2;
                    if (smw | sme) {   // flux registers of coarse/fine x sides on the block edge
#pragma unroll
                        for (int e = 0; e < 5; ++e)
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                if (m0 + e == 0 && smw) a.freg[(((size_t)dw.slot * 4 + kW) * 4 + q) * N + j - r * N] = c4_fh_scale<DIV4>() * Fh[e][q];
                                if (m0 + e == T && sme) a.freg[(((size_t)de.slot * 4 + kE) * 4 + q) * N + j - r * N] = c4_fh_scale<DIV4>() * Fh[e][q];
                            }
                    }
                }
            } else {
                const int i = 4 * (warp - 8) + seg_line;
                const double idy = c4_fh_scale<DIV4>() * a.geo.inv_dy[lvl];
                c4_segment<DIV4>(prim + (m0 + G) * WP + G + i, WP, 3, 2, g_gm1, seg, Fh);
                if (seg_store) {
#pragma unroll
                    for (int e = 0; e < 5; ++e)
                        if (m0 + e >= 0 && m0 + e < T) {
                            double* o = dUy + (m0 + e) * FYS + (i ^ (((m0 + e) & 1) * SWZ));
                            o[0 * T * FYS] = -(Fh[e + 1][0] - Fh[e][0]) * idy;
                            o[1 * T * FYS] = -(Fh[e + 1][2] - Fh[e][2]) * idy;
                            o[2 * T * FYS] = -(Fh[e + 1][1] - Fh[e][1]) * idy;
                            o[3 * T * FYS] = -(Fh[e + 1][3] - Fh[e][3]) * idy;
                        }
                    const int r = i / N;
                    const LeafDesc& ds = D[gm_of(r, 0)];
                    const LeafDesc& dn = D[gm_of(r, B - 1)];
                    const int sms = (ds.cf | (ds.cf >> 4)) & 4, smn = (dn.cf | (dn.cf >> 4)) & 8;
                    if (sms | smn) {
#pragma unroll
                        for (int e = 0; e < 5; ++e) {
                            constexpr double fs = c4_fh_scale<DIV4>();
                            const double Fu[4] = {fs * Fh[e][0], fs * Fh[e][2], fs * Fh[e][1], fs * Fh[e][3]};
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                if (m0 + e == 0 && sms) a.freg[(((size_t)ds.slot * 4 + kS) * 4 + q) * N + i - r * N] = Fu[q];
                                if (m0 + e == T && smn) a.freg[(((size_t)dn.slot * 4 + kN) * 4 + q) * N + i - r * N] = Fu[q];
                            }
                        }
                    }
                }
            }
        }
        PH_MARK(5);
        __syncthreads();   // (B)
        PH_MARK(6);
        const int lvl = D[0].level;
        const double idx = a.geo.inv_dx[lvl], idy = a.geo.inv_dy[lvl];
        double* const sU = land + b * kLandSz + kLandI;
        if (rk_un) mbar_wait(smem_u32(&mbar[2 + b]), (uint32_t)((k >> 1) & 1));
        double out[2][4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int o = (q * T + cj[r]) * FXS + (ci[r] ^ ((cj[r] & 1) * SWZ));
                const double Lr = dUx[o] + dUy[o];
                double v = uc[r][q] + dt * Lr;
                double* su = sU + cm[r] * 4 * NN + q * NN + cw[r];
                if (rk_un) v = ca * *su + cb * v;
                out[r][q] = v;
                if (kC4Stg) a.Uout[(size_t)D[cm[r]].slot * 4 * NN + q * NN + cw[r]] = v;
                else *su = v;
            }
        }
        if (!kC4Stg) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const LeafDesc& dm = D[cm[r]];
            const int cmask = dm.cf & 15, ii = cw[r] % N, jj = cw[r] / N;
            const bool edge_cf = cmask && (((cmask & 1) && ii == 0) || ((cmask & 2) && ii == N - 1) ||
                                           ((cmask & 4) && jj == 0) || ((cmask & 8) && jj == N - 1));
            if (!edge_cf) {
                if (a.check || a.want_lambda)
                    leaf_check(out[r][0], out[r][1], out[r][2], out[r][3], g, idx, idy, a.check, a.want_lambda,
                               a.lam0 ? dm.level : 0, a.err, dm.slot, a.stage, cw[r], lam);
            }
        }
        if (!kC4Stg) {
            __syncthreads();   // (C) U^(s) of the tile complete in shared memory
            if (warp == 0 && lane < K) {
                if (kBulk1D && (D[0].pad & 2)) { if (lane == 0) bulk_store(a.Uout + (size_t)D[0].slot * 4 * NN, smem_u32(sU), K * 4 * NN * 8); }
                else tma_store3(&maps.out_int, 0, 0, 4 * D[lane].slot, smem_u32(sU + lane * 4 * NN));
            }
        }
        PH_MARK(7);
    }
    if (warp == 0 && lane < K) bulk_wait0();
    if (a.want_lambda) {
        lam = warp_max_u64(lam);
        if (lane == 0 && lam) atomicMax(a.lambda_bits, lam);
    }
#ifdef AMR_PHASE_PROF
    if (prof && lane == 0)
        for (int p = 0; p < 8; ++p) atomicAdd(&g_phase[warp][p], (unsigned long long)ph_acc[p]);
#endif
}

template <int N, bool DIV4>
cudaError_t launch_c4_group_t(const StageArgs& a, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(stage_c4_group_kernel<N, DIV4>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaGroupSmem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int ntiles = a.ngroups;
    if (ntiles == 0) return cudaSuccess;
    C4Maps m;
    const double* px = a.proxy ? a.proxy : a.Uin;
    const int npx = a.proxy && a.nproxy > 0 ? a.nproxy : a.nslots;
    if (!encode_pool_map(&m.in_int, a.Uin, N, a.nslots, N, N) ||
        !encode_pool_map(&m.in_we, a.Uin, N, a.nslots, kGL, N) ||
        !encode_pool_map(&m.in_sn, a.Uin, N, a.nslots, N, kGL) ||
        !encode_pool_map(&m.px_we, px, N, npx, kGL, N) ||
        !encode_pool_map(&m.px_sn, px, N, npx, N, kGL) ||
        !encode_pool_map(&m.un_int, a.Un, N, a.nslots, N, N) ||
        !encode_pool_map(&m.out_int, a.Uout, N, a.nslots, N, N))
        return cudaErrorInvalidValue;
    StageArgs ag = a;
    ag.leaves = a.gleaves;
    const int grid = ntiles < sm_count() ? ntiles : sm_count();
#ifdef AMR_PHASE_PROF
    static const bool prof = getenv("AMR_PHASE_PROF") != nullptr;
    ag.prof = prof ? 1 : 0;
    if (prof) {
        static unsigned long long zero[16][8] = {};
        cudaMemcpyToSymbolAsync(g_phase, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s);
    }
    stage_c4_group_kernel<N, DIV4><<<grid, kTmaThreads, kTmaGroupSmem, s>>>(ag, m, ntiles);
    if (prof) {
        unsigned long long h[16][8];
        cudaMemcpyFromSymbolAsync(h, g_phase, sizeof(h), 0, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const double per = (double)grid * ((ntiles + grid - 1) / grid);
        fprintf(stderr, "group N=%d stage %d phase cycles per tile [top, mbar, c2p, waitA, issue, faces, waitB, epi]:\n", N, a.stage);
        for (int w = 0; w < 16; w += 5) {
            fprintf(stderr, "  w%02d", w);
            for (int p = 0; p < 8; ++p) fprintf(stderr, " %6.0f", h[w][p] / per);
            fprintf(stderr, "\n");
        }
    }
#else
    stage_c4_group_kernel<N, DIV4><<<grid, kTmaThreads, kTmaGroupSmem, s>>>(ag, m, ntiles);
#endif
    return cudaGetLastError();
}

// ---------------------------------------------------------------- WENO5 stage kernel for 8^2 patches (groups)
// n = 8 with WENO5: the 32 x 32 tiles of 4 x 4 same-level leaves of the Central4 group kernel (StageArgs.gleaves,
// member m at block position demorton(m)), processed like one 32 x 32 tile of stage_kernel: one halo gather for
// the block (members' interiors, outer strips from the edge members' neighbours), 32 x 35 faces per direction
// instead of 16 x (8 x 11) -- the Eq. 9 stencil's extra faces and the halo are paid once per block -- and
// per-member epilogue addressing.  Faces between members are same-level faces.  (For n = 16 the 2 x 2 blocks
// measured slower on the AMR configs -- fewer, larger CTAs -- so n = 16 keeps one CTA per patch.)
template <int SCHEME, int N>
__global__ void __launch_bounds__(Block<32>::NT, Block<32>::MINB) stage_group_kernel(const StageArgs a) {
    constexpr int T = 32, G = kGL, B = T / N, K = B * B, NN = N * N;
    constexpr int NT = Block<T>::NT;
    constexpr int W = T + 2 * G, PL = W * W, NF = T + 3;
    constexpr int CPT = T * T / NT;
    constexpr size_t PS = 4 * (size_t)NN;
    extern __shared__ __align__(16) double smem[];
    double* sQ = smem;                 // [4][W][W] conserved
    double* sF = smem + 4 * PL;        // [4][T][NF] x-fluxes, then [4][NF][T] y-fluxes
    __shared__ LeafDesc sD[K];

    const int tid = threadIdx.x;
    if (tid < K) sD[tid] = a.gleaves[(size_t)blockIdx.x * K + tid];
    __syncthreads();
    auto mem = [](int x, int y) { return (x & 1) | ((y & 1) << 1) | ((x & 2) << 1) | ((y & 2) << 2); };

    // ---- halo gather (a1): plus-shaped block tile in 16-byte chunks; a chunk never straddles two members
    {
        constexpr int CR = W / 2, CB = T * CR, CS = G * T / 2, CV = CB + 2 * CS;
        static_assert(CV % NT == 0, "a thread's chunks sit at the same positions of the 4 planes");
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sQ);
#pragma unroll
        for (int r = 0; r < CV / NT; ++r) {   // each chunk position mapped once, then its 4 component planes
            const int f = tid + r * NT;
            int i, j;
            if (f < CB) { j = f / CR; i = 2 * (f - j * CR) - G; }
            else if (f < CB + CS) { int h = f - CB; j = h / (T / 2) - G; i = 2 * (h - (j + G) * (T / 2)); }
            else { int h = f - CB - CS; j = h / (T / 2); i = 2 * (h - j * (T / 2)); j += T; }
            const int mx = i < 0 ? 0 : (i >= T ? B - 1 : i / N), my = j < 0 ? 0 : (j >= T ? B - 1 : j / N);
            const LeafDesc& d = sD[mem(mx, my)];
            int pi = i - mx * N, pj = j - my * N, sl = d.slot, sd = -1;
            bool halo = true;
            if (pi < 0) { sd = kW; pi += N; }
            else if (pi >= N) { sd = kE; pi -= N; }
            else if (pj < 0) { sd = kS; pj += N; }
            else if (pj >= N) { sd = kN; pj -= N; }
            else halo = false;
            if (halo) sl = d.side[sd];
            const double* base = !halo ? a.Uin + (size_t)sl * PS
                                       : (sl >= 0 ? side_source(a, d, sd) + (size_t)sl * PS : a.proxy + (size_t)(-1 - sl) * PS);
            const uint32_t dst = sb + (uint32_t)(((j + G) * W + (i + G)) * 8);
            const double* src = base + pj * N + pi;
#pragma unroll
            for (int kq = 0; kq < 4; ++kq) cp_async16(dst + (uint32_t)(kq * PL * 8), src + kq * NN);
        }
        cp_async_wait_all();
    }
    __syncthreads();

    const double g = a.gamma;
    const int lvl = sD[0].level;
    const double idx = a.geo.inv_dx[lvl], idy = a.geo.inv_dy[lvl];
    const bool div4 = a.div_order == 4;
    // Eq. 9 as 24 F-hat = 26 f - (f- + f+): the 1/24 goes into the divergence and the flux registers
    const double fsc = (SCHEME == 0 ? 1.0 : kWenoFluxScale) * (div4 ? 1.0 / 24.0 : 1.0), idx24 = fsc * idx, idy24 = fsc * idy;

    // ---- x faces (a4-a6): face m (left of cell m), row j (packing the idle threads of the last x pass with y faces,
    // as stage_kernel<., 32> does, was 1.3 % slower here)
    for (int e = tid; e < T * NF; e += NT) {
        int j = e / NF, m = e - j * NF - 1;
        int o = (j + G) * W + (m + G);
        double f[4];
        weno_rusanov<SCHEME == 1>(sQ + o - 3, 1, PL, 1, 2, g, a.eps, f);
#pragma unroll
        for (int q = 0; q < 4; ++q) sF[(q * T + j) * NF + m + 1] = f[q];
    }
    __syncthreads();
    double acc[CPT][4];
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
        const int c = tid + r * NT, i = c % T, j = c / T;
        const LeafDesc& dw = sD[mem(0, j / N)];
        const LeafDesc& de = sD[mem(B - 1, j / N)];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double* fr = sF + (q * T + j) * NF + i + 1;
            double fl = fr[0], fh = fr[1];
            double Fl = div4 ? fma(26.0, fl, -(fr[-1] + fh)) : fl;   // 24 F-hat
            double Fh = div4 ? fma(26.0, fh, -(fl + fr[2])) : fh;
            acc[r][q] = -(Fh - Fl) * idx24;
            if (i == 0 && ((dw.cf | (dw.cf >> 4)) & 1))   // flux registers of C/F sides on the block edge
                a.freg[(((size_t)dw.slot * 4 + kW) * 4 + q) * N + j % N] = fsc * Fl;
            if (i == T - 1 && ((de.cf | (de.cf >> 4)) & 2))
                a.freg[(((size_t)de.slot * 4 + kE) * 4 + q) * N + j % N] = fsc * Fh;
        }
    }
    __syncthreads();
    // ---- y faces: face m (below cell m), column i; normal momentum is component 2
    for (int e = tid; e < T * NF; e += NT) {
        int m = e / T - 1, i = e - (m + 1) * T;
        int o = (m + G) * W + (i + G);
        double f[4];
        weno_rusanov<SCHEME == 1>(sQ + o - 3 * W, W, PL, 2, 1, g, a.eps, f);
        sF[(0 * NF + m + 1) * T + i] = f[0];
        sF[(1 * NF + m + 1) * T + i] = f[2];
        sF[(2 * NF + m + 1) * T + i] = f[1];
        sF[(3 * NF + m + 1) * T + i] = f[3];
    }
    __syncthreads();

    // ---- y divergence, SSP-RK3 combination (a8), checks, Lambda (a9), per member
    const double dt = *a.dt;
    unsigned long long lam = 0ull;
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
        const int c = tid + r * NT, i = c % T, j = c / T;
        const LeafDesc& dm = sD[mem(i / N, j / N)];
        const LeafDesc& ds = sD[mem(i / N, 0)];
        const LeafDesc& dn = sD[mem(i / N, B - 1)];
        const int li = i % N, lj = j % N;
        const size_t off = (size_t)lj * N + li;
        const double* pin = a.Uin + (size_t)dm.slot * PS;
        const double* pn = a.Un + (size_t)dm.slot * PS;
        double* po = a.Uout + (size_t)dm.slot * PS;
        double o4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double* fr = sF + (q * NF + j + 1) * T + i;
            double fl = fr[0], fh = fr[T];
            double Fl = div4 ? fma(26.0, fl, -(fr[-T] + fh)) : fl;   // 24 F-hat
            double Fh = div4 ? fma(26.0, fh, -(fl + fr[2 * T])) : fh;
            double L = acc[r][q] - (Fh - Fl) * idy24;
            if (j == 0 && ((ds.cf | (ds.cf >> 4)) & 4)) a.freg[(((size_t)ds.slot * 4 + kS) * 4 + q) * N + li] = fsc * Fl;
            if (j == T - 1 && ((dn.cf | (dn.cf >> 4)) & 8)) a.freg[(((size_t)dn.slot * 4 + kN) * 4 + q) * N + li] = fsc * Fh;
            double v = __ldg(pin + q * NN + off) + dt * L;
            if (a.stage > 1) v = a.a * __ldg(pn + q * NN + off) + a.b * v;
            o4[q] = v;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) po[q * NN + off] = o4[q];
        const int cm = dm.cf & 15;   // C/F coarse sides are block-edge sides (members are same-level neighbours)
        const bool edge_cf = ((cm & 1) && li == 0) || ((cm & 2) && li == N - 1) || ((cm & 4) && lj == 0) ||
                             ((cm & 8) && lj == N - 1);
        if (!edge_cf) {
            if (a.check || a.want_lambda)
                leaf_check(o4[0], o4[1], o4[2], o4[3], g, idx, idy, a.check, a.want_lambda, a.lam0 ? dm.level : 0,
                           a.err, dm.slot, a.stage, (int)off, lam);
        }
    }
    if (a.want_lambda) {
        lam = warp_max_u64(lam);
        if ((tid & 31) == 0 && lam) atomicMax(a.lambda_bits, lam);
    }
}

template <int SCHEME, int N>
cudaError_t launch_group_t(const StageArgs& a, cudaStream_t s) {
    constexpr size_t smem = stage_smem<SCHEME, 32>();
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(stage_group_kernel<SCHEME, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    if (a.ngroups == 0) return cudaSuccess;
    stage_group_kernel<SCHEME, N><<<a.ngroups, Block<32>::NT, smem, s>>>(a);
    return cudaGetLastError();
}

template <int SCHEME>
cudaError_t launch_stage_s(const StageArgs& a, cudaStream_t s) {
    int T = a.geo.n / a.tiles;
    if (SCHEME == 0) {
        if (a.variant == 0 && a.geo.n == 16 && a.gleaves) {
            cudaError_t e = a.div_order == 4 ? launch_c4_group_t<16, true>(a, s) : launch_c4_group_t<16, false>(a, s);
            if (e != cudaSuccess || a.nleaves == 0) return e;   // then the leaves outside complete blocks
            return launch_c4_t<16>(a, s);
        }
        if (a.variant == 0 && a.geo.n == 8 && a.gleaves) {
            cudaError_t e = a.div_order == 4 ? launch_c4_group_t<8, true>(a, s) : launch_c4_group_t<8, false>(a, s);
            if (e != cudaSuccess || a.nleaves == 0) return e;
            return launch_c4_t<8>(a, s);
        }
        if (a.variant == 0 && a.geo.n == 32)
            return a.div_order == 4 ? launch_c4_tma_t<32, true>(a, s) : launch_c4_tma_t<32, false>(a, s);
        if (a.variant == 0 && a.geo.n == 64)
            return a.div_order == 4 ? launch_c4_tma_t<64, true>(a, s) : launch_c4_tma_t<64, false>(a, s);
        switch (a.geo.n) {
            case 8: return launch_c4_t<8>(a, s);
            case 16: return launch_c4_t<16>(a, s);
            case 32: return launch_c4_t<32>(a, s);
            case 64: return launch_c4_t<64>(a, s);
            default: return cudaErrorInvalidValue;
        }
    }
    if (a.variant == 0 && a.gleaves && a.geo.n == 8) {   // WENO 4 x 4 block tiles, then the rest
        cudaError_t e = launch_group_t<SCHEME, 8>(a, s);
        if (e != cudaSuccess || a.nleaves == 0) return e;
    }
    if (T == 8) return launch_stage_t<SCHEME, 8>(a, s);
    if (T == 16) return launch_stage_t<SCHEME, 16>(a, s);
    if (T == 32) return launch_stage_t<SCHEME, 32>(a, s);
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- coarse values for prolongation (O8)
// Value of component k of coarse cell (rx, ry) given relative to the parent patch
// (level l-1, position Pp, Qp); out-of-domain cells follow the BC rule (O7).
// Uold != nullptr (subcycling, S2): the coarse level linearly in time, Uold + tfrac (U - Uold), before the BC sign.
__device__ __forceinline__ double coarse_value(const double* U, const int32_t* coarse, int n, int lc, int Pp, int Qp,
                                               int rx, int ry, int k, const Geometry& geo, const double* Uold,
                                               double tfrac) {
    double sgn = 1.0;
    int Ig = Pp * n + rx, Jg = Qp * n + ry;
    const int NX = geo.nc[0][lc], NY = geo.nc[1][lc];
    if (Ig < 0 && geo.bc[0] != kBcPeriodic) {
        if (geo.bc[0] == kBcTransmissive) Ig = 0; else { Ig = -1 - Ig; if (k == 1) sgn = -1.0; }
    } else if (Ig >= NX && geo.bc[1] != kBcPeriodic) {
        if (geo.bc[1] == kBcTransmissive) Ig = NX - 1; else { Ig = 2 * NX - 1 - Ig; if (k == 1) sgn = -1.0; }
    }
    if (Jg < 0 && geo.bc[2] != kBcPeriodic) {
        if (geo.bc[2] == kBcTransmissive) Jg = 0; else { Jg = -1 - Jg; if (k == 2) sgn = -1.0; }
    } else if (Jg >= NY && geo.bc[3] != kBcPeriodic) {
        if (geo.bc[3] == kBcTransmissive) Jg = NY - 1; else { Jg = 2 * NY - 1 - Jg; if (k == 2) sgn = -1.0; }
    }
    rx = Ig - Pp * n;
    ry = Jg - Qp * n;
    int bx = rx < 0 ? -1 : (rx >= n ? 1 : 0);
    int by = ry < 0 ? -1 : (ry >= n ? 1 : 0);
    int slot = coarse[(by + 1) * 3 + (bx + 1)];
    int lx = rx - bx * n, ly = ry - by * n;
    const size_t o = (size_t)slot * 4 * n * n + (size_t)k * n * n + (size_t)ly * n + lx;
    double v = U[o];
    if (Uold) v = Uold[o] + tfrac * (v - Uold[o]);
    return sgn * v;
}

__device__ __forceinline__ double mc_limiter(double a, double b) {
    if (a * b <= 0.0) return 0.0;
    double m = fabs(a + b) * 0.5;   // min of the three by comparisons (fmin would drop a NaN; same values otherwise)
    if (2.0 * fabs(a) < m) m = 2.0 * fabs(a);
    if (2.0 * fabs(b) < m) m = 2.0 * fabs(b);
    return a > 0.0 ? m : -m;
}

// O8 for fine cell (I, J) (global at level l, may be unwrapped by one patch)
__device__ __forceinline__ double prolong_value(const double* U, const int32_t* coarse, int n, int l, int P, int Q,
                                                int I, int J, int k, const Geometry& geo, const double* Uold = nullptr,
                                                double tfrac = 0.0) {
    int Pp = P >> 1, Qp = Q >> 1;
    int Ic = I >> 1, Jc = J >> 1;   // arithmetic shift = floor division by 2
    int ax = I & 1, by = J & 1;
    int rx = Ic - Pp * n, ry = Jc - Qp * n;
    double V = coarse_value(U, coarse, n, l - 1, Pp, Qp, rx, ry, k, geo, Uold, tfrac);
    double sx = mc_limiter(V - coarse_value(U, coarse, n, l - 1, Pp, Qp, rx - 1, ry, k, geo, Uold, tfrac),
                           coarse_value(U, coarse, n, l - 1, Pp, Qp, rx + 1, ry, k, geo, Uold, tfrac) - V);
    double sy = mc_limiter(V - coarse_value(U, coarse, n, l - 1, Pp, Qp, rx, ry - 1, k, geo, Uold, tfrac),
                           coarse_value(U, coarse, n, l - 1, Pp, Qp, rx, ry + 1, k, geo, Uold, tfrac) - V);
    double t = V + ((2 * ax - 1) * 0.25) * sx;
    return t + ((2 * by - 1) * 0.25) * sy;
}

// ---------------------------------------------------------------- ghost / proxy fill (O7, O8)
__global__ void ghost_kernel(const ProxyTask* __restrict__ tasks, int ntasks, int g, const AuxArgs a) {
    const int n = a.geo.n;
    const int per = g * n;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)ntasks * per) return;
    const int task = (int)(t / per), e = (int)(t - (long long)task * per);
    const ProxyTask pt = tasks[task];
    const int along = e % n, depth = e / n;
    int li, lj;   // ghost cell, patch-local
    switch (pt.side) {
        case kW: li = depth - g; lj = along; break;
        case kE: li = n + depth; lj = along; break;
        case kS: li = along; lj = depth - g; break;
        default: li = along; lj = n + depth; break;
    }
    const int pli = pt.side == kW ? li + n : (pt.side == kE ? li - n : li);
    const int plj = pt.side == kS ? lj + n : (pt.side == kN ? lj - n : lj);
    const size_t nn = (size_t)n * n;
    double* dst = a.proxy + (size_t)pt.proxy * 4 * nn + (size_t)plj * n + pli;
    if (pt.kind == 0) {
        // physical boundary: source is an interior cell of the leaf itself (A25)
        int bc = a.geo.bc[pt.side];
        int si = li, sj = lj;
        double sx = 1.0, sy = 1.0;
        if (pt.side == kW) { si = bc == kBcTransmissive ? 0 : -1 - li; if (bc == kBcReflective) sx = -1.0; }
        if (pt.side == kE) { si = bc == kBcTransmissive ? n - 1 : 2 * n - 1 - li; if (bc == kBcReflective) sx = -1.0; }
        if (pt.side == kS) { sj = bc == kBcTransmissive ? 0 : -1 - lj; if (bc == kBcReflective) sy = -1.0; }
        if (pt.side == kN) { sj = bc == kBcTransmissive ? n - 1 : 2 * n - 1 - lj; if (bc == kBcReflective) sy = -1.0; }
        const double* src = a.U + (size_t)pt.slot * 4 * nn + (size_t)sj * n + si;
        dst[0] = src[0];
        dst[nn] = sx * src[nn];
        dst[2 * nn] = sy * src[2 * nn];
        dst[3 * nn] = src[3 * nn];
    } else {
        const int I = pt.P * n + li, J = pt.Q * n + lj;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            dst[k * nn] = prolong_value(a.Uc, pt.coarse, n, pt.level, pt.P, pt.Q, I, J, k, a.geo, a.Uold, a.tfrac);
    }
}

// One CTA per proxy strip: the coarse values a C/F strip's prolongation reads (its 2 x n/2 coarse cells and their
// slope neighbours, time-interpolated for subcycling) are evaluated ONCE into shared memory by coarse_value, then
// every fine ghost cell applies prolong_value's arithmetic to them -- bitwise the per-cell kernel's result with
// ~16x fewer global reads (each coarse value was re-read by up to 20 fine cells x stencil points).
constexpr int kGhostThreads = 128;
// One C/F or physical-boundary ghost strip by a group of nth threads (this one: tid; group-uniform pt; cs: shared
// staging of 4 (g/2 + 2)(n/2 + 2) doubles; sync() orders the group between staging and use).  ghost_tile_kernel:
// one block per strip; the fused post-stage kernel: one warp per strip.
template <class Sync>
__device__ __forceinline__ void ghost_strip(const ProxyTask& pt, int g, const AuxArgs& a, double* cs, int tid, int nth,
                                            Sync sync) {
    const int n = a.geo.n;
    const size_t nn = (size_t)n * n;
    // ghost cells of the strip, patch-local (li, lj) ranges
    int li0, li1, lj0, lj1;
    switch (pt.side) {
        case kW: li0 = -g; li1 = -1; lj0 = 0; lj1 = n - 1; break;
        case kE: li0 = n; li1 = n + g - 1; lj0 = 0; lj1 = n - 1; break;
        case kS: li0 = 0; li1 = n - 1; lj0 = -g; lj1 = -1; break;
        default: li0 = 0; li1 = n - 1; lj0 = n; lj1 = n + g - 1; break;
    }
    const int ncell = (li1 - li0 + 1) * (lj1 - lj0 + 1);
    if (pt.kind == 0) {   // physical boundary: a plain copy (A25), as in ghost_kernel
        const int bc = a.geo.bc[pt.side];
        for (int e = tid; e < ncell; e += nth) {
            const int w = li1 - li0 + 1, li = li0 + e % w, lj = lj0 + e / w;
            const int pli = pt.side == kW ? li + n : (pt.side == kE ? li - n : li);
            const int plj = pt.side == kS ? lj + n : (pt.side == kN ? lj - n : lj);
            double* dst = a.proxy + (size_t)pt.proxy * 4 * nn + (size_t)plj * n + pli;
            int si = li, sj = lj;
            double sx = 1.0, sy = 1.0;
            if (pt.side == kW) { si = bc == kBcTransmissive ? 0 : -1 - li; if (bc == kBcReflective) sx = -1.0; }
            if (pt.side == kE) { si = bc == kBcTransmissive ? n - 1 : 2 * n - 1 - li; if (bc == kBcReflective) sx = -1.0; }
            if (pt.side == kS) { sj = bc == kBcTransmissive ? 0 : -1 - lj; if (bc == kBcReflective) sy = -1.0; }
            if (pt.side == kN) { sj = bc == kBcTransmissive ? n - 1 : 2 * n - 1 - lj; if (bc == kBcReflective) sy = -1.0; }
            const double* src = a.U + (size_t)pt.slot * 4 * nn + (size_t)sj * n + si;
            dst[0] = src[0];
            dst[nn] = sx * src[nn];
            dst[2 * nn] = sy * src[2 * nn];
            dst[3 * nn] = src[3 * nn];
        }
        return;
    }
    const int Pp = pt.P >> 1, Qp = pt.Q >> 1;
    // coarse cells (relative to the parent) the strip reads: its own coarse cells +- 1 for the slopes
    const int rx0 = ((pt.P * n + li0) >> 1) - Pp * n - 1, rx1 = ((pt.P * n + li1) >> 1) - Pp * n + 1;
    const int ry0 = ((pt.Q * n + lj0) >> 1) - Qp * n - 1, ry1 = ((pt.Q * n + lj1) >> 1) - Qp * n + 1;
    const int wx = rx1 - rx0 + 1, wy = ry1 - ry0 + 1, plane = wx * wy;
    // staged in batches of kGhostBatch values per thread: all loads of a batch are issued before the first store
    // (one dependent global round trip per batch instead of one per value)
    constexpr int kGhostBatch = 8;
    for (int e0 = tid; e0 < 4 * plane; e0 += kGhostBatch * nth) {
        double v[kGhostBatch];
#pragma unroll
        for (int b = 0; b < kGhostBatch; ++b) {
            const int e = e0 + b * nth;
            if (e < 4 * plane) {
                const int k = e / plane, r = e - k * plane, ry = ry0 + r / wx, rx = rx0 + r % wx;
                v[b] = coarse_value(a.Uc, pt.coarse, n, pt.level - 1, Pp, Qp, rx, ry, k, a.geo, a.Uold, a.tfrac);
            }
        }
#pragma unroll
        for (int b = 0; b < kGhostBatch; ++b)
            if (e0 + b * nth < 4 * plane) cs[e0 + b * nth] = v[b];
    }
    sync();
    for (int e = tid; e < ncell; e += nth) {
        const int w = li1 - li0 + 1, li = li0 + e % w, lj = lj0 + e / w;
        const int pli = pt.side == kW ? li + n : (pt.side == kE ? li - n : li);
        const int plj = pt.side == kS ? lj + n : (pt.side == kN ? lj - n : lj);
        double* dst = a.proxy + (size_t)pt.proxy * 4 * nn + (size_t)plj * n + pli;
        const int I = pt.P * n + li, J = pt.Q * n + lj;
        const int ax = I & 1, by = J & 1;
        const int cx = (I >> 1) - Pp * n - rx0, cy = (J >> 1) - Qp * n - ry0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {   // prolong_value's arithmetic on the shared coarse values
            const double* c = cs + k * plane + cy * wx + cx;
            const double V = c[0];
            const double sx = mc_limiter(V - c[-1], c[1] - V);
            const double sy = mc_limiter(V - c[-wx], c[wx] - V);
            const double t = V + ((2 * ax - 1) * 0.25) * sx;
            dst[k * nn] = t + ((2 * by - 1) * 0.25) * sy;
        }
    }
}

// ---------------------------------------------------------------- prolongation of new patches (O8)
__global__ void prolong_kernel(const ProlongTask* __restrict__ tasks, int ntasks, const AuxArgs a) {
    const int n = a.geo.n;
    const size_t nn = (size_t)n * n;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)ntasks * (long long)nn) return;
    const int task = (int)(t / (long long)nn), e = (int)(t - (long long)task * nn);
    const ProlongTask pt = tasks[task];
    const int li = e % n, lj = e / n;
    const int I = pt.P * n + li, J = pt.Q * n + lj;
    double* dst = a.Uw + (size_t)pt.slot * 4 * nn + e;
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[k * nn] = prolong_value(a.U, pt.coarse, n, pt.level, pt.P, pt.Q, I, J, k, a.geo);
}

// ---------------------------------------------------------------- restriction (O9)
// O9 for parent cell e of restriction task `task`: ((a + b) + (c + d)) * 0.25 of the 2 x 2 children cells
__device__ __forceinline__ void restrict_cell(const RestrictTask* __restrict__ tasks, long long t, const AuxArgs& a) {
    const int n = a.geo.n;
    const size_t nn = (size_t)n * n;
    const int task = (int)(t / (long long)nn), e = (int)(t - (long long)task * nn);
    const int i = e % n, j = e / n;
    const int ca = (2 * i) / n, cb = (2 * j) / n;
    const int fi = 2 * i - ca * n, fj = 2 * j - cb * n;
    // the two fields this cell needs, loaded directly (a copy of the task indexed by ca + 2 cb went through local memory)
    const int child = tasks[task].child[ca + 2 * cb], parent = tasks[task].parent;
    const double* f = a.U + (size_t)child * 4 * nn + (size_t)fj * n + fi;   // children (read)
    double* dst = a.Uw + (size_t)parent * 4 * nn + e;
    // every child value loaded before the first store (the stores may alias the loads as far as the compiler knows,
    // so a load-store sequence per component would be four dependent round trips); fi even: 16-byte pairs
    double2 v[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double* fk = f + k * nn;
        v[k][0] = *reinterpret_cast<const double2*>(fk);
        v[k][1] = *reinterpret_cast<const double2*>(fk + n);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[k * nn] = ((v[k][0].x + v[k][0].y) + (v[k][1].x + v[k][1].y)) * 0.25;
}

__global__ void restrict_kernel(const RestrictTask* __restrict__ tasks, int ntasks, const AuxArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)ntasks * a.geo.n * a.geo.n) return;
    restrict_cell(tasks, t, a);
}


// ---------------------------------------------------------------- flux correction (O12)
__global__ void __launch_bounds__(kGhostThreads) ghost_tile_kernel(const ProxyTask* __restrict__ tasks, int g,
                                                                  const AuxArgs a) {
    extern __shared__ double cs[];   // [4][ry span][rx span]
    const ProxyTask pt = tasks[blockIdx.x];
    ghost_strip(pt, g, a, cs, threadIdx.x, blockDim.x, [] { __syncthreads(); });
}

// O12 correction of one coarse boundary cell (work item t of 4 n per reflux task); Lambda (stage 3) into lam
__device__ __forceinline__ void reflux_cell(const RefluxTask* __restrict__ tasks, int ntasks, long long t,
                                            const AuxArgs& a, unsigned long long& lam) {
    const int n = a.geo.n;
    const size_t nn = (size_t)n * n;
    int task = 0, i = 0, j = 0, act = 0;
    if (t < (long long)ntasks * 4 * n) {
        task = (int)(t / (4 * n));
        const int e = (int)(t - (long long)task * 4 * n);
        bool ok = true;
        if (e < n) { i = 0; j = e; }
        else if (e < 2 * n) { i = n - 1; j = e - n; }
        else if (e < 3 * n) { i = e - 2 * n; j = 0; ok = i != 0 && i != n - 1; }
        else { i = e - 3 * n; j = n - 1; ok = i != 0 && i != n - 1; }
        const int touch = (i == 0 ? 1 : 0) | (i == n - 1 ? 2 : 0) | (j == 0 ? 4 : 0) | (j == n - 1 ? 8 : 0);
        act = ok ? touch & tasks[task].mask : 0;
    }
    if (act) {
        // the task's fields read where needed (a copy of the task indexed by side / half went through local memory)
        const RefluxTask& rt = tasks[task];
        const double coef = a.b * (*a.dt);
        double* U = a.Uw + (size_t)rt.slot * 4 * nn + (size_t)j * n + i;
        double u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = U[k * nn];
        const int l = rt.level;
        // fixed order: x-low, x-high, y-low, y-high (bitwise rank invariance, O12)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if (!(act & (1 << s))) continue;
            const int along = s < 2 ? j : i;
            const int opp = s ^ 1;
            const double ih = s < 2 ? a.geo.inv_dx[l] : a.geo.inv_dy[l];
            const double sigma = (s & 1) ? 1.0 : -1.0;
            const int f0 = 2 * along, fl = f0 / n, fp = f0 - fl * n;
            const int fleaf = rt.fine[s][fl];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double Fc = a.freg[(((size_t)rt.slot * 4 + s) * 4 + k) * n + along];
                const double* ff = a.freg + (((size_t)fleaf * 4 + opp) * 4 + k) * n + fp;
                double delta = Fc - 0.5 * (ff[0] + ff[1]);
                u[k] += coef * sigma * delta * ih;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) U[k * nn] = u[k];
        if (a.check || a.want_lambda)
            leaf_check(u[0], u[1], u[2], u[3], a.gamma, a.geo.inv_dx[l], a.geo.inv_dy[l], a.check, a.want_lambda,
                       a.lam0 ? l : 0, a.err, rt.slot, a.stage, j * n + i, lam);
    }
}

__global__ void reflux_kernel(const RefluxTask* __restrict__ tasks, int ntasks, const AuxArgs a) {
    // every lane stays to the end: Lambda is warp-reduced before one atomic per warp
    unsigned long long lam = 0ull;
    reflux_cell(tasks, ntasks, (long long)blockIdx.x * blockDim.x + threadIdx.x, a, lam);
    if (a.want_lambda) {
        lam = warp_max_u64(lam);
        if ((threadIdx.x & 31) == 0 && lam) atomicMax(a.lambda_bits, lam);
    }
}

// The work between two stage kernels in ONE cooperative launch (instead of reflux + one restriction launch per
// level + the next stage's ghost fill): O12 reflux of the coarse leaves; grid barrier; O9 restriction level by
// level, finest first, a grid barrier after each; then the O7/O8 ghost strips of the next stage's input (this
// stage's output).  The same per-cell arithmetic as the separate kernels, so the results are bitwise theirs.
constexpr int kPostThreads = 256;
__global__ void __launch_bounds__(kPostThreads) post_stage_kernel(const PostArgs p) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double post_cs[];   // ghost staging, one [4][g/2+2][n/2+2] slice per warp
    const int n = p.a.geo.n;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    unsigned long long lam = 0ull;
    const long long nre = (long long)p.nr * 4 * n;
    for (long long t = tid; t < nre; t += nthr) reflux_cell(p.rtasks, p.nr, t, p.a, lam);
    if (p.a.want_lambda) {
        lam = warp_max_u64(lam);
        if ((threadIdx.x & 31) == 0 && lam) atomicMax(p.a.lambda_bits, lam);
    }
    // the restriction of the finest level present shares the reflux phase: its children are leaves with nothing
    // finer, which the reflux never touches, and it writes covered patches, which the reflux never reads (disjoint
    // data: the result is bitwise the phase-by-phase one; one grid barrier and one dependent round trip fewer)
    int lf = p.levels - 1;
    while (lf >= 1 && p.nrl[lf] == 0) --lf;
    if (lf >= 1) {
        const long long w = (long long)p.nrl[lf] * n * n;
        for (long long t = tid; t < w; t += nthr) restrict_cell(p.rl[lf], t, p.a);
    }
    grid.sync();
    for (int l = lf - 1; l >= 1; --l) {
        if (p.nrl[l] == 0) continue;
        const long long w = (long long)p.nrl[l] * n * n;
        for (long long t = tid; t < w; t += nthr) restrict_cell(p.rl[l], t, p.a);
        grid.sync();
    }
    // ghost strips: one warp per strip (a strip is g x n cells)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* cs = post_cs + (size_t)wib * 4 * (p.g / 2 + 2) * (n / 2 + 2);
    const int nw = gridDim.x * (kPostThreads / 32);
    for (int task = blockIdx.x * (kPostThreads / 32) + wib; task < p.np; task += nw) {
        const ProxyTask pt = p.ptasks[task];   // (a private copy: the strip code re-reads the task's fields)
        ghost_strip(pt, p.g, p.a, cs, lane, 32, [] { __syncwarp(); });
        __syncwarp();   // cs is reused by the warp's next strip
    }
}

// ---------------------------------------------------------------- Lambda (O13) over leaves
// Lambda over all leaves (after a regrid / set_state): one warp per leaf, grid-stride over the leaves, the maximum
// reduced over the block before ONE atomic per block (a block per leaf with one atomic per warp queued ~8 same-address
// atomics per leaf -- 10^5 on the shock-bubble mesh)
__global__ void __launch_bounds__(256) lambda_kernel(const LeafDesc* __restrict__ leaves, int nleaves, const AuxArgs a) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int n = a.geo.n;
    const size_t nn = (size_t)n * n;
    unsigned long long lam = 0ull;
    for (int leaf = blockIdx.x * 8 + wib; leaf < nleaves; leaf += gridDim.x * 8) {
        const LeafDesc d = leaves[leaf];
        const double* U = a.U + (size_t)d.slot * 4 * nn;
        const double idx = a.geo.inv_dx[d.level], idy = a.geo.inv_dy[d.level];
#pragma unroll 4
        for (int e = lane; e < (int)nn; e += 32) {
            double s = wave_speed(U[e], U[nn + e], U[2 * nn + e], U[3 * nn + e], a.gamma, idx, idy);
            if (a.lam0) s = ldexp(s, -d.level);
            unsigned long long bits = (unsigned long long)__double_as_longlong(s);
            lam = bits > lam ? bits : lam;
        }
    }
    lam = warp_max_u64(lam);
    __shared__ unsigned long long sl[8];
    if (lane == 0) sl[wib] = lam;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) lam = sl[w] > lam ? sl[w] : lam;
        if (lam) atomicMax(a.lambda_bits, lam);
    }
}

__global__ void set2_kernel(double* p, double a, double b) {
    p[0] = a;
    p[1] = b;
}

__device__ __forceinline__ void dt_kernel_body(double* dt, unsigned long long* lambda_bits, int32_t* err, double dt_fixed,
                                               double cfl) {
    double lam = __longlong_as_double((long long)*lambda_bits);
    double d = dt_fixed > 0.0 ? dt_fixed : cfl / lam;
    if (!(d > 0.0) || !isfinite(d)) {
        if (atomicCAS(err, 0, 2) == 0) { err[1] = -1; err[2] = 0; err[3] = -1; }
    }
    *dt = d;
    dt[kMaxLevels] += d;   // simulated time (amr_stats.sim_time)
    *lambda_bits = 0ull;
}

__global__ void dt_kernel(double* dt, unsigned long long* lambda_bits, int32_t* err, double dt_fixed, double cfl) {
    dt_kernel_body(dt, lambda_bits, err, dt_fixed, cfl);
}

// subcycling (S1): dt_l = dt_0 / 2^l for every level, from dt[0]
__global__ void dt_levels_kernel(double* dt, int levels) {
    for (int l = 1; l < levels; ++l) dt[l] = ldexp(dt[0], -l);
}

// subcycling (S3): flux registers of C/F sides accumulated over a step, acc = (assign ? 0 : acc) + w F-hat
__global__ void accumulate_kernel(const AccTask* __restrict__ tasks, int ntasks, int n, const double* __restrict__ freg,
                                  double* __restrict__ acc, double w_coarse, double w_fine, int assign_coarse,
                                  int assign_fine) {
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)ntasks * 4 * n) return;
    const int task = (int)(t / (4 * n)), e = (int)(t - (long long)task * 4 * n);
    const AccTask at = tasks[task];
    const size_t o = (((size_t)at.slot * 4 + at.side) * 4) * n + e;   // [slot][side][k][n], e = k n + along
    const bool fine = at.kind == 2;
    const double w = fine ? w_fine : w_coarse;
    const double prev = (fine ? assign_fine : assign_coarse) ? 0.0 : acc[o];
    acc[o] = prev + w * freg[o];
}

// dt of a graph-replayed step: (dt_fixed, cfl) read from device memory written by set2_kernel before the replay
__global__ void dt_dev_kernel(double* dt, unsigned long long* lambda_bits, int32_t* err, const double* params) {
    dt_kernel_body(dt, lambda_bits, err, params[0], params[1]);
}

// ---------------------------------------------------------------- flags (O6)
// O6 indicator per leaf: one WARP per leaf (a block-per-leaf version waited on a block reduction and one
// descriptor -> data load chain per 256 cells); the per-cell arithmetic and the u64 maximum are unchanged.  Compiled
// for 4 blocks per SM (64 registers, 12 bytes of spill): the latency-bound loads gain more from the extra warps
// (shock-bubble flags phase 0.091 -> 0.079 ms per regrid) than the spill costs
__global__ void __launch_bounds__(256, 4) flags_kernel(const LeafDesc* __restrict__ leaves, int nleaves, const AuxArgs a,
                                                   double* maxeta, int32_t* amb) {
    const int leaf = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (leaf >= nleaves) return;
    const LeafDesc d = leaves[leaf];
    const int n = a.geo.n;
    const size_t nn = (size_t)n * n, PS = 4 * nn;
    const double* own = a.U + (size_t)d.slot * PS;
    const double dx = a.geo.dx[d.level], dy = a.geo.dy[d.level];
    const double hix = 0.5 * a.geo.inv_dx[d.level], hiy = 0.5 * a.geo.inv_dy[d.level];
    const double th = a.theta, tc = a.theta * a.coarsen_fraction;
    auto rho = [&](int i, int j) -> double {
        const double* b = own;
        if (i < 0) { int s = d.side[kW]; b = s >= 0 ? a.U + (size_t)s * PS : a.proxy + (size_t)(-1 - s) * PS; i += n; }
        else if (i >= n) { int s = d.side[kE]; b = s >= 0 ? a.U + (size_t)s * PS : a.proxy + (size_t)(-1 - s) * PS; i -= n; }
        else if (j < 0) { int s = d.side[kS]; b = s >= 0 ? a.U + (size_t)s * PS : a.proxy + (size_t)(-1 - s) * PS; j += n; }
        else if (j >= n) { int s = d.side[kN]; b = s >= 0 ? a.U + (size_t)s * PS : a.proxy + (size_t)(-1 - s) * PS; j -= n; }
        return b[(size_t)j * n + i];
    };
    unsigned long long m = 0ull;
    int am = 0;
#pragma unroll 4
    for (int e = lane; e < (int)nn; e += 32) {
        int i = e % n, j = e / n;
        // central differences and eta = dx |grad rho| / rho with the reciprocal spacings and the stage path's fast
        // reciprocal / square root (A41: within a few ulp of the divisions; A32's 1e-9 band covers the flags)
        double gx = (rho(i + 1, j) - rho(i - 1, j)) * hix;
        double gy = (rho(i, j + 1) - rho(i, j - 1)) * hiy;
        const double g2 = fma(gx, gx, gy * gy);
        double eta = dx * (g2 > 0.0 ? fast_sqrt(g2) : g2) * fast_rcp(rho(i, j));   // (fast_sqrt(0) is NaN)
        unsigned long long b = (unsigned long long)__double_as_longlong(eta);
        m = b > m ? b : m;
        if (fabs(eta - th) <= 1e-9 * th || fabs(eta - tc) <= 1e-9 * tc) am = 1;
    }
    m = warp_max_u64(m);
    am = __any_sync(0xffffffffu, am);
    if (lane == 0) {
        maxeta[leaf] = __longlong_as_double((long long)m);
        amb[leaf] = am;
    }
}

// ---------------------------------------------------------------- totals (O18), fixed-order per-leaf sums
__global__ void totals_kernel(const LeafDesc* __restrict__ leaves, const AuxArgs a, double* partial) {
    const LeafDesc d = leaves[blockIdx.x];
    const int n = a.geo.n;
    const size_t nn = (size_t)n * n;
    const double* U = a.U + (size_t)d.slot * 4 * nn;
    __shared__ double s[4][256];
    for (int k = 0; k < 4; ++k) {
        double acc = 0.0;
        for (int e = threadIdx.x; e < (int)nn; e += 256) acc += U[k * nn + e];
        s[k][threadIdx.x] = acc;
    }
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
            for (int k = 0; k < 4; ++k) s[k][threadIdx.x] += s[k][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double dv = a.geo.dx[d.level] * a.geo.dy[d.level];
        for (int k = 0; k < 4; ++k) partial[4 * (size_t)blockIdx.x + k] = s[k][0] * dv;
    }
}

// ---------------------------------------------------------------- packed <-> pool copies
__global__ void scatter_kernel(const double* __restrict__ packed, const int32_t* __restrict__ slots, long long total,
                               int ps, double* __restrict__ U, int to_pool) {
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        long long p = t / ps, e = t - p * ps;
        size_t pool = (size_t)slots[p] * ps + e;
        if (to_pool) U[pool] = packed[t];
        else const_cast<double*>(packed)[t] = U[pool];
    }
}

inline unsigned grid_for(long long work, int block) { return (unsigned)((work + block - 1) / block); }

}  // namespace

cudaError_t launch_stage(int scheme, const StageArgs& a, cudaStream_t s) {
    if (a.variant == 2)   // unfused: four kernels per stage
        return scheme == 0 ? launch_unfused<0>(a, s) : (scheme == 1 ? launch_unfused<1>(a, s) : launch_unfused<2>(a, s));
    if (a.variant == 3) {   // one launch of the per-tile fused kernel per leaf patch
        StageArgs b = a;
        b.variant = 1;
        b.nleaves = 1;
        for (int l = 0; l < a.nleaves; ++l) {
            b.leaves = a.leaves + l;
            cudaError_t e = launch_stage(scheme, b, s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    if (scheme == 0) return launch_stage_s<0>(a, s);
    if (scheme == 1) return launch_stage_s<1>(a, s);
    return launch_stage_s<2>(a, s);
}

size_t unfused_scratch_doubles(int n, int nleaves) {
    const size_t Wd = (size_t)n + 2 * kUnfG;
    return (size_t)nleaves * (4 * Wd * Wd + 2 * 4 * (size_t)n * (n + 3));
}

int stage_launches_per_stage(int variant, int nleaves) {
    return variant == 2 ? 4 : (variant == 3 ? nleaves : 1);
}

size_t stage_smem_bytes(int scheme, int n) {
    int T = n > 32 ? 32 : n;
    if (scheme == 0) return T == 8 ? stage_smem<0, 8>() : (T == 16 ? stage_smem<0, 16>() : stage_smem<0, 32>());
    return T == 8 ? stage_smem<1, 8>() : (T == 16 ? stage_smem<1, 16>() : stage_smem<1, 32>());
}

cudaError_t launch_ghost(const ProxyTask* tasks, int ntasks, int g, const AuxArgs& a, cudaStream_t s) {
    if (ntasks <= 0) return cudaSuccess;
    if (kGhostTile) {   // one CTA per strip, coarse values staged in shared memory
        const size_t smem = sizeof(double) * 4 * (g / 2 + 2) * (a.geo.n / 2 + 2);
        ghost_tile_kernel<<<ntasks, kGhostThreads, smem, s>>>(tasks, g, a);
        return cudaGetLastError();
    }
    long long work = (long long)ntasks * g * a.geo.n;
    ghost_kernel<<<grid_for(work, 256), 256, 0, s>>>(tasks, ntasks, g, a);
    return cudaGetLastError();
}

cudaError_t launch_reflux(const RefluxTask* tasks, int ntasks, const AuxArgs& a, cudaStream_t s) {
    if (ntasks <= 0) return cudaSuccess;
    long long work = (long long)ntasks * 4 * a.geo.n;
    reflux_kernel<<<grid_for(work, 128), 128, 0, s>>>(tasks, ntasks, a);
    return cudaGetLastError();
}

#ifdef AMR_HAVE_NCCL_H
__global__ void window_peer_ptrs_kernel(ncclWindow_t w, int world, void** out) {
    const int q = threadIdx.x;
    if (q < world) out[q] = ncclGetPeerPointer(w, 0, q);
}
#endif

#ifdef AMR_HAVE_NCCL_H
// peer_map 1 stage fence (NEXT #3: "synchronise stages with ncclLsaBarrierSession"): one CTA opens a
// session on barrier 0 of the device communicator's LSA team and syncs -- arrive stores epoch + 1 into every peer's
// inbox with release semantics (system scope), wait spins on this rank's inboxes with acquire -- so work queued
// after this kernel on the stream runs after every rank's work queued before its own fence kernel, with the peers'
// pool writes visible to this rank's loads over NVLink.  No host round trip and no NCCL collective kernel.
__global__ void __launch_bounds__(32) lsa_fence_kernel(const ncclDevComm dc) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}
#endif

cudaError_t launch_lsa_fence(const void* devcomm, cudaStream_t s) {
#ifdef AMR_HAVE_NCCL_H
    if (!devcomm) return cudaErrorInvalidValue;
    lsa_fence_kernel<<<1, 32, 0, s>>>(*reinterpret_cast<const ncclDevComm*>(devcomm));
    return cudaGetLastError();
#else
    (void)devcomm; (void)s;
    return cudaErrorNotSupported;
#endif
}

cudaError_t launch_window_peer_ptrs(const void* win, int world, void** d_out, cudaStream_t s) {
#ifdef AMR_HAVE_NCCL_H
    if (!win || world < 1 || world > 64) return cudaErrorInvalidValue;
    window_peer_ptrs_kernel<<<1, 64, 0, s>>>(reinterpret_cast<ncclWindow_t>(const_cast<void*>(win)), world, d_out);
    return cudaGetLastError();
#else
    (void)win; (void)world; (void)d_out; (void)s;
    return cudaErrorNotSupported;
#endif
}

cudaError_t launch_post_stage(const PostArgs& p, cudaStream_t s) {
    const int n = p.a.geo.n;
    const size_t smem = sizeof(double) * (kPostThreads / 32) * 4 * (p.g / 2 + 2) * (n / 2 + 2);
    static int max_blocks = 0;
    static size_t for_smem = 0;
    if (!max_blocks || for_smem != smem) {
        int occ = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, post_stage_kernel, kPostThreads, smem);
        if (e != cudaSuccess) return e;
        // at most 4 blocks per SM (A/B with AMR_POST_BPS: 2 / 4 / 8 within noise on configs[2], 4 = the separate
        // launches' time on configs[3]): the grid barriers cost more with more blocks, and the phases are short
        static const int bps = [] { const char* e = getenv("AMR_POST_BPS"); return e ? atoi(e) : 4; }();   // A/B
        max_blocks = std::max(1, std::min(occ, bps)) * sm_count();
        for_smem = smem;
    }
    long long need = ((long long)p.nr * 4 * n + kPostThreads - 1) / kPostThreads;
    for (int l = 1; l < p.levels; ++l)
        need = std::max(need, ((long long)p.nrl[l] * n * n + kPostThreads - 1) / kPostThreads);
    need = std::max(need, ((long long)p.np + kPostThreads / 32 - 1) / (kPostThreads / 32));
    const int grid = (int)std::max(1LL, std::min(need, (long long)max_blocks));
    void* args[] = {const_cast<PostArgs*>(&p)};
    return cudaLaunchCooperativeKernel((const void*)post_stage_kernel, dim3(grid), dim3(kPostThreads), args, smem, s);
}

cudaError_t launch_restrict(const RestrictTask* tasks, int ntasks, const AuxArgs& a, cudaStream_t s) {
    if (ntasks <= 0) return cudaSuccess;
    long long work = (long long)ntasks * a.geo.n * a.geo.n;
    restrict_kernel<<<grid_for(work, 256), 256, 0, s>>>(tasks, ntasks, a);
    return cudaGetLastError();
}

cudaError_t launch_prolong(const ProlongTask* tasks, int ntasks, const AuxArgs& a, cudaStream_t s) {
    if (ntasks <= 0) return cudaSuccess;
    long long work = (long long)ntasks * a.geo.n * a.geo.n;
    prolong_kernel<<<grid_for(work, 256), 256, 0, s>>>(tasks, ntasks, a);
    return cudaGetLastError();
}

cudaError_t launch_lambda(const LeafDesc* leaves, int nleaves, const AuxArgs& a, cudaStream_t s) {
    if (nleaves <= 0) return cudaSuccess;
    const int blocks = std::min((nleaves + 7) / 8, 4 * sm_count());
    lambda_kernel<<<blocks, 256, 0, s>>>(leaves, nleaves, a);
    return cudaGetLastError();
}

cudaError_t launch_dt_dev(double* dt, unsigned long long* lambda_bits, int32_t* err, const double* params,
                          cudaStream_t s) {
    dt_dev_kernel<<<1, 1, 0, s>>>(dt, lambda_bits, err, params);
    return cudaGetLastError();
}

cudaError_t launch_dt_levels(double* dt, int levels, cudaStream_t s) {
    dt_levels_kernel<<<1, 1, 0, s>>>(dt, levels);
    return cudaGetLastError();
}

cudaError_t launch_accumulate(const AccTask* tasks, int ntasks, int n, const double* freg, double* acc, double w_coarse,
                              double w_fine, int assign_coarse, int assign_fine, cudaStream_t s) {
    if (ntasks <= 0) return cudaSuccess;
    const long long work = (long long)ntasks * 4 * n;
    accumulate_kernel<<<grid_for(work, 256), 256, 0, s>>>(tasks, ntasks, n, freg, acc, w_coarse, w_fine, assign_coarse,
                                                          assign_fine);
    return cudaGetLastError();
}

cudaError_t launch_set2(double* p, double a, double b, cudaStream_t s) {
    set2_kernel<<<1, 1, 0, s>>>(p, a, b);
    return cudaGetLastError();
}

cudaError_t launch_dt(double* dt, unsigned long long* lambda_bits, int32_t* err, double dt_fixed, double cfl,
                      cudaStream_t s) {
    dt_kernel<<<1, 1, 0, s>>>(dt, lambda_bits, err, dt_fixed, cfl);
    return cudaGetLastError();
}

cudaError_t launch_flags(const LeafDesc* leaves, int nleaves, const AuxArgs& a, double* maxeta, int32_t* amb,
                         cudaStream_t s) {
    if (nleaves <= 0) return cudaSuccess;
    flags_kernel<<<(unsigned)((nleaves + 7) / 8), 256, 0, s>>>(leaves, nleaves, a, maxeta, amb);
    return cudaGetLastError();
}

// Flag compaction: one thread per leaf and per sibling group (a parent whose 4 children are leaves);
// the refine bit of a leaf, eta > theta below the finest level, and the coarsen bit of a sibling group,
// max child eta < theta * coarsen_fraction (Alg. 2 / A15), are appended as (slot, bits) to a compact list with one
// atomic per warp, so the host reads only the requests.  Same comparisons and NaN handling as the full host path.
__global__ void flags_compact_kernel(const LeafDesc* __restrict__ leaves, int nleaves, const int32_t* __restrict__ sib,
                                     int nsib, const double* __restrict__ maxeta, double th, double tc, int top,
                                     int32_t* list, int32_t* count) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    int slot = -1, bits = 0;
    if (k < nleaves) {
        const double e = maxeta[k];
        if (leaves[k].level < top && e > th) { slot = leaves[k].slot; bits = 1; }
    } else if (k - nleaves < nsib) {
        const int32_t* g = sib + 5 * (k - nleaves);
        double m = 0.0;
        for (int q = 0; q < 4; ++q) {
            const double e = maxeta[g[1 + q]];
            if (!(e <= m)) m = e;
        }
        if (m < tc) { slot = g[0]; bits = 2; }
    }
    const unsigned want = __ballot_sync(0xffffffffu, bits != 0);
    if (!want) return;
    const int lane = threadIdx.x & 31, leader = __ffs(want) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(want));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (bits) {
        const int at = base + __popc(want & ((1u << lane) - 1u));
        list[2 * at] = slot;
        list[2 * at + 1] = bits;
    }
}

cudaError_t launch_flags_compact(const LeafDesc* leaves, int nleaves, const int32_t* sib, int nsib,
                                 const double* maxeta, double th, double tc, int top, int32_t* list, int32_t* count,
                                 cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int32_t), s);
    if (e != cudaSuccess || nleaves + nsib <= 0) return e;
    flags_compact_kernel<<<grid_for((long long)nleaves + nsib, 256), 256, 0, s>>>(leaves, nleaves, sib, nsib, maxeta,
                                                                                   th, tc, top, list, count);
    return cudaGetLastError();
}

// Peer pull (NEXT #3, halo_mode 1): one CTA per received slot loads the slot's `per` doubles straight from the
// owning rank's pool, mapped into this process (NVLink peer memory; another virtual rank's buffer on one GPU), into
// the same slot of the local buffer -- no pack / unpack kernels, no staging buffers, no transport call.  16-byte
// vector loads (every slot region is a multiple of 16 bytes and 16-byte aligned).
__global__ void peer_pull_kernel(const int32_t* __restrict__ slots, const int32_t* __restrict__ peers,
                                 const double* const* __restrict__ bases, size_t off, double* __restrict__ dst, int per) {
    const size_t slot = (size_t)slots[blockIdx.x];
    const double2* src = reinterpret_cast<const double2*>(bases[peers[blockIdx.x]] + off + slot * per);
    double2* out = reinterpret_cast<double2*>(dst + slot * per);
    const int nv = per / 2;
    for (int e = threadIdx.x; e < nv; e += blockDim.x) out[e] = src[e];
}

cudaError_t launch_peer_pull(const int32_t* slots, const int32_t* peers, int n, const double* const* bases,
                             size_t off, double* dst, int per, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (per % 2) return cudaErrorInvalidValue;
    peer_pull_kernel<<<n, 256, 0, s>>>(slots, peers, bases, off, dst, per);
    return cudaGetLastError();
}

// Band items of the halo exchange (comm.h): item = slot * 32 + code; code < 16: rows 4 code .. 4 code + 3 (a row
// band), 16: columns 0..3, 17: columns n-4..n-1; 16 n doubles each (4 variables x 4 n cells), in [var][band cell]
// order.  The pool offset of element e of an item:
__device__ __forceinline__ size_t band_offset(int32_t item, int e, int n) {
    const size_t slot = (size_t)(item >> 5);
    const int code = item & 31, per_var = 4 * n;
    const int var = e / per_var, r = e - var * per_var;
    int i, j;
    if (code < 16) { j = 4 * code + r / n; i = r % n; }
    else { j = r >> 2; i = (code == 16 ? 0 : n - 4) + (r & 3); }
    return ((slot * 4 + var) * n + j) * (size_t)n + i;
}
__global__ void band_copy_kernel(const double* __restrict__ packed, const int32_t* __restrict__ items, long long total,
                                 int n, double* __restrict__ U, int to_pool) {
    const int per = 16 * n;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long k = t / per;
        const size_t o = band_offset(items[k], (int)(t - k * per), n);
        if (to_pool) U[o] = packed[t];
        else const_cast<double*>(packed)[t] = U[o];
    }
}
__global__ void band_pull_kernel(const int32_t* __restrict__ items, const int32_t* __restrict__ peers,
                                 const double* const* __restrict__ bases, size_t off, double* __restrict__ dst, int n) {
    const int32_t item = items[blockIdx.x];
    const double* src = bases[peers[blockIdx.x]] + off;
    for (int e = threadIdx.x; e < 16 * n; e += blockDim.x) {
        const size_t o = band_offset(item, e, n);
        dst[o] = src[o];   // the same band of the same slot and RK buffer in the owner's pool
    }
}

cudaError_t launch_band_scatter(const double* packed, const int32_t* items, int nitem, double* U, int n, cudaStream_t s) {
    if (nitem <= 0) return cudaSuccess;
    const long long total = (long long)nitem * 16 * n;
    unsigned blocks = grid_for(total, 256);
    if (blocks > 148u * 64u) blocks = 148u * 64u;
    band_copy_kernel<<<blocks, 256, 0, s>>>(packed, items, total, n, U, 1);
    return cudaGetLastError();
}
cudaError_t launch_band_gather(const double* U, const int32_t* items, int nitem, double* packed, int n, cudaStream_t s) {
    if (nitem <= 0) return cudaSuccess;
    const long long total = (long long)nitem * 16 * n;
    unsigned blocks = grid_for(total, 256);
    if (blocks > 148u * 64u) blocks = 148u * 64u;
    band_copy_kernel<<<blocks, 256, 0, s>>>(packed, items, total, n, const_cast<double*>(U), 0);
    return cudaGetLastError();
}
cudaError_t launch_band_pull(const int32_t* items, const int32_t* peers, int nitem, const double* const* bases,
                             size_t off, double* dst, int n, cudaStream_t s) {
    if (nitem <= 0) return cudaSuccess;
    band_pull_kernel<<<nitem, 128, 0, s>>>(items, peers, bases, off, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_scatter(const double* packed, const int32_t* slots, int npatch, double* U, int per, cudaStream_t s) {
    if (npatch <= 0) return cudaSuccess;
    long long total = (long long)npatch * per;
    unsigned blocks = grid_for(total, 256);
    if (blocks > 148u * 64u) blocks = 148u * 64u;
    scatter_kernel<<<blocks, 256, 0, s>>>(packed, slots, total, per, U, 1);
    return cudaGetLastError();
}

cudaError_t launch_gather(const double* U, const int32_t* slots, int npatch, double* packed, int per, cudaStream_t s) {
    if (npatch <= 0) return cudaSuccess;
    long long total = (long long)npatch * per;
    unsigned blocks = grid_for(total, 256);
    if (blocks > 148u * 64u) blocks = 148u * 64u;
    scatter_kernel<<<blocks, 256, 0, s>>>(packed, slots, total, per, const_cast<double*>(U), 0);
    return cudaGetLastError();
}

cudaError_t launch_totals(const LeafDesc* leaves, int nleaves, const AuxArgs& a, double* partial, cudaStream_t s) {
    if (nleaves <= 0) return cudaSuccess;
    totals_kernel<<<nleaves, 256, 0, s>>>(leaves, a, partial);
    return cudaGetLastError();
}

}  // namespace amr
