/*
 * oracle.cpp -- plain, slow, obviously-correct CPU ORACLE of the AMR
 * compressible-Euler hot path of arXiv 2508.05020.
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  It shares no
 * code with the CUDA product path and must never be reached from it.
 *
 * Every function names the passage it follows:
 *   P:Lnn  = /root/reference/PAPER.md line nn (section / equation given too)
 *   O1-O18 = SURVEY.md s8(c) oracle definitions; A1-A42 = readings
 * No blocking, fusion or reordering: each step is written in the order the
 * definition states it, on std::map-keyed patches, in fp64.
 * Build: g++ -O2 -ffp-contract=off -fPIC -shared (no fast-math).
 */
#include "oracle.h"

#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

enum { BC_PERIODIC = 0, BC_TRANSMISSIVE = 1, BC_REFLECTIVE = 2 };
const int NV = 4;   /* (rho, rho u, rho v, rho e): Eq. 10 vector U */

/* O1: patch key (level, P, Q); canonical order (level, Q, P) (O3). */
struct Key {
    int l, P, Q;
};
bool operator<(const Key& a, const Key& b) {
    if (a.l != b.l) return a.l < b.l;
    if (a.Q != b.Q) return a.Q < b.Q;
    return a.P < b.P;
}

/* O1: Moore directions in Fig. 2 nbr order: N, E, S, W, NE, SE, SW, NW. */
const int MOORE[8][2] = {{0, 1}, {1, 0}, {0, -1}, {-1, 0}, {1, 1}, {1, -1}, {-1, -1}, {-1, 1}};

void fail(const std::string& m) { throw std::runtime_error(m); }

/* Deterministic parallelism over patches ("OpenMP over patches only"): f(e) for e in [0, n)
 * writes only data owned by item e, so the result does not depend on the thread count or schedule.  An
 * exception inside an item is re-thrown after the loop (the one of the lowest item, as a serial loop would). */
template <class F>
void par_for(long n, F f) {
    long bad = n;
    int kind = 0;
    std::string msg;
#pragma omp parallel for schedule(dynamic, 1)
    for (long e = 0; e < n; ++e) {
        try {
            f(e);
        } catch (const std::domain_error& x) {
#pragma omp critical(orc_err)
            if (e < bad) { bad = e; kind = 1; msg = x.what(); }
        } catch (const std::exception& x) {
#pragma omp critical(orc_err)
            if (e < bad) { bad = e; kind = 2; msg = x.what(); }
        }
    }
    if (kind == 1) throw std::domain_error(msg);
    if (kind == 2) throw std::runtime_error(msg);
}

typedef std::map<Key, std::vector<double>> Field;   /* per patch U[4][n][n] */

struct Oracle {
    orc_config c;
    std::map<Key, char> tree;   /* active patches -> has_children (Fig. 2 child[]) */
    Field U;                    /* U^n */
    std::string err;

    int n() const { return c.n; }
    /* O1: level-l patch and cell extents */
    int NP(int ax, int l) const { return (c.base[ax] / c.n) << l; }
    int NC(int ax, int l) const { return c.base[ax] << l; }
    /* O1: dx_l = (hi - lo) / (N * 2^l) */
    double h(int ax, int l) const {
        return (c.hi[ax] - c.lo[ax]) / ((double)c.base[ax] * (double)(1 << l));
    }
    bool periodic(int ax) const { return c.bc[2 * ax] == BC_PERIODIC; }
    bool active(const Key& k) const { return tree.count(k) != 0; }
    bool has_children(const Key& k) const {
        auto it = tree.find(k);
        return it != tree.end() && it->second;
    }
    int ghost_width() const { return 4; }   /* A8: enough for every scheme */
};

int posmod(int a, int b) { int r = a % b; return r < 0 ? r + b : r; }

/* O1: wrap a patch position at level l; false when outside a non-periodic side. */
bool wrap_patch(const Oracle& o, int l, int& P, int& Q) {
    int NPx = o.NP(0, l), NPy = o.NP(1, l);
    if (P < 0 || P >= NPx) {
        if (!o.periodic(0)) return false;
        P = posmod(P, NPx);
    }
    if (Q < 0 || Q >= NPy) {
        if (!o.periodic(1)) return false;
        Q = posmod(Q, NPy);
    }
    return true;
}

/* ------------------------------------------------------------------ gas */
/* O2: Eq. 4-7.  u = m/rho, v = w/rho, p = (g-1)(E - (m u + w v)/2) */
void cons2prim(double g, const double* U, double* W) {
    double r = U[0];
    double u = U[1] / r;
    double v = U[2] / r;
    double p = (g - 1.0) * (U[3] - 0.5 * (U[1] * u + U[2] * v));
    W[0] = r; W[1] = u; W[2] = v; W[3] = p;
}
/* O2 inverse: E = p/(g-1) + rho (u^2+v^2)/2 */
void prim2cons(double g, const double* W, double* U) {
    U[0] = W[0];
    U[1] = W[0] * W[1];
    U[2] = W[0] * W[2];
    U[3] = W[3] / (g - 1.0) + 0.5 * W[0] * (W[1] * W[1] + W[2] * W[2]);
}
/* Eq. 1-3 / Eq. 10 flux along x: (m, m u + p, w u, (E + p) u); (E+p) = rho h (Eq. 5) */
void euler_flux_x(double g, const double* U, double* F) {
    double W[4];
    cons2prim(g, U, W);
    F[0] = U[1];
    F[1] = U[1] * W[1] + W[3];
    F[2] = U[2] * W[1];
    F[3] = (U[3] + W[3]) * W[1];
}

/* ------------------------------------------------------------------ schemes */
/* O8 / A38: monotonised-central limiter */
double mc(double a, double b) {
    if (a * b <= 0.0) return 0.0;
    double m = std::fabs(a + b) / 2.0;
    if (2.0 * std::fabs(a) < m) m = 2.0 * std::fabs(a);
    if (2.0 * std::fabs(b) < m) m = 2.0 * std::fabs(b);
    return a > 0.0 ? m : -m;
}

/* O10 / A2: WENO5-JS point-value interpolation to x_{i+1/2} from v0..v4 = cells i-2..i+2
 * ("convex superposition ... reach the 5th-order linear interpolation") */
double weno5(const double* v, double eps) {
    double q0 = (3.0 * v[0] - 10.0 * v[1] + 15.0 * v[2]) / 8.0;
    double q1 = (-v[1] + 6.0 * v[2] + 3.0 * v[3]) / 8.0;
    double q2 = (3.0 * v[2] + 6.0 * v[3] - v[4]) / 8.0;
    double t;
    double b0, b1, b2;
    t = v[0] - 2.0 * v[1] + v[2];
    b0 = 13.0 / 12.0 * t * t;
    t = v[0] - 4.0 * v[1] + 3.0 * v[2];
    b0 = b0 + 0.25 * t * t;
    t = v[1] - 2.0 * v[2] + v[3];
    b1 = 13.0 / 12.0 * t * t;
    t = v[1] - v[3];
    b1 = b1 + 0.25 * t * t;
    t = v[2] - 2.0 * v[3] + v[4];
    b2 = 13.0 / 12.0 * t * t;
    t = 3.0 * v[2] - 4.0 * v[3] + v[4];
    b2 = b2 + 0.25 * t * t;
    double a0 = (1.0 / 16.0) / ((eps + b0) * (eps + b0));
    double a1 = (10.0 / 16.0) / ((eps + b1) * (eps + b1));
    double a2 = (5.0 / 16.0) / ((eps + b2) * (eps + b2));
    return (a0 * q0 + a1 * q1 + a2 * q2) / (a0 + a1 + a2);
}

/* O10 step 1 / A4: left (rows) and right (columns) eigenvectors of the x-flux Jacobian
 * at the arithmetic-mean primitive state of the two cells (Lm row-major [k][m],
 * Rm row-major [m][k] so that column k is r_k). */
void eigen_x(double g, const double* WL, const double* WR, double* Lm, double* Rm) {
    double r = 0.5 * (WL[0] + WR[0]);
    double u = 0.5 * (WL[1] + WR[1]);
    double v = 0.5 * (WL[2] + WR[2]);
    double p = 0.5 * (WL[3] + WR[3]);
    double cs = std::sqrt(g * p / r);
    double q = 0.5 * (u * u + v * v);
    double H = cs * cs / (g - 1.0) + q;
    double b1 = (g - 1.0) / (cs * cs);
    double b2 = b1 * q;
    double L[4][4] = {
        {0.5 * (b2 + u / cs), 0.5 * (-b1 * u - 1.0 / cs), 0.5 * (-b1 * v), 0.5 * b1},
        {1.0 - b2, b1 * u, b1 * v, -b1},
        {-v, 0.0, 1.0, 0.0},
        {0.5 * (b2 - u / cs), 0.5 * (-b1 * u + 1.0 / cs), 0.5 * (-b1 * v), 0.5 * b1}};
    double Rc[4][4] = {/* columns r_1..r_4 */
                       {1.0, u - cs, v, H - u * cs},
                       {1.0, u, v, q},
                       {0.0, 0.0, 1.0, v},
                       {1.0, u + cs, v, H + u * cs}};
    for (int k = 0; k < 4; ++k)
        for (int m = 0; m < 4; ++m) {
            Lm[4 * k + m] = L[k][m];
            Rm[4 * m + k] = Rc[k][m];
        }
}

/* Eq. 11-12: Rusanov flux along x */
void rusanov_x(double g, const double* UL, const double* UR, double* F) {
    double WL[4], WR[4], FL[4], FR[4];
    cons2prim(g, UL, WL);
    cons2prim(g, UR, WR);
    double cL = std::sqrt(g * WL[3] / WL[0]);
    double cR = std::sqrt(g * WR[3] / WR[0]);
    double sR = cR + std::fabs(WR[1]);
    double sL = cL + std::fabs(WL[1]);
    double S = sR > sL ? sR : sL;
    euler_flux_x(g, UL, FL);
    euler_flux_x(g, UR, FR);
    for (int k = 0; k < 4; ++k) F[k] = 0.5 * (FR[k] + FL[k]) - 0.5 * S * (UR[k] - UL[k]);
}

/* O10: face flux f_{i+1/2} along x from conserved cells i-2..i+3 (cells[6][4]). */
void face_flux_x(const orc_config& c, const double cells[6][4], double* F) {
    double g = c.gamma;
    if (c.scheme == 0) {
        /* Central4 (Eq. 8 read edge-from-node, A6/A7):
         * interpolate p, T = p/rho, u, v; rho_e = p_e/T_e; E_e = p_e/(g-1) + rho_e |u_e|^2/2 */
        double phi[4][4];   /* [cell i-1..i+2][p,T,u,v] */
        for (int s = 0; s < 4; ++s) {
            double W[4];
            cons2prim(g, cells[s + 1], W);
            phi[s][0] = W[3];
            phi[s][1] = W[3] / W[0];
            phi[s][2] = W[1];
            phi[s][3] = W[2];
        }
        double e[4];
        for (int k = 0; k < 4; ++k)
            e[k] = 9.0 / 16.0 * (phi[1][k] + phi[2][k]) - 1.0 / 16.0 * (phi[0][k] + phi[3][k]);
        double pe = e[0], Te = e[1], ue = e[2], ve = e[3];
        double re = pe / Te;
        double Ee = pe / (g - 1.0) + 0.5 * re * (ue * ue + ve * ve);
        F[0] = re * ue;
        F[1] = re * ue * ue + pe;
        F[2] = re * ue * ve;
        F[3] = (Ee + pe) * ue;
        return;
    }
    /* WENO5-JS + Rusanov (O10 steps 1-5) */
    double Lm[16], Rm[16];
    if (c.characteristic) {
        double WL[4], WR[4];
        cons2prim(g, cells[2], WL);
        cons2prim(g, cells[3], WR);
        eigen_x(g, WL, WR, Lm, Rm);
    } else {
        for (int a = 0; a < 16; ++a) Lm[a] = Rm[a] = (a % 5 == 0) ? 1.0 : 0.0;   /* A35 */
    }
    double w[6][4];
    for (int j = 0; j < 6; ++j)
        for (int k = 0; k < 4; ++k) {
            double s = 0.0;
            for (int m = 0; m < 4; ++m) s += Lm[4 * k + m] * cells[j][m];
            w[j][k] = s;
        }
    double wl[4], wr[4];
    for (int k = 0; k < 4; ++k) {
        double vl[5] = {w[0][k], w[1][k], w[2][k], w[3][k], w[4][k]};
        double vr[5] = {w[5][k], w[4][k], w[3][k], w[2][k], w[1][k]};
        wl[k] = weno5(vl, c.weno_eps);
        wr[k] = weno5(vr, c.weno_eps);
    }
    double UL[4], UR[4];
    for (int m = 0; m < 4; ++m) {
        double sl = 0.0, sr = 0.0;
        for (int k = 0; k < 4; ++k) {
            sl += Rm[4 * m + k] * wl[k];
            sr += Rm[4 * m + k] * wr[k];
        }
        UL[m] = sl;
        UR[m] = sr;
    }
    rusanov_x(g, UL, UR, F);
}

/* ------------------------------------------------------------------ composite data access */
/* value of component k at level-l cell (I,J) from the active patch containing it (in-domain, wrapped) */
double patch_value(const Oracle& o, const Field& S, int l, int I, int J, int k) {
    int n = o.n();
    Key key{l, I / n, J / n};
    auto it = S.find(key);
    if (it == S.end() || !o.active(key)) {
        char b[160];
        std::snprintf(b, sizeof b, "no active patch at level %d holds cell (%d,%d)", l, I, J);
        fail(b);
    }
    int i = I - key.P * n, j = J - key.Q * n;
    return it->second[(k * n + j) * n + i];
}

/* O7 applied at a coarse level for O8 slopes: out-of-domain positions use the BC rule
 * (transmissive clamp; reflective mirror with negated normal momentum). */
double coarse_value(const Oracle& o, const Field& S, int l, int I, int J, int k) {
    double sgn = 1.0;
    int NCx = o.NC(0, l), NCy = o.NC(1, l);
    if (I < 0 || I >= NCx) {
        if (o.periodic(0)) {
            I = posmod(I, NCx);
        } else {
            int bc = I < 0 ? o.c.bc[0] : o.c.bc[1];
            if (bc == BC_TRANSMISSIVE) I = I < 0 ? 0 : NCx - 1;
            else { I = I < 0 ? -1 - I : 2 * NCx - 1 - I; if (k == 1) sgn = -1.0; }
        }
    }
    if (J < 0 || J >= NCy) {
        if (o.periodic(1)) {
            J = posmod(J, NCy);
        } else {
            int bc = J < 0 ? o.c.bc[2] : o.c.bc[3];
            if (bc == BC_TRANSMISSIVE) J = J < 0 ? 0 : NCy - 1;
            else { J = J < 0 ? -1 - J : 2 * NCy - 1 - J; if (k == 2) sgn = -1.0; }
        }
    }
    return sgn * patch_value(o, S, l, I, J, k);
}

/* O8: MC-limited linear prolongation of fine cell (I,J) at level l (in-domain, wrapped) */
double prolong_value(const Oracle& o, const Field& S, int l, int I, int J, int k) {
    int Ic = I / 2, Jc = J / 2;
    int a = I % 2, b = J % 2;
    double V = coarse_value(o, S, l - 1, Ic, Jc, k);
    double sx = mc(V - coarse_value(o, S, l - 1, Ic - 1, Jc, k),
                   coarse_value(o, S, l - 1, Ic + 1, Jc, k) - V);
    double sy = mc(V - coarse_value(o, S, l - 1, Ic, Jc - 1, k),
                   coarse_value(o, S, l - 1, Ic, Jc + 1, k) - V);
    double t = V + ((2 * a - 1) * 0.25) * sx;
    return t + ((2 * b - 1) * 0.25) * sy;
}

/* O7: ghost cell (I,J) (global level-l index, unwrapped) of a side strip of leaf p */
double ghost_value(const Oracle& o, const Field& S, const Key& p, int I, int J, int k) {
    int l = p.l;
    int NCx = o.NC(0, l), NCy = o.NC(1, l);
    bool outx = (I < 0 || I >= NCx) && !o.periodic(0);
    bool outy = (J < 0 || J >= NCy) && !o.periodic(1);
    if (outx || outy) {
        /* physical boundary: the source is an interior cell of p itself (A25) */
        double sgn = 1.0;
        if (outx) {
            int bc = I < 0 ? o.c.bc[0] : o.c.bc[1];
            if (bc == BC_TRANSMISSIVE) I = I < 0 ? 0 : NCx - 1;
            else { I = I < 0 ? -1 - I : 2 * NCx - 1 - I; if (k == 1) sgn = -sgn; }
        }
        if (outy) {
            int bc = J < 0 ? o.c.bc[2] : o.c.bc[3];
            if (bc == BC_TRANSMISSIVE) J = J < 0 ? 0 : NCy - 1;
            else { J = J < 0 ? -1 - J : 2 * NCy - 1 - J; if (k == 2) sgn = -sgn; }
        }
        return sgn * patch_value(o, S, l, I, J, k);
    }
    I = posmod(I, NCx);
    J = posmod(J, NCy);
    int n = o.n();
    if (o.active(Key{l, I / n, J / n})) return patch_value(o, S, l, I, J, k);
    return prolong_value(o, S, l, I, J, k);
}

/* a tile of leaf p: interior plus the four g-deep side strips; corners are NaN (A26) */
std::vector<double> build_tile(const Oracle& o, const Field& S, const Key& p, int g) {
    int n = o.n(), w = n + 2 * g;
    std::vector<double> t((size_t)NV * w * w, std::nan(""));
    const std::vector<double>& u = S.at(p);
    for (int k = 0; k < NV; ++k)
        for (int j = -g; j < n + g; ++j)
            for (int i = -g; i < n + g; ++i) {
                bool inx = i >= 0 && i < n, iny = j >= 0 && j < n;
                double val;
                if (inx && iny) val = u[(k * n + j) * n + i];
                else if (inx || iny) val = ghost_value(o, S, p, p.P * n + i, p.Q * n + j, k);
                else continue;
                t[((size_t)k * w + (j + g)) * w + (i + g)] = val;
            }
    return t;
}

/* ------------------------------------------------------------------ spatial operator */
/* O10: L(U) on one leaf; also returns Fhat on x-faces [k][j][0..n] and y-faces [k][0..n][i]
 * (face m = the face left of / below cell m). */
void spatial_operator(const Oracle& o, const std::vector<double>& tile, int l, std::vector<double>& L,
                      std::vector<double>& FhX, std::vector<double>& FhY) {
    int n = o.n(), g = o.ghost_width(), w = n + 2 * g;
    double dx = o.h(0, l), dy = o.h(1, l);
    auto T = [&](int k, int j, int i) { return tile[((size_t)k * w + (j + g)) * w + (i + g)]; };
    FhX.assign((size_t)NV * n * (n + 1), 0.0);
    FhY.assign((size_t)NV * (n + 1) * n, 0.0);
    /* x-faces: f at faces m = -1..n+1 (left of cell m), rows j */
    for (int j = 0; j < n; ++j) {
        std::vector<double> f((size_t)(n + 3) * NV);
        for (int m = -1; m <= n + 1; ++m) {
            double cells[6][4];
            for (int s = 0; s < 6; ++s)
                for (int k = 0; k < NV; ++k) cells[s][k] = T(k, j, m - 3 + s);
            face_flux_x(o.c, cells, &f[(size_t)(m + 1) * NV]);
        }
        for (int m = 0; m <= n; ++m)
            for (int k = 0; k < NV; ++k) {
                double fm = f[(size_t)(m + 1) * NV + k];
                double fh = fm;
                if (o.c.div_order == 4) {
                    /* Eq. 9 in flux form (O10): 13/12 f_m - 1/24 (f_{m-1} + f_{m+1}) */
                    fh = 13.0 / 12.0 * fm - 1.0 / 24.0 * (f[(size_t)m * NV + k] + f[(size_t)(m + 2) * NV + k]);
                }
                FhX[((size_t)k * n + j) * (n + 1) + m] = fh;
            }
    }
    /* y-faces: rotate (rho, m, w, E) -> (rho, w, m, E), x-flux, rotate back (O10 "swap") */
    for (int i = 0; i < n; ++i) {
        std::vector<double> f((size_t)(n + 3) * NV);
        for (int m = -1; m <= n + 1; ++m) {
            double cells[6][4];
            for (int s = 0; s < 6; ++s) {
                int j = m - 3 + s;
                cells[s][0] = T(0, j, i);
                cells[s][1] = T(2, j, i);
                cells[s][2] = T(1, j, i);
                cells[s][3] = T(3, j, i);
            }
            double fr[4];
            face_flux_x(o.c, cells, fr);
            double* d = &f[(size_t)(m + 1) * NV];
            d[0] = fr[0]; d[1] = fr[2]; d[2] = fr[1]; d[3] = fr[3];
        }
        for (int m = 0; m <= n; ++m)
            for (int k = 0; k < NV; ++k) {
                double fm = f[(size_t)(m + 1) * NV + k];
                double fh = fm;
                if (o.c.div_order == 4)
                    fh = 13.0 / 12.0 * fm - 1.0 / 24.0 * (f[(size_t)m * NV + k] + f[(size_t)(m + 2) * NV + k]);
                FhY[((size_t)k * (n + 1) + m) * n + i] = fh;
            }
    }
    L.assign((size_t)NV * n * n, 0.0);
    for (int k = 0; k < NV; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                double lx = -(FhX[((size_t)k * n + j) * (n + 1) + i + 1] - FhX[((size_t)k * n + j) * (n + 1) + i]) / dx;
                double ly = (FhY[((size_t)k * (n + 1) + j + 1) * n + i] - FhY[((size_t)k * (n + 1) + j) * n + i]) / dy;
                L[((size_t)k * n + j) * n + i] = lx - ly;
            }
}

/* ------------------------------------------------------------------ tree (O3-O5) */
void refine(Oracle& o, const Key& p) {
    /* Alg. 1 RefinePatch, O4 */
    if (o.has_children(p)) return;
    if (!o.active(p)) fail("refine of inactive patch");
    for (int d = 0; d < 8; ++d) {
        int P = p.P + MOORE[d][0], Q = p.Q + MOORE[d][1];
        if (!wrap_patch(o, p.l, P, Q)) continue;
        if (!o.active(Key{p.l, P, Q})) {
            Key r{p.l - 1, P / 2, Q / 2};
            if (p.l == 0 || !o.active(r)) fail("R2 violated before refinement");
            refine(o, r);
        }
    }
    for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a) o.tree[Key{p.l + 1, 2 * p.P + a, 2 * p.Q + b}] = 0;
    o.tree[p] = 1;
}

bool children_all_leaves(const Oracle& o, const Key& p) {
    if (!o.has_children(p)) return false;
    for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a)
            if (o.has_children(Key{p.l + 1, 2 * p.P + a, 2 * p.Q + b})) return false;
    return true;
}

/* O5 / A16: IsCoarseningAllowed -- R2-exact prose rule or Alg. 2 literal */
bool coarsen_allowed(const Oracle& o, const Key& p) {
    if (!children_all_leaves(o, p)) return false;
    if (o.c.coarsen_rule == 1) {
        if (p.l == 0) return false;
        for (int d = 0; d < 8; ++d) {
            int P = p.P + MOORE[d][0], Q = p.Q + MOORE[d][1];
            if (!wrap_patch(o, p.l, P, Q)) continue;
            if (o.has_children(Key{p.l, P, Q})) return false;
        }
        return true;
    }
    for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a) {
            Key ch{p.l + 1, 2 * p.P + a, 2 * p.Q + b};
            for (int d = 0; d < 8; ++d) {
                int P = ch.P + MOORE[d][0], Q = ch.Q + MOORE[d][1];
                if (!wrap_patch(o, ch.l, P, Q)) continue;
                Key q{ch.l, P, Q};
                bool is_sibling = (q.P / 2 == p.P) && (q.Q / 2 == p.Q);
                if (!is_sibling && o.has_children(q)) return false;
            }
        }
    return true;
}

void validate(const Oracle& o) {
    /* R1: every root active */
    for (int Q = 0; Q < o.NP(1, 0); ++Q)
        for (int P = 0; P < o.NP(0, 0); ++P)
            if (!o.active(Key{0, P, Q})) fail("R1 violated: missing root");
    for (auto& kv : o.tree) {
        const Key& p = kv.first;
        if (p.l > 0) {
            Key par{p.l - 1, p.P / 2, p.Q / 2};
            if (!o.has_children(par)) fail("orphan patch");
        }
        if (kv.second) {
            if (p.l + 1 >= o.c.levels) fail("children beyond max level");
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a)
                    if (!o.active(Key{p.l + 1, 2 * p.P + a, 2 * p.Q + b})) fail("children not all-or-none");
            /* R2 with the out-of-domain exemption (A18) */
            for (int d = 0; d < 8; ++d) {
                int P = p.P + MOORE[d][0], Q = p.Q + MOORE[d][1];
                if (!wrap_patch(o, p.l, P, Q)) continue;
                if (!o.active(Key{p.l, P, Q})) fail("R2 violated");
            }
        } else {
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a)
                    if (o.active(Key{p.l + 1, 2 * p.P + a, 2 * p.Q + b})) fail("leaf with children");
        }
    }
}

/* ------------------------------------------------------------------ restriction / reflux */
/* O9: 2x2 average in the fixed order ((a+b)+(c+d))*0.25, finest level first */
void restrict_parent(const Oracle& o, Field& S, const Key& p) {
    int n = o.n(), l = p.l + 1;
    std::vector<double>& up = S.at(p);
    for (int k = 0; k < NV; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                int a = (2 * i) / n, b = (2 * j) / n;
                const std::vector<double>& uc = S.at(Key{l, 2 * p.P + a, 2 * p.Q + b});
                int fi = 2 * i - a * n, fj = 2 * j - b * n;
                double f00 = uc[(k * n + fj) * n + fi], f10 = uc[(k * n + fj) * n + fi + 1];
                double f01 = uc[(k * n + fj + 1) * n + fi], f11 = uc[(k * n + fj + 1) * n + fi + 1];
                up[(k * n + j) * n + i] = ((f00 + f10) + (f01 + f11)) * 0.25;
            }
}

void restrict_all(const Oracle& o, Field& S) {
    for (int l = o.c.levels - 1; l >= 1; --l) {
        std::vector<Key> parents;   /* level l-1 patches with children; each writes only its own data */
        for (auto& kv : o.tree)
            if (kv.first.l == l - 1 && kv.second) parents.push_back(kv.first);
        par_for((long)parents.size(), [&](long e) { restrict_parent(o, S, parents[e]); });
    }
}

struct Fluxes {
    std::vector<double> X, Y;   /* Fhat of one leaf (see spatial_operator) */
};

/* O12: reflux at coarse/fine faces, sides in the order x-low, x-high, y-low, y-high */
void reflux(const Oracle& o, Field& S, const std::map<Key, Fluxes>& Fh, double bdt) {
    int n = o.n();
    for (auto& kv : o.tree) {
        const Key& p = kv.first;
        if (kv.second) continue;   /* leaves only */
        int l = p.l;
        for (int side = 0; side < 4; ++side) {
            int ax = side / 2, hi = side % 2;
            int P = p.P + (ax == 0 ? (hi ? 1 : -1) : 0), Q = p.Q + (ax == 1 ? (hi ? 1 : -1) : 0);
            if (!wrap_patch(o, l, P, Q)) continue;
            Key q{l, P, Q};
            if (!o.has_children(q)) continue;   /* not a coarse/fine face */
            double h = o.h(ax, l);
            double sigma = hi ? 1.0 : -1.0;
            std::vector<double>& u = S.at(p);
            const Fluxes& fc = Fh.at(p);
            for (int t = 0; t < n; ++t) {
                /* coarse cell K (local) and its face */
                int ci = ax == 0 ? (hi ? n - 1 : 0) : t;
                int cj = ax == 1 ? (hi ? n - 1 : 0) : t;
                int I = p.P * n + ci, J = p.Q * n + cj;
                for (int k = 0; k < NV; ++k) {
                    double Fc = ax == 0 ? fc.X[((size_t)k * n + cj) * (n + 1) + (hi ? n : 0)]
                                        : fc.Y[((size_t)k * (n + 1) + (hi ? n : 0)) * n + ci];
                    double Ff[2];
                    for (int b = 0; b < 2; ++b) {
                        /* the fine cell across the face, and the fine leaf that owns it */
                        int fI, fJ;
                        if (ax == 0) { fI = hi ? 2 * I + 2 : 2 * I - 1; fJ = 2 * J + b; }
                        else { fI = 2 * I + b; fJ = hi ? 2 * J + 2 : 2 * J - 1; }
                        fI = posmod(fI, o.NC(0, l + 1));
                        fJ = posmod(fJ, o.NC(1, l + 1));
                        Key r{l + 1, fI / n, fJ / n};
                        auto it = Fh.find(r);
                        if (it == Fh.end()) fail("reflux: fine neighbour is not a leaf");
                        int li = fI - r.P * n, lj = fJ - r.Q * n;
                        Ff[b] = ax == 0 ? it->second.X[((size_t)k * n + lj) * (n + 1) + (hi ? 0 : n)]
                                        : it->second.Y[((size_t)k * (n + 1) + (hi ? 0 : n)) * n + li];
                    }
                    double delta = Fc - 0.5 * (Ff[0] + Ff[1]);
                    u[((size_t)k * n + cj) * n + ci] += bdt * sigma * delta / h;
                }
            }
        }
    }
}

bool physical(const double* U, double g) {
    double W[4];
    cons2prim(g, U, W);
    for (int k = 0; k < 4; ++k)
        if (!std::isfinite(U[k]) || !std::isfinite(W[k])) return false;
    return W[0] > 0.0 && W[3] > 0.0;
}

/* max that keeps a NaN: once any candidate is NaN the result is NaN (a non-physical cell makes the wave speed,
 * hence dt, undefined -- O13 / S:L412 "errors: NonPositiveState"); otherwise the ordinary maximum */
double nan_max(double a, double b) {
    if (std::isnan(a) || std::isnan(b)) return std::nan("");
    return b > a ? b : a;
}

std::vector<Key> leaf_keys(const Oracle& o) {
    std::vector<Key> v;
    for (auto& kv : o.tree)
        if (!kv.second) v.push_back(kv.first);
    return v;
}

/* O13 ("max over all leaf nodes of [(|u|+c)/dx + (|v|+c)/dy]; uses each patch's own level spacing"):
 * Lambda = max over leaf cells of (|u|+c)/dx_l + (|v|+c)/dy_l.  norm_level = 1 divides each leaf's value by 2^l
 * (subcycling reading S6).  The max is order-independent, so the per-patch maxima may be taken in parallel. */
double lambda_of(const Oracle& o, bool norm_level) {
    int n = o.n();
    std::vector<Key> lv = leaf_keys(o);
    std::vector<double> pm(lv.size(), 0.0);
    par_for((long)lv.size(), [&](long e) {
        const Key& p = lv[e];
        const std::vector<double>& u = o.U.at(p);
        double dx = o.h(0, p.l), dy = o.h(1, p.l);
        double lam = 0.0;
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                double Uc[4], W[4];
                for (int k = 0; k < NV; ++k) Uc[k] = u[((size_t)k * n + j) * n + i];
                cons2prim(o.c.gamma, Uc, W);
                double cs = std::sqrt(o.c.gamma * W[3] / W[0]);
                double s = (std::fabs(W[1]) + cs) / dx + (std::fabs(W[2]) + cs) / dy;
                if (norm_level) s = s / (double)(1 << p.l);
                lam = nan_max(lam, s);
            }
        pm[e] = lam;
    });
    double lam = 0.0;
    for (double v : pm) lam = nan_max(lam, v);
    return lam;
}

double lambda_max(const Oracle& o) { return lambda_of(o, false); }

/* O11 stage s (0, 1, 2) of SSP-RK3 (Shu-Osher form S:L419): U^(s+1) from U^(s) = prev and U^n = Un on
 * every leaf, then O12 reflux (skipped when the test-only switch c.reflux is 0: the no-reflux control), then O9
 * restriction, then the positivity check of the leaves.  Leaves are independent within the stage. */
void stage(Oracle& o, const Field& Un, Field& prev, int s, double dt) {
    int n = o.n(), g = o.ghost_width();
    const double a_s[3] = {0.0, 0.75, 1.0 / 3.0};
    const double b_s[3] = {1.0, 0.25, 2.0 / 3.0};
    std::vector<Key> lv = leaf_keys(o);
    Field next = prev;
    std::vector<Fluxes> F(lv.size());
    par_for((long)lv.size(), [&](long e) {
        const Key& p = lv[e];
        std::vector<double> tile = build_tile(o, prev, p, g);
        std::vector<double> L;
        spatial_operator(o, tile, p.l, L, F[e].X, F[e].Y);
        std::vector<double>& out = next.at(p);
        const std::vector<double>& un = Un.at(p);
        const std::vector<double>& up = prev.at(p);
        for (size_t q = 0; q < out.size(); ++q) {
            if (s == 0) out[q] = un[q] + dt * L[q];
            else out[q] = a_s[s] * un[q] + b_s[s] * (up[q] + dt * L[q]);
        }
    });
    std::map<Key, Fluxes> Fh;
    for (size_t e = 0; e < lv.size(); ++e) {
        Fluxes& d = Fh[lv[e]];
        d.X.swap(F[e].X);
        d.Y.swap(F[e].Y);
    }
    if (o.c.reflux) reflux(o, next, Fh, b_s[s] * dt);
    restrict_all(o, next);
    for (const Key& p : lv) {
        const std::vector<double>& u = next.at(p);
        for (int q = 0; q < n * n; ++q) {
            double Uc[4] = {u[q], u[n * n + q], u[2 * n * n + q], u[3 * n * n + q]};
            if (o.c.check_positivity && !physical(Uc, o.c.gamma)) {
                char b[200];
                std::snprintf(b, sizeof b, "non-physical state at stage %d, patch (l=%d,P=%d,Q=%d), cell %d", s + 1,
                              p.l, p.P, p.Q, q);
                throw std::domain_error(b);
            }
        }
    }
    prev.swap(next);
}

/* O11: one SSP-RK3 step on the whole composite mesh; U^n is replaced only when all three stages succeed */
void step(Oracle& o, double dt) {
    Field prev = o.U;
    for (int s = 0; s < 3; ++s) stage(o, o.U, prev, s, dt);
    o.U.swap(prev);
}

/* ------------------------------------------------------------------ NEXT #4: Berger-Colella time subcycling
 * Readings S1-S8 (SURVEY s8(f) NEXT #4, S:L441-445 -- the paper itself uses one global dt):
 *  S1 level l advances with dt_l = dt_0 / 2^l: advance(l) takes one SSP-RK3 step of EVERY active level-l patch
 *     (leaves and covered patches), then advance(l+1) twice, then refluxes the level-l leaves and restricts
 *     level l+1 into the covered level-l patches;
 *  S2 a level-l ghost with no same-level patch is the O8 prolongation of the level-(l-1) field taken linearly in
 *     time, U_{l-1}(tau) = U_old + theta (U_new - U_old), theta = (tau - t_old) / dt_{l-1}, at the stage time tau
 *     = t + c_s dt_l with the SSP-RK3 abscissae c = (0, 1, 1/2);
 *  S3 flux registers accumulate the time integral of F-hat over a step with the SSP-RK3 quadrature weights
 *     w = (1/6, 1/6, 2/3): coarse side sum_s w_s F_s, fine side sum over both substeps of (1/2) sum_s w_s F_s;
 *  S4 reflux after the substeps: U += sigma dt_l / h (F_coarse - mean of the two fine faces), O12's sign and side
 *     order;
 *  S5 positivity is checked on the leaves after every stage of their level;
 *  S6 dt_0 = CFL / max over leaf cells of ((|u|+c)/dx_l + (|v|+c)/dy_l) / 2^l (every level at CFL <= cfl). */
const double SSP_C[3] = {0.0, 1.0, 0.5};
const double SSP_W[3] = {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0};

/* S6 */
double lambda_subcycled(const Oracle& o) { return lambda_of(o, true); }

/* C/F side classification of leaf p: 1 coarse side (same-level neighbour has children), 2 fine side (no
 * same-level neighbour inside the domain), 0 otherwise */
int cf_side(const Oracle& o, const Key& p, int side) {
    int ax = side / 2, hi = side % 2;
    int P = p.P + (ax == 0 ? (hi ? 1 : -1) : 0), Q = p.Q + (ax == 1 ? (hi ? 1 : -1) : 0);
    if (!wrap_patch(o, p.l, P, Q)) return 0;
    Key q{p.l, P, Q};
    if (!o.active(q)) return 2;
    return o.has_children(q) ? 1 : 0;
}

struct Subcycler {
    Oracle& o;
    std::vector<Field> old_state;                 /* per level: the level's patches at the start of its step */
    std::vector<double> t_old, dt_lev;            /* per level: start time and length of its current step */
    /* S3: per level, leaf -> [4 sides][NV][n] accumulated F-hat; accC: coarse sides over one step of the level,
     * accF: fine sides over the two substeps of the level within one step of its parent level */
    std::vector<std::map<Key, std::vector<double>>> accC, accF;

    explicit Subcycler(Oracle& oo) : o(oo), old_state(oo.c.levels), t_old(oo.c.levels), dt_lev(oo.c.levels),
                                     accC(oo.c.levels), accF(oo.c.levels) {}

    std::vector<double>& reg(std::map<Key, std::vector<double>>& m, const Key& p) {
        auto it = m.find(p);
        if (it == m.end()) it = m.emplace(p, std::vector<double>((size_t)4 * NV * o.n(), 0.0)).first;
        return it->second;
    }

    /* S3: F-hat on leaf p's C/F sides into its registers, with weight w (coarse side) or w/2 (fine side) */
    void accumulate(const Key& p, const Fluxes& F, double w) {
        int n = o.n();
        for (int side = 0; side < 4; ++side) {
            int kind = cf_side(o, p, side);
            if (kind == 0) continue;
            int ax = side / 2, hi = side % 2;
            std::vector<double>& a = kind == 1 ? reg(accC[p.l], p) : reg(accF[p.l], p);
            double wgt = kind == 1 ? w : 0.5 * w;
            for (int k = 0; k < NV; ++k)
                for (int t = 0; t < n; ++t) {
                    double f = ax == 0 ? F.X[((size_t)k * n + t) * (n + 1) + (hi ? n : 0)]
                                       : F.Y[((size_t)k * (n + 1) + (hi ? n : 0)) * n + t];
                    a[((size_t)side * NV + k) * n + t] += wgt * f;
                }
        }
    }

    /* S1, S2, S5: one SSP-RK3 step of every active level-l patch from t0 with dt */
    void step_level(int l, double t0, double dt) {
        int n = o.n(), g = o.ghost_width();
        const double a_s[3] = {0.0, 0.75, 1.0 / 3.0};
        const double b_s[3] = {1.0, 0.25, 2.0 / 3.0};
        Field Un;
        for (auto& kv : o.tree)
            if (kv.first.l == l) Un[kv.first] = o.U.at(kv.first);
        old_state[l] = Un;
        t_old[l] = t0;
        dt_lev[l] = dt;
        Field prev = Un;
        for (int s = 0; s < 3; ++s) {
            /* what a level-l tile reads: level l at this stage, level l-1 linearly in time (S2) */
            Field view = prev;
            if (l > 0) {
                double theta = (t0 + SSP_C[s] * dt - t_old[l - 1]) / dt_lev[l - 1];
                for (auto& kv : old_state[l - 1]) {
                    const std::vector<double>& uo = kv.second;
                    const std::vector<double>& un = o.U.at(kv.first);
                    std::vector<double> u(uo.size());
                    for (size_t e = 0; e < u.size(); ++e) u[e] = uo[e] + theta * (un[e] - uo[e]);
                    view[kv.first] = u;
                }
            }
            Field next = prev;
            std::vector<Key> pl;   /* every active level-l patch (S1); independent within the stage */
            for (auto& kv : o.tree)
                if (kv.first.l == l) pl.push_back(kv.first);
            std::vector<Fluxes> F(pl.size());
            par_for((long)pl.size(), [&](long e) {
                const Key& p = pl[e];
                std::vector<double> tile = build_tile(o, view, p, g);
                std::vector<double> L;
                spatial_operator(o, tile, l, L, F[e].X, F[e].Y);
                std::vector<double>& out = next.at(p);
                const std::vector<double>& un = Un.at(p);
                const std::vector<double>& up = prev.at(p);
                for (size_t q = 0; q < out.size(); ++q) {
                    if (s == 0) out[q] = un[q] + dt * L[q];
                    else out[q] = a_s[s] * un[q] + b_s[s] * (up[q] + dt * L[q]);
                }
            });
            for (size_t e = 0; e < pl.size(); ++e) {
                const Key& p = pl[e];
                if (o.has_children(p)) continue;
                /* leaf: flux registers (S3), positivity (S5) */
                accumulate(p, F[e], SSP_W[s]);
                const std::vector<double>& out = next.at(p);
                for (int q = 0; q < n * n; ++q) {
                    double Uc[4] = {out[q], out[n * n + q], out[2 * n * n + q], out[3 * n * n + q]};
                    if (o.c.check_positivity && !physical(Uc, o.c.gamma)) {
                        char b[200];
                        std::snprintf(b, sizeof b, "non-physical state at level %d stage %d, patch (P=%d,Q=%d), cell %d",
                                      l, s + 1, p.P, p.Q, q);
                        throw std::domain_error(b);
                    }
                }
            }
            prev.swap(next);
        }
        for (auto& kv : prev) o.U[kv.first] = kv.second;
    }

    /* S4: the coarse leaves of level l against the fine registers of level l+1 (O12 sides, order, sign) */
    void reflux_level(int l) {
        int n = o.n();
        double dt = dt_lev[l];
        for (auto& kv : o.tree) {
            const Key& p = kv.first;
            if (p.l != l || kv.second) continue;
            for (int side = 0; side < 4; ++side) {
                if (cf_side(o, p, side) != 1) continue;
                int ax = side / 2, hi = side % 2;
                double h = o.h(ax, l);
                double sigma = hi ? 1.0 : -1.0;
                std::vector<double>& u = o.U.at(p);
                const std::vector<double>& ac = reg(accC[l], p);
                for (int t = 0; t < n; ++t) {
                    int ci = ax == 0 ? (hi ? n - 1 : 0) : t;
                    int cj = ax == 1 ? (hi ? n - 1 : 0) : t;
                    int I = p.P * n + ci, J = p.Q * n + cj;
                    for (int k = 0; k < NV; ++k) {
                        double Fc = ac[((size_t)side * NV + k) * n + t];
                        double Ff[2];
                        for (int b = 0; b < 2; ++b) {
                            int fI, fJ;
                            if (ax == 0) { fI = hi ? 2 * I + 2 : 2 * I - 1; fJ = 2 * J + b; }
                            else { fI = 2 * I + b; fJ = hi ? 2 * J + 2 : 2 * J - 1; }
                            fI = posmod(fI, o.NC(0, l + 1));
                            fJ = posmod(fJ, o.NC(1, l + 1));
                            Key r{l + 1, fI / n, fJ / n};
                            if (!o.active(r) || o.has_children(r)) fail("subcycle reflux: fine neighbour is not a leaf");
                            int li = fI - r.P * n, lj = fJ - r.Q * n;
                            const std::vector<double>& af = reg(accF[l + 1], r);
                            Ff[b] = af[((size_t)(side ^ 1) * NV + k) * n + (ax == 0 ? lj : li)];
                        }
                        double delta = Fc - 0.5 * (Ff[0] + Ff[1]);
                        u[((size_t)k * n + cj) * n + ci] += dt * sigma * delta / h;
                    }
                }
            }
        }
    }

    /* O9 for one level pair: level l+1 into the covered level-l patches, fixed order */
    void restrict_level(int l) {
        int n = o.n();
        for (auto& kv : o.tree) {
            const Key& p = kv.first;
            if (p.l != l || !kv.second) continue;
            std::vector<double>& up = o.U.at(p);
            for (int k = 0; k < NV; ++k)
                for (int j = 0; j < n; ++j)
                    for (int i = 0; i < n; ++i) {
                        int a = (2 * i) / n, b = (2 * j) / n;
                        const std::vector<double>& uc = o.U.at(Key{l + 1, 2 * p.P + a, 2 * p.Q + b});
                        int fi = 2 * i - a * n, fj = 2 * j - b * n;
                        double f00 = uc[(k * n + fj) * n + fi], f10 = uc[(k * n + fj) * n + fi + 1];
                        double f01 = uc[(k * n + fj + 1) * n + fi], f11 = uc[(k * n + fj + 1) * n + fi + 1];
                        up[(k * n + j) * n + i] = ((f00 + f10) + (f01 + f11)) * 0.25;
                    }
        }
    }

    bool level_exists(int l) const {
        if (l >= o.c.levels) return false;
        for (auto& kv : o.tree)
            if (kv.first.l == l) return true;
        return false;
    }

    /* S1: step level l, then twice the next level, then reflux and restriction at the common time */
    void advance(int l, double t0, double dt) {
        accC[l].clear();
        step_level(l, t0, dt);
        if (!level_exists(l + 1)) return;
        accF[l + 1].clear();
        advance(l + 1, t0, 0.5 * dt);
        advance(l + 1, t0 + 0.5 * dt, 0.5 * dt);
        reflux_level(l);
        restrict_level(l);
    }
};

void step_subcycled(Oracle& o, double dt0) {
    Subcycler sc(o);
    sc.advance(0, 0.0, dt0);
}

/* O6: per-leaf refinement indicator eta = dx sqrt(gx^2 + gy^2) / rho (BJ configs[0], A19) */
struct LeafFlag {
    double maxeta;
    bool ambiguous;
};
std::map<Key, LeafFlag> leaf_flags(const Oracle& o) {
    int n = o.n(), g = 1, w = n + 2;
    double th = o.c.theta, tc = o.c.theta * o.c.coarsen_frac;
    std::vector<Key> lv = leaf_keys(o);
    std::vector<LeafFlag> fl(lv.size());
    par_for((long)lv.size(), [&](long e) {
        const Key& p = lv[e];
        std::vector<double> t = build_tile(o, o.U, p, g);
        double dx = o.h(0, p.l), dy = o.h(1, p.l);
        LeafFlag f{0.0, false};
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                auto R = [&](int jj, int ii) { return t[(size_t)(jj + g) * w + (ii + g)]; };
                double gx = (R(j, i + 1) - R(j, i - 1)) / (2.0 * dx);
                double gy = (R(j + 1, i) - R(j - 1, i)) / (2.0 * dy);
                double eta = dx * std::sqrt(gx * gx + gy * gy) / R(j, i);
                if (!(eta <= f.maxeta)) f.maxeta = eta;
                /* A32: within 1e-9 relative of either threshold */
                if (std::fabs(eta - th) <= 1e-9 * th || std::fabs(eta - tc) <= 1e-9 * tc) f.ambiguous = true;
            }
        fl[e] = f;
    });
    std::map<Key, LeafFlag> out;
    for (size_t e = 0; e < lv.size(); ++e) out[lv[e]] = fl[e];
    return out;
}

/* O8 for whole new patches, then O9 -- the data half of a regrid */
void regrid_apply(Oracle& o, const std::map<Key, char>& old_tree) {
    int n = o.n();
    for (int l = 1; l < o.c.levels; ++l) {
        std::vector<Key> fresh;   /* new level-l patches; they read level l-1 only, so they are independent */
        for (auto& kv : o.tree)
            if (kv.first.l == l && !old_tree.count(kv.first)) fresh.push_back(kv.first);
        std::vector<std::vector<double>> val(fresh.size());
        par_for((long)fresh.size(), [&](long e) {
            const Key& p = fresh[e];
            std::vector<double> u((size_t)NV * n * n);
            for (int k = 0; k < NV; ++k)
                for (int j = 0; j < n; ++j)
                    for (int i = 0; i < n; ++i)
                        u[((size_t)k * n + j) * n + i] = prolong_value(o, o.U, l, p.P * n + i, p.Q * n + j, k);
            val[e].swap(u);
        });
        for (size_t e = 0; e < fresh.size(); ++e) o.U[fresh[e]].swap(val[e]);
    }
    for (auto it = o.U.begin(); it != o.U.end();) {
        if (!o.tree.count(it->first)) it = o.U.erase(it);
        else ++it;
    }
    restrict_all(o, o.U);
}

void regrid_requests(Oracle& o, const std::set<Key>& ref, const std::set<Key>& crs, int* nr, int* nc) {
    std::map<Key, char> old_tree = o.tree;
    int n_ref = 0, n_crs = 0;
    /* refinement pass (O4): flagged leaves below the top level, canonical order */
    for (const Key& p : ref) {
        if (!o.active(p) || o.has_children(p) || p.l >= o.c.levels - 1) continue;
        refine(o, p);
    }
    /* coarsening pass (O5): levels fine to coarse, canonical order within a level */
    for (int l = o.c.levels - 2; l >= 0; --l)
        for (const Key& p : crs) {
            if (p.l != l || !o.active(p)) continue;
            if (!coarsen_allowed(o, p)) continue;
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a) o.tree.erase(Key{l + 1, 2 * p.P + a, 2 * p.Q + b});
            o.tree[p] = 0;
        }
    validate(o);
    for (auto& kv : o.tree)
        if (!old_tree.count(kv.first) && kv.first.l > 0) ++n_ref;
    for (auto& kv : old_tree)
        if (!o.tree.count(kv.first)) ++n_crs;
    regrid_apply(o, old_tree);
    if (nr) *nr = n_ref;
    if (nc) *nc = n_crs;
}

Oracle* H(void* h) { return static_cast<Oracle*>(h); }

template <class F>
int guarded(void* h, F f) {
    if (!h) return 1;
    try {
        f();
        return 0;
    } catch (const std::domain_error& e) {
        H(h)->err = e.what();
        return 3;
    } catch (const std::exception& e) {
        H(h)->err = e.what();
        return 4;
    }
}

}  // namespace

/* ------------------------------------------------------------------ C API */
extern "C" {

void* orc_create(const orc_config* cfg) {
    if (!cfg) return nullptr;
    const orc_config& c = *cfg;
    if (c.n < 8 || c.base[0] % c.n || c.base[1] % c.n || c.base[0] <= 0 || c.base[1] <= 0) return nullptr;
    if (c.levels < 1 || c.levels > 12 || !(c.gamma > 1.0)) return nullptr;
    for (int ax = 0; ax < 2; ++ax)
        if ((c.bc[2 * ax] == BC_PERIODIC) != (c.bc[2 * ax + 1] == BC_PERIODIC)) return nullptr;
    Oracle* o = new Oracle();
    o->c = c;
    /* R1 scaffold */
    for (int Q = 0; Q < o->NP(1, 0); ++Q)
        for (int P = 0; P < o->NP(0, 0); ++P) {
            o->tree[Key{0, P, Q}] = 0;
            o->U[Key{0, P, Q}] = std::vector<double>((size_t)NV * c.n * c.n, 0.0);
        }
    return o;
}

void orc_destroy(void* h) { delete H(h); }
const char* orc_error(void* h) { return h ? H(h)->err.c_str() : "null handle"; }
int orc_num_patches(void* h) { return h ? (int)H(h)->tree.size() : -1; }

int orc_get_tree(void* h, int cap, int* level, int* P, int* Q, int* leaf, int* nchild_leaf) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        if (cap < (int)o.tree.size()) fail("capacity");
        int e = 0;
        for (auto& kv : o.tree) {
            level[e] = kv.first.l;
            P[e] = kv.first.P;
            Q[e] = kv.first.Q;
            leaf[e] = kv.second ? 0 : 1;
            if (nchild_leaf) nchild_leaf[e] = children_all_leaves(o, kv.first) ? 1 : 0;
            ++e;
        }
    });
}

int orc_validate(void* h) { return guarded(h, [&] { validate(*H(h)); }); }

int orc_set_patch(void* h, int l, int P, int Q, const double* U) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        Key k{l, P, Q};
        if (!o.active(k)) fail("set_patch: inactive patch");
        o.U[k].assign(U, U + (size_t)NV * o.n() * o.n());
    });
}

int orc_get_patch(void* h, int l, int P, int Q, double* U) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        Key k{l, P, Q};
        if (!o.active(k)) fail("get_patch: inactive patch");
        const std::vector<double>& u = o.U.at(k);
        std::memcpy(U, u.data(), u.size() * sizeof(double));
    });
}

int orc_restrict_all(void* h) { return guarded(h, [&] { restrict_all(*H(h), H(h)->U); }); }

int orc_lambda(void* h, double* lam) { return guarded(h, [&] { *lam = lambda_max(*H(h)); }); }
int orc_lambda_subcycled(void* h, double* lam) { return guarded(h, [&] { *lam = lambda_subcycled(*H(h)); }); }

int orc_stage1(void* h, double dt) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        Field prev = o.U;
        stage(o, o.U, prev, 0, dt);
        o.U.swap(prev);
    });
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_get_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int orc_totals(void* h, double* out4) {
    /* O18: M_k = sum over leaf cells of U_k dx dy, accumulated in long double */
    return guarded(h, [&] {
        Oracle& o = *H(h);
        int n = o.n();
        long double s[4] = {0, 0, 0, 0};
        for (auto& kv : o.tree) {
            if (kv.second) continue;
            double dv = o.h(0, kv.first.l) * o.h(1, kv.first.l);
            const std::vector<double>& u = o.U.at(kv.first);
            for (int k = 0; k < NV; ++k)
                for (int e = 0; e < n * n; ++e) s[k] += (long double)u[(size_t)k * n * n + e] * dv;
        }
        for (int k = 0; k < 4; ++k) out4[k] = (double)s[k];
    });
}

int orc_step(void* h, double dt, double cfl, double* dt_used) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        double d = dt;
        if (!(d > 0.0)) {
            if (!(cfl > 0.0)) fail("need dt > 0 or cfl > 0");
            double lam = lambda_max(o);
            if (!(lam > 0.0) || !std::isfinite(lam)) throw std::domain_error("non-finite wave speed");
            d = cfl / lam;   /* O13 */
        }
        step(o, d);
        if (dt_used) *dt_used = d;
    });
}

int orc_step_subcycled(void* h, double dt0, double cfl, double* dt_used) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        double d = dt0;
        if (!(d > 0.0)) {
            if (!(cfl > 0.0)) fail("need dt > 0 or cfl > 0");
            double lam = lambda_subcycled(o);
            if (!(lam > 0.0) || !std::isfinite(lam)) throw std::domain_error("non-finite wave speed");
            d = cfl / lam;   /* S6 */
        }
        step_subcycled(o, d);
        if (dt_used) *dt_used = d;
    });
}

int orc_flags(void* h, int cap, double* maxeta, unsigned char* refine_out, unsigned char* coarsen_out,
              unsigned char* ambiguous) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        if (cap < (int)o.tree.size()) fail("capacity");
        std::map<Key, LeafFlag> lf = leaf_flags(o);
        double th = o.c.theta, tc = o.c.theta * o.c.coarsen_frac;
        int e = 0;
        for (auto& kv : o.tree) {
            const Key& p = kv.first;
            double m = std::nan("");
            bool rf = false, cf = false, amb = false;
            if (!kv.second) {
                m = lf.at(p).maxeta;
                amb = lf.at(p).ambiguous;
                rf = p.l < o.c.levels - 1 && m > th;
            } else if (children_all_leaves(o, p)) {
                m = 0.0;
                for (int b = 0; b < 2; ++b)
                    for (int a = 0; a < 2; ++a) {
                        const LeafFlag& f = lf.at(Key{p.l + 1, 2 * p.P + a, 2 * p.Q + b});
                        if (!(f.maxeta <= m)) m = f.maxeta;
                        amb = amb || f.ambiguous;
                    }
                cf = m < tc;
            }
            maxeta[e] = m;
            refine_out[e] = rf;
            coarsen_out[e] = cf;
            ambiguous[e] = amb;
            ++e;
        }
    });
}

int orc_regrid_with_requests(void* h, int m, const int* l, const int* P, const int* Q, const unsigned char* rf,
                             const unsigned char* cf, int* n_refined, int* n_coarsened) {
    return guarded(h, [&] {
        std::set<Key> ref, crs;
        for (int e = 0; e < m; ++e) {
            if (rf[e]) ref.insert(Key{l[e], P[e], Q[e]});
            if (cf[e]) crs.insert(Key{l[e], P[e], Q[e]});
        }
        regrid_requests(*H(h), ref, crs, n_refined, n_coarsened);
    });
}

int orc_regrid(void* h, int* n_refined, int* n_coarsened) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        int np = (int)o.tree.size();
        std::vector<double> me(np);
        std::vector<unsigned char> rf(np), cf(np), am(np);
        if (orc_flags(h, np, me.data(), rf.data(), cf.data(), am.data())) fail(o.err);
        std::set<Key> ref, crs;
        int e = 0;
        for (auto& kv : o.tree) {
            if (rf[e]) ref.insert(kv.first);
            if (cf[e]) crs.insert(kv.first);
            ++e;
        }
        regrid_requests(o, ref, crs, n_refined, n_coarsened);
    });
}

int orc_ghost_tile(void* h, int l, int P, int Q, int g, double* tile) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        Key k{l, P, Q};
        if (!o.active(k)) fail("ghost_tile: inactive patch");
        if (g < 1 || g > o.n()) fail("ghost width");
        std::vector<double> t = build_tile(o, o.U, k, g);
        std::memcpy(tile, t.data(), t.size() * sizeof(double));
    });
}

int orc_rhs(void* h, int l, int P, int Q, double* Lout) {
    return guarded(h, [&] {
        Oracle& o = *H(h);
        Key k{l, P, Q};
        if (!o.active(k) || o.has_children(k)) fail("rhs: not a leaf");
        std::vector<double> t = build_tile(o, o.U, k, o.ghost_width());
        std::vector<double> L, fx, fy;
        spatial_operator(o, t, l, L, fx, fy);
        std::memcpy(Lout, L.data(), L.size() * sizeof(double));
    });
}

void orc_cons2prim(double gamma, const double* U, double* W) { cons2prim(gamma, U, W); }
void orc_prim2cons(double gamma, const double* W, double* U) { prim2cons(gamma, W, U); }
void orc_euler_flux_x(double gamma, const double* U, double* F) { euler_flux_x(gamma, U, F); }
void orc_rusanov_x(double gamma, const double* UL, const double* UR, double* F) { rusanov_x(gamma, UL, UR, F); }
double orc_weno5(const double* v, double eps) { return weno5(v, eps); }
void orc_eigen_x(double gamma, const double* WL, const double* WR, double* Lm, double* Rm) {
    eigen_x(gamma, WL, WR, Lm, Rm);
}
void orc_face_flux_x(const orc_config* cfg, const double* cells, double* F) {
    double c6[6][4];
    std::memcpy(c6, cells, sizeof c6);
    face_flux_x(*cfg, c6, F);
}
double orc_mc(double a, double b) { return mc(a, b); }

}  // extern "C"
