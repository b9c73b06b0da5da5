"""Seeded synthetic inputs for the hot path: the BASELINE.json configs as concrete ICs.

This module is shared by the oracle side (tests) and the CUDA side (tests, bench)
and therefore holds NONE of the method's arithmetic: only the initial conditions
(s8(d) D1-D5, A21-A30) and the counter-based
SplitMix64 generator.  Each IC is evaluated as point values at cell centres
(A33) and returned as conserved variables (rho, rho u, rho v, rho e) with
rho e = p/(gamma-1) + rho (u^2+v^2)/2, the IC's definition (Eq. 4-6).

Config dict keys: lo, hi, base, n, levels, gamma, bc (x-lo, x-hi, y-lo, y-hi),
scheme, characteristic, div_order, weno_eps, theta, coarsen_frac, coarsen_rule,
ic (name), seed, cfl, regrid_every.
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = 1.4

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """O15: SplitMix64 finaliser (Steele, Lea, Flood 2014), vectorised over uint64."""
    with np.errstate(over="ignore"):
        z = (np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, k, lo: float, hi: float):
    """O15: u(seed,k) = (sm64(sm64(seed) ^ k) >> 11) * 2^-53; value = lo + (hi-lo)*u (no FMA)."""
    s = splitmix64(np.uint64(seed))
    z = splitmix64(s ^ np.asarray(k, dtype=np.uint64))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    t = (hi - lo) * u
    return lo + t


def to_conserved(rho, u, v, p, gamma=GAMMA):
    rho, u, v, p = (np.asarray(a, dtype=np.float64) for a in (rho, u, v, p))
    E = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    return np.stack([rho, rho * u, rho * v, E])


def cell_centres(cfg, l, P, Q):
    """O1: centres (lo + (I+1/2) dx_l) of patch (l,P,Q); returns X[n][n], Y[n][n] (index [j][i])."""
    n = cfg["n"]
    dx = (cfg["hi"][0] - cfg["lo"][0]) / (cfg["base"][0] * float(1 << l))
    dy = (cfg["hi"][1] - cfg["lo"][1]) / (cfg["base"][1] * float(1 << l))
    I = P * n + np.arange(n)
    J = Q * n + np.arange(n)
    x = cfg["lo"][0] + (I + 0.5) * dx
    y = cfg["lo"][1] + (J + 0.5) * dy
    X, Y = np.meshgrid(x, y)
    return X, Y


# ----------------------------------------------------------------- initial conditions (primitive)
def ic_uniform(cfg, X, Y, l=0, I=None, J=None):
    w = cfg.get("uniform_state", (1.0, 0.3, -0.2, 1.0))
    return tuple(np.full_like(X, c) for c in w)


def ic_sod(cfg, X, Y, **_):
    """BJ configs[0]: (1,0,1) left of x=0.5, (0.125,0,0.1) right; v = 0."""
    left = X < 0.5
    rho = np.where(left, 1.0, 0.125)
    p = np.where(left, 1.0, 0.1)
    z = np.zeros_like(X)
    return rho, z, z.copy(), p


def vortex_prim(cfg, X, Y, t=0.0):
    """O17: isentropic vortex (BJ configs[1]); exact solution = IC shifted by (u0 t, v0 t), centre wrapped."""
    g = cfg.get("gamma", GAMMA)
    beta = cfg.get("vortex_beta", 5.0)
    u0, v0 = cfg.get("vortex_free", (1.0, 1.0))
    Lx = cfg["hi"][0] - cfg["lo"][0]
    Ly = cfg["hi"][1] - cfg["lo"][1]
    xc0, yc0 = cfg.get("vortex_centre", (cfg["lo"][0] + 0.5 * Lx, cfg["lo"][1] + 0.5 * Ly))
    xc = cfg["lo"][0] + (xc0 + u0 * t - cfg["lo"][0]) % Lx
    yc = cfg["lo"][1] + (yc0 + v0 * t - cfg["lo"][1]) % Ly
    # nearest periodic image of the centre
    dxr = X - xc
    dyr = Y - yc
    dxr = dxr - Lx * np.round(dxr / Lx)
    dyr = dyr - Ly * np.round(dyr / Ly)
    r2 = dxr * dxr + dyr * dyr
    e = np.exp(0.5 * (1.0 - r2))
    du = -beta / (2.0 * math.pi) * e * dyr
    dv = beta / (2.0 * math.pi) * e * dxr
    T = 1.0 - (g - 1.0) * beta * beta / (8.0 * g * math.pi ** 2) * np.exp(1.0 - r2)
    rho = T ** (1.0 / (g - 1.0))
    p = rho * T
    return rho, u0 + du, v0 + dv, p


def ic_vortex(cfg, X, Y, **_):
    return vortex_prim(cfg, X, Y, 0.0)


def quadrant_states(seed):
    """A27: quadrant q in {0:(x>1/2,y>1/2), 1:(x<1/2,y>1/2), 2:(x<1/2,y<1/2), 3:(x>1/2,y<1/2)};
    key k = 4q + var, var order (rho, u, v, p); rho, p ~ U[0.1,1.5], u, v ~ U[-1,1]."""
    st = np.zeros((4, 4))
    for q in range(4):
        st[q, 0] = uniform(seed, 4 * q + 0, 0.1, 1.5)
        st[q, 1] = uniform(seed, 4 * q + 1, -1.0, 1.0)
        st[q, 2] = uniform(seed, 4 * q + 2, -1.0, 1.0)
        st[q, 3] = uniform(seed, 4 * q + 3, 0.1, 1.5)
    return st


def ic_quadrant(cfg, X, Y, **_):
    st = quadrant_states(cfg.get("seed", 1))
    xm = cfg["lo"][0] + 0.5 * (cfg["hi"][0] - cfg["lo"][0])
    ym = cfg["lo"][1] + 0.5 * (cfg["hi"][1] - cfg["lo"][1])
    q = np.where(Y > ym, np.where(X > xm, 0, 1), np.where(X < xm, 2, 3))
    return st[q, 0], st[q, 1], st[q, 2], st[q, 3]


def rankine_hugoniot(M, rho1=1.0, p1=1.0, gamma=GAMMA):
    """s8(d) D4: post-shock state of a Mach-M shock into gas at rest."""
    c1 = math.sqrt(gamma * p1 / rho1)
    p2 = p1 * (1.0 + 2.0 * gamma / (gamma + 1.0) * (M * M - 1.0))
    rho2 = rho1 * (gamma + 1.0) * M * M / ((gamma - 1.0) * M * M + 2.0)
    W = M * c1
    u2 = W * (1.0 - rho1 / rho2)
    return rho2, u2, p2, W


def ic_shock_bubble(cfg, X, Y, **_):
    """A24 / D4w: Mach 1.22 shock at x=0.2 into (1,0,0,1); bubble rho=0.138, r=0.2 at (0.6, k+0.5)."""
    g = cfg.get("gamma", GAMMA)
    rho2, u2, p2, _ = rankine_hugoniot(cfg.get("mach", 1.22), 1.0, 1.0, g)
    rho = np.ones_like(X)
    u = np.zeros_like(X)
    p = np.ones_like(X)
    nb = cfg.get("bubbles", 1)
    for k in range(nb):
        inside = (X - 0.6) ** 2 + (Y - (k + 0.5)) ** 2 < 0.2 ** 2
        rho = np.where(inside, 0.138, rho)
    post = X < 0.2
    rho = np.where(post, rho2, rho)
    u = np.where(post, u2, u)
    p = np.where(post, p2, p)
    return rho, u, np.zeros_like(X), p


def ic_implosion(cfg, X, Y, l=0, I=None, J=None, **_):
    """Eq. 13: (rho,p) = (0.125,0.140) where |x|+|y| < 0.15, else (1,1); at rest.  On the centred
    domain the cell-centre coordinates are evaluated from the cell index as |2I+1-N| h/2 so that mirrored cells get
    bit-identical |x| (cells with |x|+|y| exactly 0.15 exist at every N = 64 k and must not be decided by the
    rounding of lo + (I+1/2) h)."""
    lo, hi = cfg["lo"], cfg["hi"]
    if I is not None and J is not None and lo[0] == -hi[0] and lo[1] == -hi[1]:
        Nx, Ny = cfg["base"][0] << l, cfg["base"][1] << l
        ax = np.abs(2 * np.asarray(I, dtype=np.int64) + 1 - Nx) * (0.5 * (hi[0] - lo[0]) / Nx)
        ay = np.abs(2 * np.asarray(J, dtype=np.int64) + 1 - Ny) * (0.5 * (hi[1] - lo[1]) / Ny)
        inside = ax + ay < 0.15
    else:
        inside = np.abs(X) + np.abs(Y) < 0.15
    rho = np.where(inside, 0.125, 1.0)
    p = np.where(inside, 0.140, 1.0)
    z = np.zeros_like(X)
    return rho, z, z.copy(), p


def ic_noise(cfg, X, Y, l=0, I=None, J=None):
    """D5: per-cell (rho,u,v,p) from O15 with key 4*(J*Nx + I) + var; rho,p ~ U[0.5,2], u,v ~ U[-1,1]."""
    seed = cfg.get("seed", 7)
    Nx = cfg["base"][0] << l
    k = 4 * (J.astype(np.uint64) * np.uint64(Nx) + I.astype(np.uint64))
    rho = uniform(seed, k + np.uint64(0), 0.5, 2.0)
    u = uniform(seed, k + np.uint64(1), -1.0, 1.0)
    v = uniform(seed, k + np.uint64(2), -1.0, 1.0)
    p = uniform(seed, k + np.uint64(3), 0.5, 2.0)
    return rho, u, v, p


def ic_smooth(cfg, X, Y, **_):
    """Smooth periodic entropy/acoustic-free test state for parity (density wave advected by (u0,v0))."""
    Lx = cfg["hi"][0] - cfg["lo"][0]
    Ly = cfg["hi"][1] - cfg["lo"][1]
    a = cfg.get("amp", 0.2)
    rho = 1.0 + a * np.sin(2 * math.pi * (X - cfg["lo"][0]) / Lx) * np.cos(2 * math.pi * (Y - cfg["lo"][1]) / Ly)
    u = np.full_like(X, cfg.get("u0", 0.7))
    v = np.full_like(X, cfg.get("v0", -0.4))
    p = np.ones_like(X)
    return rho, u, v, p


def ic_blast(cfg, X, Y, **_):
    """Smooth-edged Gaussian pressure/density bump (drives refinement in AMR parity cases)."""
    xc = cfg.get("blast_centre", (0.5 * (cfg["lo"][0] + cfg["hi"][0]), 0.5 * (cfg["lo"][1] + cfg["hi"][1])))
    s = cfg.get("blast_width", 0.06)
    r2 = ((X - xc[0]) ** 2 + (Y - xc[1]) ** 2) / (s * s)
    rho = 1.0 + 1.0 * np.exp(-r2)
    p = 1.0 + 2.0 * np.exp(-r2)
    z = np.zeros_like(X)
    return rho, z + 0.1, z - 0.05, p


IC = {"uniform": ic_uniform, "sod": ic_sod, "vortex": ic_vortex, "quadrant": ic_quadrant,
      "shock_bubble": ic_shock_bubble, "implosion": ic_implosion, "noise": ic_noise,
      "smooth": ic_smooth, "blast": ic_blast}


def patch_state(cfg, l, P, Q):
    """Conserved U[4][n][n] of patch (l,P,Q) for cfg['ic'] at cell centres (A33)."""
    X, Y = cell_centres(cfg, l, P, Q)
    n = cfg["n"]
    I = np.broadcast_to((P * n + np.arange(n))[None, :], (n, n))
    J = np.broadcast_to((Q * n + np.arange(n))[:, None], (n, n))
    rho, u, v, p = IC[cfg["ic"]](cfg, X, Y, l=l, I=I, J=J)
    return np.ascontiguousarray(to_conserved(rho, u, v, p, cfg.get("gamma", GAMMA)))


def level0_state(cfg, rows=None):
    """Level-0 patches at once: array [NPy][NPx][4][n][n] (big uniform sweeps); rows = (Q0, Q1) restricts
    to patch rows Q0 <= Q < Q1 (one rank's slab)."""
    n = cfg["n"]
    Nx, Ny = cfg["base"]
    dx = (cfg["hi"][0] - cfg["lo"][0]) / Nx
    dy = (cfg["hi"][1] - cfg["lo"][1]) / Ny
    I = np.arange(Nx)
    J = np.arange(Ny) if rows is None else np.arange(rows[0] * n, rows[1] * n)
    Ny = len(J)
    x = cfg["lo"][0] + (I + 0.5) * dx
    y = cfg["lo"][1] + (J + 0.5) * dy
    X, Y = np.meshgrid(x, y)
    II, JJ = np.meshgrid(I, J)
    rho, u, v, p = IC[cfg["ic"]](cfg, X, Y, l=0, I=II, J=JJ)
    U = to_conserved(rho, u, v, p, cfg.get("gamma", GAMMA))   # [4][Ny][Nx]
    U = U.reshape(4, Ny // n, n, Nx // n, n).transpose(1, 3, 0, 2, 4)
    return np.ascontiguousarray(U)


# ----------------------------------------------------------------- the BASELINE.json configs
def _base(**kw):
    c = dict(gamma=GAMMA, characteristic=1, div_order=4, weno_eps=1e-6, theta=0.1, coarsen_frac=0.25,
             coarsen_rule="r2_exact", seed=1, cfl=0.5, regrid_every=4)
    c.update(kw)
    return c


def sod(**kw):
    """BJ configs[0] / D1 with A21 (13 roots of 16 = 208 cells, dx0 = 1/200) and A23 (strip, periodic y)."""
    return _base(name="sod", lo=(0.0, 0.0), hi=(1.04, 0.08), base=(208, 16), n=16, levels=2,
                 bc=("transmissive", "transmissive", "periodic", "periodic"), scheme="weno5", ic="sod",
                 t_end=0.2, **kw)


def vortex(N=1024, n=32, L=10.0, **kw):
    """BJ configs[1] / D2: periodic [0,10]^2, 1024^2 in 32^2 patches, Central4 (shock-free)."""
    c = dict(name="vortex", lo=(0.0, 0.0), hi=(L, L), base=(N, N), n=n, levels=1,
             bc=("periodic",) * 4, scheme="central4", ic="vortex", vortex_centre=(L / 2, L / 2))
    c.update(kw)
    return _base(**c)


def quadrant(N=512, n=16, levels=3, seed=1, **kw):
    """BJ configs[2] / D3: [0,1]^2, 512^2 base, 3 levels, 16^2 patches, transmissive, WENO5-char."""
    c = dict(name="quadrant", lo=(0.0, 0.0), hi=(1.0, 1.0), base=(N, N), n=n, levels=levels,
             bc=("transmissive",) * 4, scheme="weno5", ic="quadrant", seed=seed)
    c.update(kw)
    return _base(**c)


def shock_bubble(Nx=2048, Ny=1024, n=16, levels=4, G=1, **kw):
    """BJ configs[3] / D4 (G=1) and the D4w weak-scaling family (G copies stacked in y)."""
    c = dict(name="shock_bubble", lo=(0.0, 0.0), hi=(2.0, float(G)), base=(Nx, Ny * G), n=n, levels=levels,
             bc=("transmissive", "transmissive", "reflective", "reflective"), scheme="weno5",
             ic="shock_bubble", bubbles=G, mach=1.22)
    c.update(kw)
    return _base(**c)


def sweep(N=4096, n=32, scheme="central4", Ny=None, seed=7, **kw):
    """BJ configs[4] / D5 (and D5w with Ny != N): periodic noise, 1 level."""
    Ny = N if Ny is None else Ny
    c = dict(name="sweep", lo=(0.0, 0.0), hi=(float(N) / 4096.0, float(Ny) / 4096.0), base=(N, Ny), n=n,
             levels=1, bc=("periodic",) * 4, scheme=scheme, ic="noise", seed=seed)
    c.update(kw)
    return _base(**c)


def implosion(N=1024, n=32, scheme="weno5", **kw):
    """NEXT #2, Eq. 13: (-0.3,0.3)^2 periodic, 1024^2, CFL 0.45."""
    c = dict(name="implosion", lo=(-0.3, -0.3), hi=(0.3, 0.3), base=(N, N), n=n, levels=1,
             bc=("periodic",) * 4, scheme=scheme, ic="implosion", cfl=0.45)
    c.update(kw)
    return _base(**c)
