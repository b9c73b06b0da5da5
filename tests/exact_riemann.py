"""Exact Riemann solver for the 1D Euler equations (Toro, ch. 4) -- a pin for the oracle.

SURVEY.md s8(c) O16: pressure function f_K(p) (shock branch for p > p_K,
rarefaction branch otherwise), Newton iteration on f_L + f_R + (u_R - u_L) = 0
to |dp|/p < 1e-14, then sampling at xi = (x - x0)/t.  Independent of oracle/.
"""
from __future__ import annotations

import math

import numpy as np


def _fK(p, rK, pK, cK, g):
    if p > pK:   # shock
        A = 2.0 / ((g + 1.0) * rK)
        B = (g - 1.0) / (g + 1.0) * pK
        s = math.sqrt(A / (p + B))
        return (p - pK) * s, s * (1.0 - 0.5 * (p - pK) / (B + p))
    pr = p / pK   # rarefaction
    f = 2.0 * cK / (g - 1.0) * (pr ** ((g - 1.0) / (2.0 * g)) - 1.0)
    df = 1.0 / (rK * cK) * pr ** (-(g + 1.0) / (2.0 * g))
    return f, df


def star_state(rl, ul, pl, rr, ur, pr, g=1.4):
    cl = math.sqrt(g * pl / rl)
    cr = math.sqrt(g * pr / rr)
    p = max(1e-8, 0.5 * (pl + pr) - 0.125 * (ur - ul) * (rl + rr) * (cl + cr))
    for _ in range(200):
        fl, dfl = _fK(p, rl, pl, cl, g)
        fr, dfr = _fK(p, rr, pr, cr, g)
        dp = (fl + fr + ur - ul) / (dfl + dfr)
        pn = max(1e-12, p - dp)
        if abs(pn - p) / (0.5 * (pn + p)) < 1e-14:
            p = pn
            break
        p = pn
    fl, _ = _fK(p, rl, pl, cl, g)
    fr, _ = _fK(p, rr, pr, cr, g)
    u = 0.5 * (ul + ur) + 0.5 * (fr - fl)
    return p, u


def sample(rl, ul, pl, rr, ur, pr, xi, g=1.4):
    """Return (rho, u, p) arrays at similarity coordinates xi."""
    ps, us = star_state(rl, ul, pl, rr, ur, pr, g)
    cl = math.sqrt(g * pl / rl)
    cr = math.sqrt(g * pr / rr)
    xi = np.asarray(xi, dtype=np.float64)
    rho = np.empty_like(xi)
    u = np.empty_like(xi)
    p = np.empty_like(xi)
    gm = (g - 1.0) / (g + 1.0)
    for e, s in enumerate(xi.flat):
        if s <= us:   # left of contact
            if ps > pl:   # left shock
                rsl = rl * (ps / pl + gm) / (gm * ps / pl + 1.0)
                sl = ul - cl * math.sqrt((g + 1.0) / (2 * g) * ps / pl + (g - 1.0) / (2 * g))
                r_, u_, p_ = (rl, ul, pl) if s <= sl else (rsl, us, ps)
            else:   # left rarefaction
                rsl = rl * (ps / pl) ** (1.0 / g)
                csl = cl * (ps / pl) ** ((g - 1.0) / (2 * g))
                sh, st = ul - cl, us - csl
                if s <= sh:
                    r_, u_, p_ = rl, ul, pl
                elif s >= st:
                    r_, u_, p_ = rsl, us, ps
                else:
                    u_ = 2.0 / (g + 1.0) * (cl + (g - 1.0) / 2.0 * ul + s)
                    c = 2.0 / (g + 1.0) * (cl + (g - 1.0) / 2.0 * (ul - s))
                    r_ = rl * (c / cl) ** (2.0 / (g - 1.0))
                    p_ = pl * (c / cl) ** (2.0 * g / (g - 1.0))
        else:
            if ps > pr:   # right shock
                rsr = rr * (ps / pr + gm) / (gm * ps / pr + 1.0)
                sr = ur + cr * math.sqrt((g + 1.0) / (2 * g) * ps / pr + (g - 1.0) / (2 * g))
                r_, u_, p_ = (rr, ur, pr) if s >= sr else (rsr, us, ps)
            else:
                rsr = rr * (ps / pr) ** (1.0 / g)
                csr = cr * (ps / pr) ** ((g - 1.0) / (2 * g))
                sh, st = ur + cr, us + csr
                if s >= sh:
                    r_, u_, p_ = rr, ur, pr
                elif s <= st:
                    r_, u_, p_ = rsr, us, ps
                else:
                    u_ = 2.0 / (g + 1.0) * (-cr + (g - 1.0) / 2.0 * ur + s)
                    c = 2.0 / (g + 1.0) * (cr - (g - 1.0) / 2.0 * (ur - s))
                    r_ = rr * (c / cr) ** (2.0 / (g - 1.0))
                    p_ = pr * (c / cr) ** (2.0 * g / (g - 1.0))
        rho.flat[e], u.flat[e], p.flat[e] = r_, u_, p_
    return rho, u, p


def shock_speed_right(rl, ul, pl, rr, ur, pr, g=1.4):
    ps, _ = star_state(rl, ul, pl, rr, ur, pr, g)
    cr = math.sqrt(g * pr / rr)
    return ur + cr * math.sqrt((g + 1.0) / (2 * g) * ps / pr + (g - 1.0) / (2 * g))
